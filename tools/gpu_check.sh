for d in 3 1; do echo "dbg $d"; SK_SEL_DEBUG=$d timeout 300 python tools/decode_probe.py 2>&1 | grep -E "select|floor"; done
