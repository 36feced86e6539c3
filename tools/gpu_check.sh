timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for d in 0 1 2; do echo "dbg $d"; SK_SEL_DEBUG=$d timeout 300 python tools/decode_probe.py 2>&1 | grep -E "select"; done
