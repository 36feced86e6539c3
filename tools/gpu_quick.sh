# quick GPU loop: tests (optionally filtered by $1) + decode probes
timeout 1500 python -m pytest tests -m gpu -q -x ${1:+-k "$1"} 2>&1 | tail -5
SK_LIB_PATH=tools/ab/lib_DT.so timeout 300 python tools/decode_stamp_probe.py 2>&1 | tail -4
timeout 300 python tools/select_probe.py 2>&1 | grep case
timeout 600 python tools/pdl_probe.py 2>&1 | tail -4
SK_LAYERS=32 timeout 600 python tools/graph_probe.py 2>&1 | tail -1
