timeout 1500 python -m pytest tests -m gpu -q -x -k "decode or graph or batch or parity or edges or window" 2>&1 | tail -2
SK_LIB_PATH=tools/ab/lib_DT.so timeout 300 python tools/decode_stamp_probe.py 2>&1 | tail -2
timeout 600 python tools/pdl_probe.py 2>&1 | tail -4
