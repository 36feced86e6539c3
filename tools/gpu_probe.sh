timeout 1500 python -m pytest tests -m gpu -q -x -k "decode or batch or graph or append or window or parity" 2>&1 | tail -2
timeout 600 python tools/batched_probe.py 2>&1 | tail -1
SK_LAYERS=32 timeout 600 python tools/graph_probe.py 2>&1 | tail -1
