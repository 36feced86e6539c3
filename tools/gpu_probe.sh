timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python tools/batched_probe.py 2>&1 | tail -1
SK_LAYERS=32 timeout 600 python tools/graph_probe.py 2>&1 | tail -1
