timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python tools/decode_probe.py 2>&1 | tail -6
