timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/decode_probe.py 2>&1 | grep -E "select|fuse=0|floor|rror"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill ms', d['value'], d['roofline']['frac'], 'decode', d['decode']['us_per_step'])"
