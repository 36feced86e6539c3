timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/decode_probe.py 2>&1 | grep -E "fuse=0"
SK_DEC_DEBUG=3 timeout 300 python tools/decode_probe.py 2>&1 | grep -E "fuse=0"
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --decode-steps 16 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill', d['value'], 'decode', d['decode']['us_per_step'], 'batched', d['decode_batched']['us_per_step'], d['decode_batched']['roofline']['frac'])"
