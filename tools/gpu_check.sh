timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/decode_probe.py 2>&1 | grep -E "fuse=0"
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --decode-steps 16 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill', d['value'], 'decode', d['decode']['us_per_step'], 'batched', d['decode_batched']['us_per_step'], d['decode_batched']['roofline']['frac'])"
SK_SWEEP_OUT=gpurun_out/sweep_r01b.jsonl timeout 1800 python tools/sweep.py 2>&1 | cut -c 1-60,200-400 | tail -12
