timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu --batch 0 --decode-steps 8 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill', d['value'], 'e2e', d['e2e'])"
