timeout 300 python tools/decode_probe.py 2>&1 | grep -E "select|decode|floor"
for k in decode_kernel select_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/ncu2_$k python tools/profile_workload.py > /dev/null 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill ms', d['value'], d['roofline']['frac'], 'decode', d['decode']['us_per_step'])"
