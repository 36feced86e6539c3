# K2 A/B: GPU suite + decode probes + select probe
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -q -x ) > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python tools/pdl_probe.py > gpurun_out/pdl_probe.log 2>&1
timeout 300 python tools/select_probe.py > gpurun_out/select_probe.log 2>&1
timeout 300 python tools/batched_probe.py > gpurun_out/batched_probe.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; grep -B2 -A25 "^E " gpurun_out/pytest_gpu.log | head -40; tail -n4 gpurun_out/pdl_probe.log; tail -n2 gpurun_out/select_probe.log; tail -n2 gpurun_out/batched_probe.log
