# decode A/B: GPU suite + cfg2 / cfg4 decode probes
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -q -x ) > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python tools/pdl_probe.py > gpurun_out/pdl_probe.log 2>&1
timeout 300 python tools/batched_probe.py > gpurun_out/batched_probe.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; grep -B2 -A25 "^E " gpurun_out/pytest_gpu.log | head -60; tail -4 gpurun_out/pdl_probe.log; tail -3 gpurun_out/batched_probe.log
