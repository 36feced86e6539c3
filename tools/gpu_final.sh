# end-of-round refresh: GPU tests, smoke, bench, launch list, ncu of the new K1b gather kernel
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_workload.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_kernel -c 1 -o gpurun_out/ncu_gather_kernel python tools/chunk_probe.py > gpurun_out/ncu_gather.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -1 gpurun_out/bench.log | cut -c1-400
