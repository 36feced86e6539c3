# round-2 (final) artefacts: GPU tests, smoke, bench (both arms), launch
# list, ncu of every kernel (cfg2 layer) plus the staged K3 and K1 fast path
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_workload.py > /dev/null 2>&1
for k in select_kernel decode_kernel append_kernel append_one_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/ncu_r02d_$k python tools/profile_workload.py > gpurun_out/ncu_$k.log 2>&1
done
SK_LAYERS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 20 -c 1 \
  -o gpurun_out/ncu_r02d_decode_kernel_cfg4 python tools/batched_probe.py > gpurun_out/ncu_decode_cfg4.log 2>&1
timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis --section WarpStateStats --section LaunchStats --section Occupancy --section InstructionStats --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active --clock-control none -k regex:prefill_kernel -c 1 -o gpurun_out/ncu_r02d_prefill_kernel python tools/profile_workload.py > gpurun_out/ncu_prefill_kernel.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -1 gpurun_out/bench.log | cut -c1-300; tail -1 gpurun_out/bench_ref.log | cut -c1-300
