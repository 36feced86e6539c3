# round artefacts: GPU tests, smoke, full bench, launch list, ncu --set full of each hot kernel
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_workload.py > /dev/null 2>&1
for k in decode_kernel select_kernel append_kernel append_one_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/ncu_$k python tools/profile_workload.py > gpurun_out/ncu_$k.log 2>&1
done
# the full set's source-counter pass does not complete on the TMEM-P prefill kernel: section list
timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis --section WarpStateStats --section LaunchStats --section Occupancy --section InstructionStats --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active --clock-control none -k regex:prefill_kernel -c 1 -o gpurun_out/ncu_prefill_kernel python tools/profile_workload.py > gpurun_out/ncu_prefill_kernel.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -1 gpurun_out/bench.log
