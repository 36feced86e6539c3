# decode/select probes + one ncu --set full capture per hot kernel
set -x
timeout 300 python tools/decode_probe.py > gpurun_out/probe.log 2>&1
for k in decode_kernel select_kernel append_one_kernel prefill_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/ncu_$k python tools/profile_workload.py > gpurun_out/ncu_$k.log 2>&1
done
cat gpurun_out/probe.log
