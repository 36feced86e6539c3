# ncu of K2 phase A alone (ablation build) and the full K2, source-level stall sampling
mkdir -p gpurun_out
SK_LIB_PATH=tools/ab/lib_A1.so timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:select_kernel -s 5 -c 1 -o gpurun_out/ncu_k2_phaseA python tools/select_probe.py cfg2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:select_kernel -s 5 -c 1 -o gpurun_out/ncu_k2_full python tools/select_probe.py cfg2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:decode_kernel -s 5 -c 1 -o gpurun_out/ncu_k3 python tools/profile_workload.py > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
