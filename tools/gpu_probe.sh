SK_CTX=32768 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"append_kernel" -c 1 -o gpurun_out/ncu_k1b python tools/profile_workload.py > /dev/null 2>&1
ls gpurun_out/ncu_k1b.ncu-rep
