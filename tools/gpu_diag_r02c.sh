# round-2 (third session) diagnostics: rest of the GPU suite, decode probes,
# K2 phase-B stamps, ncu (stall reasons + source) of the cfg4 K3 and K2
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -q ) > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python tools/pdl_probe.py > gpurun_out/pdl_probe.log 2>&1
timeout 300 python tools/batched_probe.py > gpurun_out/batched_probe.log 2>&1
SK_LIB_PATH=tools/ab/lib_T.so timeout 300 python tools/select_stamp_probe.py > gpurun_out/select_stamps.log 2>&1
SK_LAYERS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 20 -c 1 \
  -o gpurun_out/ncu_c_decode_cfg4 python tools/batched_probe.py > gpurun_out/ncu_decode_cfg4.log 2>&1
SK_LAYERS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:select_kernel -s 4 -c 1 \
  -o gpurun_out/ncu_c_select_cfg4 python tools/batched_probe.py > gpurun_out/ncu_select_cfg4.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -4 gpurun_out/pdl_probe.log; tail -3 gpurun_out/batched_probe.log; tail -8 gpurun_out/select_stamps.log
