mkdir -p gpurun_out
timeout 300 python tools/select_probe.py > gpurun_out/select_probe.log 2>&1
SK_LAYERS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg4_launches.csv python tools/batched_probe.py > /dev/null 2>&1
SK_LAYERS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 20 -c 1 \
  -o gpurun_out/ncu_d_decode_cfg4 python tools/batched_probe.py > gpurun_out/ncu_decode_cfg4.log 2>&1
cat gpurun_out/select_probe.log | tail -6
