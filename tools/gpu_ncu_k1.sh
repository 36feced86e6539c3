#!/usr/bin/env bash
cd "$(dirname "$0")/.."
timeout 900 ncu --set full --import-source on --clock-control none -k regex:append_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_k1_fast -f python tools/append_probe.py > gpurun_out/ncu_k1_fast.log 2>&1
tail -2 gpurun_out/ncu_k1_fast.log
