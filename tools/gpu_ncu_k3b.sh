#!/usr/bin/env bash
# one full-set ncu capture of the staged K3 (cfg4 batched, one CTA per stream)
cd "$(dirname "$0")/.."
SK_LAYERS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -s 20 -c 1 \
  -o gpurun_out/ncu_k3_staged -f python tools/batched_probe.py > gpurun_out/ncu_k3_staged.log 2>&1
tail -3 gpurun_out/ncu_k3_staged.log
