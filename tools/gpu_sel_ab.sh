#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for v in main SELOLD main SELOLD; do
  if [ $v = main ]; then lib=""; else lib=tools/ab/lib_$v.so; fi
  echo "== $v"; SK_LIB_PATH=$lib timeout 300 python tools/batched_probe.py 2>&1 | grep -E "batched|Error"
  SK_LIB_PATH=$lib timeout 300 python tools/pdl_probe.py 2>&1 | grep -E "pdl=1|Error"
done
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_select_bound.py tests/test_gpu_recall.py -x -q 2>&1 | tail -2
