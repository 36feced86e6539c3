#!/usr/bin/env bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_parity.py -x -q 2>&1 | tail -4
for v in main NS0 main NS0; do
  if [ $v = main ]; then lib=""; else lib=tools/ab/lib_$v.so; fi
  echo "== $v"; SK_LIB_PATH=$lib timeout 300 python tools/batched_probe.py 2>&1 | grep -E "batched|Error"
done
