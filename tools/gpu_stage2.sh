#!/usr/bin/env bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q 2>&1 | tail -2
for v in main main; do
  echo "== $v"; timeout 300 python tools/batched_probe.py 2>&1 | grep -E "batched|Error"
done
