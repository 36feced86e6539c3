#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for v in main main; do
  echo "== $v"; timeout 300 python tools/append_probe.py 2>&1 | grep -E "bulk|Error"
done
timeout 900 python -m pytest tests -m gpu -x -q -k "append or load or golden or snapshot or chunk or quant" 2>&1 | tail -2
