#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for v in main SF0 main SF0; do
  if [ $v = main ]; then lib=""; else lib=tools/ab/lib_$v.so; fi
  echo "== $v"; SK_LIB_PATH=$lib timeout 300 python tools/append_probe.py 2>&1 | grep -E "bulk|Error"
done
