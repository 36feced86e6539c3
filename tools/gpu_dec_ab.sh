#!/usr/bin/env bash
# decode K3 ablations in the PDL-chained graph (tools/pdl_probe.py)
cd "$(dirname "$0")/.."
for v in main DA2 DA3 DA4 DM2; do
  if [ $v = main ]; then lib=""; else lib=tools/ab/lib_$v.so; fi
  echo "== $v"; SK_LIB_PATH=$lib timeout 300 python tools/pdl_probe.py 2>&1 | grep -E "step|Error" 
done
