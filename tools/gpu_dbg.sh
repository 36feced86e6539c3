for m in 0 5 6; do
  SK_NVCC_EXTRA="-DSK_DBG=$m" SK_FORCE_BUILD=1 python paper_2502_14866_b200/_build.py > /dev/null 2>&1
  echo "== mode $m"; timeout 120 python tools/decode_probe.py 2>&1 | grep -E "select"
done
