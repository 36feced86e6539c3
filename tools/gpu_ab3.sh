for v in "1 16" "2 8" "2 16" "1 8"; do set -- $v
  SK_FORCE_BUILD=1 SK_NVCC_EXTRA="-DSK_SEL_MINB=$1 -DSK_SEL_LOG_PER_SLOT=$2" python paper_2502_14866_b200/_build.py > /dev/null 2>&1
  echo "minb $1 log/slot $2"; timeout 300 python tools/decode_probe.py 2>&1 | grep select
done
