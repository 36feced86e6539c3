SK_LIB_OUT=/tmp/libA.so SK_OBJ_DIR=objA SK_NVCC_EXTRA="-DSK_TMEM_P=1" python paper_2502_14866_b200/_build.py > /dev/null 2>&1 || echo "build A failed"
cp paper_2502_14866_b200/libsparsekv_b200.so /tmp/libB.so
SK_LIB_PATH=/tmp/libA.so timeout 900 python -m pytest tests -m gpu -x -q -k "prefill or blockwise or engine or shards" 2>&1 | tail -2
for i in 1 2 3; do
  SK_LIB_PATH=/tmp/libA.so timeout 300 python tools/prefill_probe.py 2>&1 | tail -1
  SK_LIB_PATH=/tmp/libB.so timeout 300 python tools/prefill_probe.py 2>&1 | tail -1
done
