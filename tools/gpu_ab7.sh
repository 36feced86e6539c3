SK_LIB_OUT=/tmp/libA.so SK_OBJ_DIR=objA SK_NVCC_EXTRA="-DSK_POLY_FROM=48" python paper_2502_14866_b200/_build.py > /dev/null 2>&1 || echo "build A failed"
SK_LIB_OUT=/tmp/libC.so SK_OBJ_DIR=objC SK_NVCC_EXTRA="-DSK_POLY_FROM=56" python paper_2502_14866_b200/_build.py > /dev/null 2>&1 || echo "build C failed"
cp paper_2502_14866_b200/libsparsekv_b200.so /tmp/libB.so
SK_LIB_PATH=/tmp/libA.so timeout 900 python -m pytest tests -m gpu -x -q -k "prefill or blockwise" 2>&1 | tail -1
for i in 1 2; do for L in A B C; do
  SK_LIB_PATH=/tmp/lib$L.so timeout 300 python tools/prefill_probe.py 2>&1 | tail -1
done; done
