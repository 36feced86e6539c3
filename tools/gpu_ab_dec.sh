SK_LIB_OUT=/tmp/libA.so SK_OBJ_DIR=objA SK_SRC_OVERRIDE="decode.cu=tools/ab/decode_prev.cu" python paper_2502_14866_b200/_build.py > /dev/null 2>&1 || echo "build A failed"
SK_LIB_OUT=/tmp/libC.so SK_OBJ_DIR=objC SK_NVCC_EXTRA="-DSK_DEC_CL=16" python paper_2502_14866_b200/_build.py > /dev/null 2>&1 || echo "build C failed"
cp paper_2502_14866_b200/libsparsekv_b200.so /tmp/libB.so
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
SK_LIB_PATH=/tmp/libC.so timeout 600 python -m pytest tests -m gpu -x -q -k decode 2>&1 | tail -2
for i in 1 2; do for L in A B C; do echo "lib $L"; SK_LIB_PATH=/tmp/lib$L.so timeout 300 python tools/decode_probe.py 2>&1 | grep -E "fuse=0"; done; done
