set -x
export SK_NVCC_EXTRA=-DSK_DECODE_TIMING SK_FORCE_BUILD=1
python paper_2502_14866_b200/_build.py > gpurun_out/tl_build.log 2>&1
timeout 300 python tools/decode_timeline.py > gpurun_out/timeline.log 2>&1
cat gpurun_out/timeline.log
timeout 300 python tools/decode_probe.py 2>&1 | grep -E "select|pps=2" 
