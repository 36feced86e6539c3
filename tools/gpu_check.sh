B='timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --decode-steps 8 --layers 8'
P='import json,sys; d=json.loads(sys.stdin.read()); print("prefill ms", d["value"], d["roofline"]["frac"], "decode", d["decode"]["us_per_step"])'
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/decode_probe.py 2>&1 | grep -E "fuse=0"
for v in "0 64" "0 48" "1 64" "1 48" "0 40"; do set -- $v
  SK_FORCE_BUILD=1 SK_NVCC_EXTRA="-DSK_PF_ORDER=$1 -DSK_POLY_FROM=$2" python paper_2502_14866_b200/_build.py > /dev/null 2>&1
  echo "order $1 poly $2"; $B 2>&1 | tail -1 | python -c "$P"
done
