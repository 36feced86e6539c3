# A/B of K2 builds: tools/ab/lib_A*.so vs the in-tree library (B), select_probe x2
mkdir -p gpurun_out
for i in 1 2; do
  for L in tools/ab/lib_A*.so; do
    echo $L; SK_LIB_PATH=$L timeout 300 python tools/select_probe.py 2>&1 | grep case
  done
  echo B; timeout 300 python tools/select_probe.py 2>&1 | grep case
done
