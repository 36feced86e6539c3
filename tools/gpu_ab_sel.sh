# A/B of K2 builds: tools/ab/libA*.so vs the in-tree library (B), select_probe x2
for i in 1 2; do
  for L in tools/ab/libA1.so tools/ab/libA2.so tools/ab/libA3.so; do
    echo $L; SK_LIB_PATH=$L timeout 300 python tools/select_probe.py 2>&1 | grep select
  done
  echo B; timeout 300 python tools/select_probe.py 2>&1 | grep select
done
