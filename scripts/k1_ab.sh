# same-box A/B of exact-kernel builds: abtest/<name>/libgdi.so vs the in-tree lib
# (pyising resolves libgdi.so through RUNPATH, so LD_LIBRARY_PATH wins)
for rep in 1 2; do
  for v in ${AB:-A}; do
    LD_LIBRARY_PATH=$PWD/abtest/$v timeout 300 python scripts/k1_timing.py ${CONFIGS:-G22,G1,G55,G81pm1} 1024 1000 2>&1 | grep -o '"config": "[A-Za-z0-9]*".*"ms": [0-9.]*' | sed "s/^/[$v] /"
  done
  timeout 300 python scripts/k1_timing.py ${CONFIGS:-G22,G1,G55,G81pm1} 1024 1000 2>&1 | grep -o '"config": "[A-Za-z0-9]*".*"ms": [0-9.]*' | sed "s/^/[tree] /"
done
