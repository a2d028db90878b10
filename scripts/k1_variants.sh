# exact-kernel timing per forced k1_window variant (1000 sweeps, R=1024)
for v in ${VARIANTS:-"" window_sync}; do
  GDI_FORCE_KERNEL=$v timeout 300 python scripts/k1_timing.py ${CONFIGS:-G22,G1,G55,G81pm1} 1024 1000 2>&1 | grep -o '"config": "[A-Za-z0-9]*".*"ms": [0-9.]*' | sed "s/^/[${v:-default}] /"
done
