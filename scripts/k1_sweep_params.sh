# k1_window producer tuning: lanes per stream (KP), segment length (SEGL),
# rounds buffered (NR); 1000 sweeps, timing only (scripts/k1_timing.py)
for c in ${CONFIGS:-G22 G55}; do
  for v in ${VARIANTS:-"1 128 2" "4 128 4" "4 64 4" "4 64 8" "4 32 8" "4 128 2" "2 128 4"}; do
    set -- $v
    GDI_WINDOW_KP=$1 GDI_WINDOW_SEGL=$2 GDI_WINDOW_NR=$3 timeout 120 python scripts/k1_timing.py $c 1024 ${SWEEPS:-1000} 2>&1 | grep -o '"ms": [0-9.]*' | sed "s/^/$c kp=$1 segl=$2 nr=$3 /"
  done
done
