# k1_window producer segment length at a fixed 2048-draw ring (rounds need not divide it)
for sl in 128 160 192 224 256; do
  GDI_WINDOW_RING=2048 GDI_WINDOW_SEGL=$sl timeout 120 python scripts/k1_timing.py ${CONFIGS:-G22,G1} 1024 1000 2>&1 | grep -o '"config": "[A-Za-z0-9]*".*"ms": [0-9.]*' | sed "s/^/segl=$sl /"
done
