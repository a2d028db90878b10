for v in "4 128" "2 256" "8 64"; do set -- $v
GDI_WINDOW_NR=$1 GDI_WINDOW_SEGL=$2 timeout 120 python scripts/k1_timing.py G22,G1 1024 1000 2>&1 | grep -o '"config": "[A-Za-z0-9]*".*"ms": [0-9.]*' | sed "s/^/nr=$1 segl=$2 /"
done
