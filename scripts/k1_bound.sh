for c in G22 G55; do
  for d in 4 12; do
    GDI_PIPE_DEBUG=$d timeout 120 python scripts/k1_timing.py $c 1024 1000 2>&1 | grep -E "prof|ms" | sed "s/^/$c debug=$d /"
  done
done
