# K4 launch list + one full capture each of k4_sweep and k4_finish (M1, 20 sweeps), warm L2 (--cache-control none)
R=random:1000000:4000000:1000001
TAG=${TAG:-k4}
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python scripts/k4_probe.py $R 1 20 > gpurun_out/${TAG}_launches.log 2>&1
for K in k4_sweep k4_finish; do
ncu --set full --import-source on --clock-control none --cache-control none -k regex:$K -s 10 -c 1 -f -o gpurun_out/${TAG}_${K}_M1 \
  python scripts/k4_probe.py $R 1 20 > gpurun_out/${TAG}_$K.log 2>&1
done
