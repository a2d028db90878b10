# Round-2 closing captures after the lane-0 scan and the hoisted tail chain
# (K2, K4): bench lines of G22 (default), G55 and M1, ncu of k2_chains (G22)
# and k4_sweep / k4_finish (M1, warm L2). Outputs in gpurun_out/r02f_*.
set -x
python bench.py > gpurun_out/r02f_bench_G22.json 2> gpurun_out/r02f_bench_G22.err
python bench.py --config G55 > gpurun_out/r02f_bench_G55.json 2> gpurun_out/r02f_bench_G55.err
python bench.py --config M1 --mode throughput > gpurun_out/r02f_bench_M1.json 2> gpurun_out/r02f_bench_M1.err
ncu --set full --import-source on --clock-control none -k regex:k2_chains -c 1 -f -o gpurun_out/r02f_k2_chains_G22 \
  python scripts/k2_probe2.py G22 1024 1000 > gpurun_out/r02f_k2.log 2>&1
for K in k4_sweep k4_finish; do
ncu --set full --import-source on --clock-control none --cache-control none -k regex:$K -s 10 -c 1 -f -o gpurun_out/r02f_${K}_M1 \
  python scripts/k4_probe.py random:1000000:4000000:1000001 1 20 > gpurun_out/r02f_$K.log 2>&1
done
