# Round-2 (late) profile set, one GPU: bench lines of every config, the bench
# launch list, ncu --set full of the changed kernels (k2_chains G22, k4_sweep +
# k4_finish M1 with warm L2, the K3 evaluation kernels on G22 x1024 and M1).
# Outputs in gpurun_out/r02c_*; scripts/make_traffic.py turns the captures
# into profiles/roofline_traffic.json.
set -x
for c in G22 G1 G55 G81pm1; do python bench.py --config $c > gpurun_out/r02c_bench_$c.json 2> gpurun_out/r02c_bench_$c.err; done
python bench.py --config M1 --mode throughput > gpurun_out/r02c_bench_M1.json 2> gpurun_out/r02c_bench_M1.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02c_bench_reference.json 2> gpurun_out/r02c_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02c_bench_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k2_chains -c 1 -f -o gpurun_out/r02c_k2_chains_G22 \
  python scripts/k2_probe2.py G22 1024 1000 > gpurun_out/r02c_k2.log 2>&1
for K in k4_sweep k4_finish; do
ncu --set full --import-source on --clock-control none --cache-control none -k regex:$K -s 10 -c 1 -f -o gpurun_out/r02c_${K}_M1 \
  python scripts/k4_probe.py random:1000000:4000000:1000001 1 20 > gpurun_out/r02c_$K.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k3_ -s 8 -c 2 -f -o gpurun_out/r02c_k3_G22 \
  python scripts/k3_probe.py random:2000:19990:22 1024 4 > gpurun_out/r02c_k3_G22.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k3_ -s 8 -c 2 -f -o gpurun_out/r02c_k3_M1 \
  python scripts/k3_probe.py random:1000000:4000000:1000001 1 4 > gpurun_out/r02c_k3_M1.log 2>&1
