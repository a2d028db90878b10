# Round-2 final profile set (one GPU): bench lines of every config and the
# reference arm, the bench launch list, ncu --set full of the kernels changed
# late in the round (k1_block on G55 and G1, the rows variant on G81+-1,
# k2_chains on G55). Outputs in gpurun_out/r02e_*.
set -x
for c in G22 G1 G55 G81pm1; do python bench.py --config $c > gpurun_out/r02e_bench_$c.json 2> gpurun_out/r02e_bench_$c.err; done
python bench.py --config M1 --mode throughput > gpurun_out/r02e_bench_M1.json 2> gpurun_out/r02e_bench_M1.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02e_bench_reference.json 2> gpurun_out/r02e_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02e_bench_launches.log 2>&1
for c in G55 G1 G81pm1; do
ncu --set full --import-source on --clock-control none -k regex:k1_block -c 1 -f -o gpurun_out/r02e_k1_block_$c \
  python scripts/k1_timing.py $c 1024 1000 > gpurun_out/r02e_k1_$c.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k2_chains -c 1 -f -o gpurun_out/r02e_k2_chains_G55 \
  python scripts/k2_probe2.py G55 1024 1000 > gpurun_out/r02e_k2_G55.log 2>&1
