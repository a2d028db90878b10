# Round-2 profile set (one GPU): bench launch list, ncu --set full of the three
# sweep kernels (k1_block G22 exact, k2_chains G22 pooled, k4_sweep + k4_finish
# M1 with warm L2) and the L2 read-bandwidth probe. Outputs in gpurun_out/r02_*.
set -x
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k1_block -c 1 -f -o gpurun_out/r02_k1_block_G22 \
  python scripts/k1_timing.py G22 1024 1000 > gpurun_out/r02_k1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k2_chains -c 1 -f -o gpurun_out/r02_k2_chains_G22 \
  python scripts/k2_probe2.py G22 1024 1000 > gpurun_out/r02_k2.log 2>&1
TAG=r02 bash scripts/k4_prof.sh
python -c "
import sys; sys.path.insert(0,'.')
import json, paper_1908_00210_b200 as pi
v=[pi.probe_l2_bandwidth(48<<20, 50) for _ in range(5)]
print(json.dumps({'l2_read_gbs_runs': v, 'l2_read_gbs': max(v), 'method': 'probe.cu l2_read: 16-byte __ldcg loads of a 48 MB buffer (warm, L2-resident), grid 4 CTAs/SM x 512 threads, 50 passes, CUDA events; max of 5 runs'}))
" > gpurun_out/r02_l2_peak.json 2>&1
