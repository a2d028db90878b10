# k1 profile: per-phase sweep times and one ncu --set full capture of the exact kernel (G22 x 1024 x 1000)
CFG=${CFG:-G22}
python scripts/k1_phase.py $CFG > gpurun_out/phase_$CFG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:${KERNEL:-k1_block} -c 1 -f -o gpurun_out/${TAG:-k1b}_$CFG \
  python scripts/k1_timing.py $CFG 1024 1000 > gpurun_out/ncu_$CFG.log 2>&1
