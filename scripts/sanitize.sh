# compute-sanitizer runs: memcheck + racecheck + synccheck of the
# exact kernel on G1 x 8 replicas (bit-exact against the oracle too), memcheck of
# the pooled kernels. Logs in gpurun_out/r02_sanitizer_*.txt.
CS=compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 20 python scripts/sanitize_run.py exact 8 50 > gpurun_out/r02_sanitizer_k1_block_$tool.txt 2>&1
done
GDI_FORCE_KERNEL=window timeout 900 $CS --tool racecheck --print-limit 20 python scripts/sanitize_run.py exact 8 50 > gpurun_out/r02_sanitizer_k1_window_racecheck.txt 2>&1
timeout 900 $CS --tool memcheck --print-limit 20 python scripts/sanitize_run.py pooled 8 20 > gpurun_out/r02_sanitizer_k2_chains_memcheck.txt 2>&1
timeout 900 $CS --tool memcheck --print-limit 20 python scripts/sanitize_run.py part 1 5 > gpurun_out/r02_sanitizer_k4_memcheck.txt 2>&1
timeout 900 $CS --tool racecheck --print-limit 5 python scripts/sanitize_run.py pooled 8 5 > gpurun_out/r02_sanitizer_k2_chains_racecheck.txt 2>&1
for f in gpurun_out/r02_sanitizer_*.txt; do echo "== $f"; tail -3 $f; done
