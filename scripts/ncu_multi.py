"""Key metrics of every kernel in an ncu --set full report (one row per launch).

usage: python scripts/ncu_multi.py REPORT TITLE
"""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sectors.sum',
        'smsp__inst_executed.sum', 'sm__inst_executed.avg.per_cycle_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__grid_size', 'launch__block_size',
        'launch__registers_per_thread', 'launch__shared_mem_per_block_dynamic',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']
rep, title = sys.argv[1], sys.argv[2]
rows = list(csv.reader(subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                                      text=True).stdout.splitlines()))
h, u = rows[0], rows[1]
ix = {x: i for i, x in enumerate(h)}
print(f"# {title}\n# source: {rep} (ncu --set full)")
for r in rows[2:]:
    print(f"\nkernel: {r[ix['Kernel Name']]}")
    for k in KEYS:
        if k in ix:
            print(f"  {k:56s} {r[ix[k]]:>20s} {u[ix[k]]}")
