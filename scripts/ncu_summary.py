"""Summarise an ncu --set full report (raw page) + a launch-list CSV into text for profiles/."""
import csv, subprocess, sys
from collections import defaultdict

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'l1tex__t_bytes.sum', 'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'sm__inst_executed.avg.per_cycle_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'launch__shared_mem_per_block_dynamic', 'sm__cycles_elapsed.avg', 'smsp__sass_inst_executed_op_shared_ld.sum',
        'smsp__sass_inst_executed_op_global_ld.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']

def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2]

def main():
    rep, title = sys.argv[1], sys.argv[2]
    h, u, v = raw(rep)
    ix = {x: i for i, x in enumerate(h)}
    print(f"# {title}\n# source: {rep} (ncu --set full --clock-control none, one launch)")
    print(f"kernel: {v[ix['Kernel Name']] if 'Kernel Name' in ix else '?'}")
    for k in KEYS:
        if k in ix:
            print(f"{k:58s} {v[ix[k]]:>22s} {u[ix[k]]}")
    stalls = [(x, float(v[i].replace(',', '') or 0)) for i, x in enumerate(h)
              if x.startswith('smsp__pcsamp_warps_issue_stalled_') and not x.endswith('not_issued')]
    tot = sum(s for _, s in stalls) or 1
    print("warp-state samples (top):")
    for x, s in sorted(stalls, key=lambda t: -t[1])[:10]:
        print(f"  {x[33:]:40s} {100 * s / tot:5.1f}%")

if __name__ == '__main__':
    main()
