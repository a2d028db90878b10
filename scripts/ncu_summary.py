"""Summarise an ncu --set full report (raw page) into text for profiles/.

usage: python scripts/ncu_summary.py REPORT TITLE [UPDATES_PER_LAUNCH [VISITS_PER_CHAIN]]
With the spin updates one launch performs, also prints the per-update DRAM
bytes, L2 bytes (lts__t_sectors x 32) and shared-memory wavefronts; with the
visits of one replica chain, the SM cycles per visit (exact mode)."""
import csv, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sectors.sum',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'sm__inst_executed.avg.per_cycle_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'launch__shared_mem_per_block_dynamic', 'sm__cycles_elapsed.avg', 'smsp__sass_inst_executed_op_shared_ld.sum',
        'smsp__sass_inst_executed_op_global_ld.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']

SCALE = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'sector': 1, '': 1, 'inst': 1, 'cycle': 1}


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2]


def values(rep):
    h, u, v = raw(rep)
    d = {}
    for i, k in enumerate(h):
        try:
            d[k] = float(v[i].replace(',', '')) * SCALE.get(u[i], 1)
        except ValueError:
            d[k] = v[i]
    return h, u, v, d


def main():
    rep, title = sys.argv[1], sys.argv[2]
    upl = float(sys.argv[3]) if len(sys.argv) > 3 else None
    vpc = float(sys.argv[4]) if len(sys.argv) > 4 else None
    h, u, v, d = values(rep)
    ix = {x: i for i, x in enumerate(h)}
    print(f"# {title}\n# source: {rep} (ncu --set full, one launch)")
    print(f"kernel: {v[ix['Kernel Name']] if 'Kernel Name' in ix else '?'}")
    for k in KEYS:
        if k in ix:
            print(f"{k:58s} {v[ix[k]]:>22s} {u[ix[k]]}")
    dram = d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
    l2 = 32 * d.get('lts__t_sectors.sum', 0)
    wf = d.get('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 0)
    print(f"{'DRAM bytes per launch (read + write)':58s} {dram:>22.0f}")
    print(f"{'L2 bytes per launch (lts__t_sectors x 32)':58s} {l2:>22.0f}")
    if upl:
        print(f"{'updates per launch':58s} {upl:>22.0f}")
        print(f"{'DRAM bytes per update':58s} {dram / upl:>22.4f}")
        print(f"{'L2 bytes per update':58s} {l2 / upl:>22.4f}")
        print(f"{'shared-memory wavefronts per update':58s} {wf / upl:>22.4f}")
    if vpc:
        print(f"{'SM cycles per visit of one replica chain':58s} {d.get('sm__cycles_elapsed.avg', 0) / vpc:>22.2f}")
    stalls = [(x, float(v[i].replace(',', '') or 0)) for i, x in enumerate(h)
              if x.startswith('smsp__pcsamp_warps_issue_stalled_') and not x.endswith('not_issued')]
    tot = sum(s for _, s in stalls) or 1
    print("warp-state samples (top):")
    for x, s in sorted(stalls, key=lambda t: -t[1])[:10]:
        print(f"  {x[33:]:40s} {100 * s / tot:5.1f}%")


if __name__ == '__main__':
    main()
