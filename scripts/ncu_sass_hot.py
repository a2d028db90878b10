"""Per-SASS-instruction hot list of an ncu report (source page, SASS view):
address, instruction, executions, stall samples; optional range dump."""
import csv, subprocess, sys

def rows(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout.splitlines()
    r = list(csv.reader(out[1:]))
    h = r[0]
    return h, r[1:]

def main():
    rep = sys.argv[1]
    h, rs = rows(rep)
    ia, isrc, isam, iex = h.index('Address'), h.index('Source'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
    tot = sum(int(r[isam] or 0) for r in rs) or 1
    if len(sys.argv) > 2 and sys.argv[2] == 'dump':
        lo, hi = int(sys.argv[3]), int(sys.argv[4])
        for k, r in enumerate(rs[lo:hi], lo):
            print(f"{k:5d} {int(r[iex] or 0):>12d} {int(r[isam] or 0):>6d} {r[isrc]}")
        return
    top = sorted(range(len(rs)), key=lambda k: -int(rs[k][isam] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]
    for k in sorted(top):
        r = rs[k]
        print(f"{k:5d} {int(r[iex] or 0):>12d} {100*int(r[isam] or 0)/tot:5.1f}% {r[isrc]}")

main()
