"""Per-source-line instruction and stall-sample shares of an ncu report (source page, CUDA+SASS view)."""
import csv, subprocess, sys

out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout.splitlines()
f, agg = None, []
for r in csv.reader(out):
    if r and r[0] == 'File Path':
        f = r[1].split('/')[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        try:
            agg.append((float(r[7] or 0), float(r[4] or 0), f, r[0], r[1]))
        except ValueError:
            pass
ti = sum(a[0] for a in agg) or 1
ts = sum(a[1] for a in agg) or 1
print(f"instructions {ti:.0f}, stall samples {ts:.0f}")
key = 1 if len(sys.argv) > 3 and sys.argv[3] == 'samples' else 0
for a in sorted(agg, key=lambda a: -a[key])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"inst {a[0] / ti:6.1%}  samples {a[1] / ts:6.1%}  {a[2]}:{a[3]:>4} {a[4][:100]}")
