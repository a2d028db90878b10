"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]; ix = {x: i for i, x in enumerate(h)}
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try:
        v = float(r[ix['Metric Value']].replace(',', ''))
    except ValueError:
        continue
    k = r[ix['Kernel Name']]
    agg[k][0] += 1; agg[k][1] += v
tot = sum(t for _, t in agg.values())
print(f"# launch list: {sys.argv[1]} (gpu__time_duration.sum, cold-cache serialised; compare shares)")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:5d} launches {t / 1e6:10.3f} ms {100 * t / tot:6.2f}%  {k[:110]}")
