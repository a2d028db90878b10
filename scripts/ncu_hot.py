"""Summarise an ncu --page source --csv --print-source sass dump: top SASS lines by samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
top = sorted(data, key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
agg = {c: sum(float(r[ix[c]] or 0) for r in data) for c in stall_cols}
print("total samples", tot)
print("stalls:", ", ".join(f"{c[6:]}={v/tot:.1%}" for c, v in sorted(agg.items(), key=lambda x: -x[1]) if v > 0.005 * tot))
for r in top:
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    st = sorted(((float(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{r[ix['Address']]:>6} {s/tot:6.1%} {r[ix['Source']][:60]:60s} " + " ".join(f"{n}={v/max(s,1):.0%}" for v, n in st if v))
