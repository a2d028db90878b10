# K4 global-tail length vs time and balance (M1 and a 100k graph, several seeds)
for t in 32 16 8 4; do
  for rec in random:1000000:4000000:1000001 random:100000:400000:77; do
    GDI_K4_TAIL=$t timeout 200 python scripts/k4_probe.py $rec 4 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('tail=$t', '$rec'.split(':')[1], round(d['ms'],3), d['cut'][:4], d['imbalance'][:4], d['imb_trace_r0'][-5:])
"
  done
done
