# same-box A/B of K4 builds (abtest/<name>/libgdi.so vs the in-tree lib): time and quality
for rep in 1 2; do
  for v in ${AB:-inl} tree; do
    if [ $v = tree ]; then LLP=; else LLP=$PWD/abtest/$v; fi
    LD_LIBRARY_PATH=$LLP timeout 300 python scripts/k4_probe.py random:1000000:4000000:1000001 1 20 random:1000000:4000000:1000001 1 200 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('$v', d['sweeps'], round(d['ms'],3), d.get('sm_mhz'), d['cut'][:4], d['imbalance'][:4])
  else: print(l.rstrip()[:200])
"
  done
done
