# same-box A/B of K4 builds (abtest/<name>/libgdi.so vs in-tree): time and balance
for v in ${AB:-D1} tree; do
  for rec in random:1000000:4000000:1000001 random:100000:400000:77; do
    if [ $v = tree ]; then LLP=; else LLP=$PWD/abtest/$v; fi
    LD_LIBRARY_PATH=$LLP timeout 200 python scripts/k4_probe.py $rec ${R:-1} 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('$v', '$rec'.split(':')[1], round(d['ms'],3), d['cut'][:4], d['imbalance'][:4], d['imb_trace_r0'][-4:])
"
  done
done
