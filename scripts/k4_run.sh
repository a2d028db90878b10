# K4 probe: M1 / 100k timing + quality across tuning knobs, then the K4 tests.
# CFGS: space-separated refresh,cta_tail,tail,fresh tuples
for cfg in ${CFGS:-1,4,16,1 1,4,16,0 -1,4,16,1}; do
  IFS=, read rf ct tl fr <<< "$cfg"
  GDI_K4_REFRESH=$rf GDI_K4_CTA_TAIL=$ct GDI_K4_TAIL=$tl GDI_K4_FRESH=${fr:-1} timeout 300 python scripts/k4_probe.py random:1000000:4000000:1000001 1 20 random:100000:400000:77 1 20 random:1000000:4000000:1000001 1 200 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print('refresh,cta,tail,fresh $cfg', d['recipe'].split(':')[1], d['sweeps'], round(d['ms'],3), d.get('sm_mhz'), d['cut'][:4], d['imbalance'][:4], d['counter_ok'], d['final_sum_ok'])
  else: print(l.rstrip()[:300])
"
done
