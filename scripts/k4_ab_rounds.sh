# same-box A/B of K4 builds in abtest/*: M1 20-sweep median time + balance
for rep in 1 2; do
  for v in tree ${AB:-r3 r4 r6}; do
    if [ $v = tree ]; then LLP=; else LLP=$PWD/abtest/$v; fi
    echo -n "$v "; LD_LIBRARY_PATH=$LLP timeout 300 python scripts/k4_balance_probe.py random:1000000:4000000:1000001 20 4 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['median_ms'],4), d['mean_cut'], d['imb_hist'])"
  done
done
