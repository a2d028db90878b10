import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, paper_1908_00210_b200 as pi
from tests.helpers import golden_configs, product_graph
doc = golden_configs()["G1"]
g = product_graph(doc["recipe"]); prob = pi.MinCutProblem.with_default_coefficients(g)
for det in (False, True):
    fr=[]; cuts=[]
    for blk in range(4):
        p = pi.AnnealParams(); p.sweeps = 1000
        if det: p.deterministic = True
        else: p.workers = 8
        seeds = np.arange(1 + 1024*blk, 1025 + 1024*blk, dtype=np.uint64)
        s = pi.Session(prob, p, 1024); s.set_seeds(seeds); s.launch(); s.sync(); o = s.fetch(spins=False)
        fr.append((o["imbalance"] == 0).mean()); cuts.append(o["cut"].mean())
    print("det" if det else "thru", np.round(fr,4), np.mean(fr), np.mean(cuts))
