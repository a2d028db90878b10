"""Vertex-partitioned K4 quality/time vs emulated rank count (one GPU)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1908_00210_b200 as pi
from paper_1908_00210_b200 import sharding as sh
from tests.helpers import product_graph

recipe = sys.argv[1].split(":"); sweeps = int(sys.argv[2])
fused = len(sys.argv) > 4 and sys.argv[4] == "fused"
g = product_graph(recipe)
prob = pi.MinCutProblem.with_default_coefficients(g)
p = pi.AnnealParams(); p.sweeps, p.workers = sweeps, 8
for w in [int(x) for x in sys.argv[3].split(",")]:
    for seed in (1, 2):
        torch.cuda.synchronize(); t = time.time()
        out = sh.emulate_partitioned(prob, p, seed, w, fused=fused)
        torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps({"fused": fused, "world": w, "seed": seed, "cut": out["cut"], "imb": out["imbalance"],
                          "imb_tail": out["trace_imbalance"][-6:].tolist(), "agree": out["rank_spins_agree"],
                          "wall_s": round(dt, 3)}), flush=True)
