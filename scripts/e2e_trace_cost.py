import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1908_00210_b200 as pi
from bench import build_graph, CONFIGS
g = build_graph(pi, CONFIGS["G22"][0]); R, S = CONFIGS["G22"][1], CONFIGS["G22"][2]
prob = pi.MinCutProblem.with_default_coefficients(g)
p = pi.AnnealParams(); p.sweeps = S; p.workers = 1; p.deterministic = True
seeds = np.arange(1, R + 1, dtype=np.uint64)
for tr in (True, False, True):
    ts = []
    for i in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        d = pi.anneal_batch_fresh(prob, p, seeds, tr)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    print("trace", tr, [round(x * 1e3, 1) for x in ts], "kernel", round(d["seconds"] * 1e3, 1), flush=True)
