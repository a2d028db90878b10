"""Balanced fraction of the pooled mode vs the exact mode on the 12k-vertex hub
graph of tests/test_gpu_hub.py (200 sweeps), over R replicas, repeated."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1908_00210_b200 as pi
from tests.test_gpu_hub import hub_graph

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n, edges = hub_graph()
g = pi.Graph.from_edges(n, edges)
prob = pi.MinCutProblem.with_default_coefficients(g)
seeds = np.arange(1, R + 1, dtype=np.uint64)
out = []
for det in (True, False, False, False):
    p = pi.AnnealParams()
    p.sweeps = 200
    if det:
        p.deterministic = True
    else:
        p.workers = 8
    s = pi.Session(prob, p, R)
    s.set_seeds(seeds)
    s.launch()
    s.sync()
    f = s.fetch(spins=False)
    out.append((s.kernel, round(float((f["imbalance"] == 0).mean()), 4), round(float(f["cut"].mean()), 1)))
print(out)
