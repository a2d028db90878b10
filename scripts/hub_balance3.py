"""Hub-graph balanced fraction of the pooled mode (k2_chains, 256 replicas per
session, several seed blocks) and G22/G55 pooled timing; for same-box A/B."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1908_00210_b200 as pi
from tests.test_gpu_hub import hub_graph

n, edges = hub_graph()
g = pi.Graph.from_edges(n, edges)
prob = pi.MinCutProblem.with_default_coefficients(g)
fr = []
for b in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    p = pi.AnnealParams()
    p.sweeps, p.workers = 200, 8
    s = pi.Session(prob, p, 256)
    s.set_seeds(np.arange(1 + 256 * b, 257 + 256 * b, dtype=np.uint64))
    s.launch()
    s.sync()
    fr.append(float((s.fetch(spins=False)["imbalance"] == 0).mean()))
print("hub balanced", s.kernel, round(float(np.mean(fr)), 4), np.round(fr, 3).tolist())
