"""Small anneals for compute-sanitizer runs: exact mode (k1_block, or the kernel
GDI_FORCE_KERNEL picks) on G1 x R replicas, checked against the oracle; or the
pooled mode (k2_chains / K4) on small graphs.

usage: python scripts/sanitize_run.py exact|pooled|part [R] [SWEEPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1908_00210_b200 as pi

mode = sys.argv[1]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8
S = int(sys.argv[3]) if len(sys.argv) > 3 else 50
p = pi.AnnealParams()
p.sweeps = S
if mode == "exact":
    from oracle import oracle as o

    g = pi.random_graph(800, 19176, 1)
    p.deterministic = True
    s = pi.Session(pi.MinCutProblem.with_default_coefficients(g), p, R, trace=True)
    s.set_seeds(np.arange(1, R + 1, dtype=np.uint64))
    s.launch()
    s.sync()
    out = s.fetch(spins=True, trace=True)
    og = o.random_graph(800, 19176, 1)
    for i in range(R):
        assert out["spins"][i].tolist() == o.anneal(og, i + 1, sweeps=S)["spins"].tolist()
    print(s.kernel, "ok: bit-exact vs oracle,", R, "replicas")
else:
    p.workers = 8
    g = pi.random_graph(2000, 19990, 22) if mode == "pooled" else pi.random_graph(20000, 80000, 5)
    s = pi.Session(pi.MinCutProblem.with_default_coefficients(g), p, R, trace=True)
    s.set_seeds(np.arange(1, R + 1, dtype=np.uint64))
    s.launch()
    s.sync()
    out = s.fetch(spins=True, trace=True)
    sums = out["spins"].astype(np.int64).sum(1)
    assert (out["balance_counter"] == sums).all()
    print(s.kernel, "ok: counter == spin sum,", R, "replicas")
