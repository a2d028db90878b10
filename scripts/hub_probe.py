import sys; sys.path.insert(0,'.')
import numpy as np, paper_1908_00210_b200 as pi
from tests.test_gpu_hub import hub_graph
n, edges = hub_graph(); g = pi.Graph.from_edges(n, edges); prob = pi.MinCutProblem.with_default_coefficients(g)
for R in (1, 256):
    seeds = np.arange(1, R+1, dtype=np.uint64)
    for det in (True, False):
        p = pi.AnnealParams(); p.sweeps = 200
        if det: p.deterministic = True
        else: p.workers = 8
        s = pi.Session(prob, p, R, trace=True); s.set_seeds(seeds); s.launch(); s.sync()
        out = s.fetch(spins=True, trace=True)
        print(R, det, s.kernel, out["cut"].mean(), (out["imbalance"]==0).mean(), np.bincount(out["imbalance"])[:8], out["trace"][0,-5:,2] if R==1 else "")
