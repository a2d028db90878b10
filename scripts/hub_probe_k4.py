import sys; sys.path.insert(0,'.')
import numpy as np, paper_1908_00210_b200 as pi
from tests.test_gpu_hub import hub_graph
for hd in (0, 6000):
    n, edges = hub_graph(n=100000, extra=400000, hub_deg=max(hd, 1), seed=8)
    g = pi.Graph.from_edges(n, edges); prob = pi.MinCutProblem.with_default_coefficients(g)
    for sw in (20, 200):
        p = pi.AnnealParams(); p.sweeps = sw; p.workers = 8
        s = pi.Session(prob, p, 1, trace=True); s.set_seeds(np.array([1], dtype=np.uint64)); s.launch(); s.sync()
        out = s.fetch(spins=True, trace=True)
        print(hd, sw, s.kernel, out["cut"][0], out["imbalance"][0], out["trace"][0, -8:, 2].tolist(), g.max_degree)
