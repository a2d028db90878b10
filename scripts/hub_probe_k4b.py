import sys; sys.path.insert(0,'.')
import numpy as np, paper_1908_00210_b200 as pi
from tests.test_gpu_hub import hub_graph
from tests.helpers import product_graph
import torch
gs = {"hub100k": pi.Graph.from_edges(*hub_graph(n=100000, extra=400000, hub_deg=6000, seed=8)),
      "M1": product_graph(["random", "1000000", "4000000", "1000001"])}
for name, g in gs.items():
    prob = pi.MinCutProblem.with_default_coefficients(g)
    for det in (True, False):
        if det and name == "M1": continue
        p = pi.AnnealParams(); p.sweeps = 20
        if det: p.deterministic = True
        else: p.workers = 8
        st = torch.cuda.Stream()
        s = pi.Session(prob, p, 1, stream=st.cuda_stream, trace=True); s.set_seeds(np.array([1], dtype=np.uint64))
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); s.launch(); e1.record(st); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        s.sync(); out = s.fetch(spins=True, trace=True)
        print(name, "exact" if det else "pooled", s.kernel, round(min(ts), 3), out["cut"][0], out["imbalance"][0])
