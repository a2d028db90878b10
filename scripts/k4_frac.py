"""M1 (20 sweeps) time and cut over seeds for the current K4 settings."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch, json
import paper_1908_00210_b200 as pi
from tests.helpers import product_graph
g = product_graph(["random", "1000000", "4000000", "1000001"])
prob = pi.MinCutProblem.with_default_coefficients(g)
p = pi.AnnealParams(); p.sweeps = 20; p.workers = 8
st = torch.cuda.Stream()
cuts, ts, imbs = [], [], []
for seed in range(1, 7):
    s = pi.Session(prob, p, 1, stream=st.cuda_stream, trace=True); s.set_seeds(np.array([seed], dtype=np.uint64))
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); s.launch(); e1.record(st); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    s.sync(); out = s.fetch(spins=False, trace=False); cuts.append(int(out["cut"][0])); imbs.append(int(out["imbalance"][0]))
print(json.dumps({"ms_min": min(ts), "cuts": cuts, "mean_rel": float(np.mean(cuts)) / 1252631 - 1, "max_rel": max(cuts) / 1252631 - 1, "imb": imbs}))
