"""K3 timing probe: evaluate_device on random spins, CUDA-event times per call.

usage: python scripts/k3_probe.py RECIPE R [REPS]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1908_00210_b200 as pi
from tests.helpers import product_graph

recipe, R = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
g = product_graph(recipe.split(":"))
prob = pi.MinCutProblem.with_default_coefficients(g)
ev = pi.Evaluator(prob)
rng = np.random.default_rng(1)
sp = np.where(rng.random((R, g.num_nodes)) < 0.5, 1, -1).astype(np.int8)
d = torch.from_numpy(sp).cuda()
res = torch.zeros((R, 2), dtype=torch.int64, device="cuda")
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ts = []
for i in range(reps + 3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ev.evaluate_device(d.data_ptr(), R, res.data_ptr(), 0, st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
ref = ev.evaluate(sp[:1])
print(f"{recipe} R={R}: median {statistics.median(ts)*1e3:.1f} us, min {min(ts)*1e3:.1f} us; "
      f"check {int(res[0,0].item()) == int(ref['cut'][0])}")
