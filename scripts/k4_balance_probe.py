"""K4 end-of-anneal balance over many seeds (single-device Session path and,
with --part, the partitioned driver with a NCCL world of one rank).

usage: python scripts/k4_balance_probe.py RECIPE SWEEPS SEEDS [--part]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1908_00210_b200 as pi
from tests.helpers import product_graph

recipe, sweeps, nseeds = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
part = "--part" in sys.argv
g = product_graph(recipe.split(":"))
prob = pi.MinCutProblem.with_default_coefficients(g)
p = pi.AnnealParams()
p.sweeps, p.workers = sweeps, 8
imbs, cuts, ms = [], [], []
if part:
    import torch.distributed as dist
    from paper_1908_00210_b200 import sharding as sh
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29537")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    pi.set_device(0)
    for s in range(1, nseeds + 1):
        pa = sh.PartitionedAnneal(prob, p, s, dist, 0)
        for _ in range(2):
            r = pa.run()
            imbs.append(int(r["imbalance"]))
            cuts.append(int(r["cut"]))
        pa.close()
    dist.destroy_process_group()
else:
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    s = pi.Session(prob, p, 1, stream=st.cuda_stream, trace=True)
    for seed in range(1, nseeds + 1):
        for _ in range(2):
            s.set_seeds(np.array([seed], dtype=np.uint64))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            s.launch()
            e1.record(st)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            out = s.fetch(spins=True, trace=True)
            imbs.append(int(out["imbalance"][0]))
            cuts.append(int(out["cut"][0]))
print(json.dumps({"recipe": recipe, "part": part, "env": {k: v for k, v in os.environ.items() if k.startswith("GDI_")},
                  "imb_hist": {str(k): imbs.count(k) for k in sorted(set(imbs))}, "mean_cut": float(np.mean(cuts)),
                  "cuts": cuts,
                  "median_ms": float(np.median(ms)) if ms else None}))
