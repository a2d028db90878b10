"""Throughput-mode (K2) timing + quality on the G-set configs, R replicas, against the exact mode on the same seeds.

usage: python scripts/k2_probe2.py CONFIG[,CONFIG...] [R] [SWEEPS]   (CONFIG: a bench config or a recipe
       like random:1000:9990:47)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1908_00210_b200 as pi
from bench import CONFIGS, build_graph


def timed(prob, p, R):
    st = torch.cuda.Stream()
    s = pi.Session(prob, p, R, stream=st.cuda_stream, trace=True)
    s.set_seeds(np.arange(1, R + 1, dtype=np.uint64))
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.launch()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    s.sync()
    return s.kernel, min(ts), s.fetch(spins=True, trace=True)


R = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
S = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
for cfg in sys.argv[1].split(","):
    if cfg in CONFIGS:
        g = build_graph(pi, CONFIGS[cfg][0])
    else:
        from tests.helpers import product_graph
        g = product_graph(cfg.split(":"))
    prob = pi.MinCutProblem.with_default_coefficients(g)
    pt = pi.AnnealParams()
    pt.sweeps, pt.workers = S, 8
    pe = pi.AnnealParams()
    pe.sweeps, pe.deterministic = S, True
    kt, mt, t = timed(prob, pt, R)
    ke, me, e = timed(prob, pe, R)
    bal = t["imbalance"] <= g.num_nodes % 2
    print(json.dumps({"config": cfg, "R": R, "sweeps": S, "thru_kernel": kt, "thru_ms": round(mt, 3),
                      "thru_updates_per_s": R * g.num_nodes * S / (mt * 1e-3), "exact_kernel": ke,
                      "exact_ms": round(me, 3), "speedup": round(me / mt, 3),
                      "thru_mean_cut": float(t["cut"].mean()), "exact_mean_cut": float(e["cut"].mean()),
                      "thru_best_bal": int(t["cut"][bal].min()) if bal.any() else None,
                      "exact_best": int(e["cut"].min()), "thru_frac_bal": float(bal.mean()),
                      "exact_frac_bal": float((e["imbalance"] <= g.num_nodes % 2).mean()),
                      "counter_ok": bool((t["balance_counter"] == t["spins"].astype(np.int64).sum(1)).all()),
                      "trace_cut_ok": bool((t["trace"][:, -1, 1] == t["cut"]).all()),
                      "thru_cuts": t["cut"][:10].tolist(), "thru_imb": t["imbalance"][:10].tolist()}), flush=True)
