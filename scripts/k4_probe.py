"""K4 (vertex-partitioned throughput sweep) timing + quality on large / single-replica configs.

usage: python scripts/k4_probe.py RECIPE R SWEEPS [RECIPE R SWEEPS ...]
  RECIPE like random:1000000:4000000:1000001 or torus_pm1:100:200:81
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1908_00210_b200 as pi
from tests.helpers import product_graph


def sm_clock():
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        return pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    except Exception:
        return None


def run(recipe, R, sweeps):
    t0 = time.time()
    g = product_graph(recipe.split(":"))
    tg = time.time() - t0
    prob = pi.MinCutProblem.with_default_coefficients(g)
    p = pi.AnnealParams()
    p.sweeps, p.workers = sweeps, 8
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
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
    clk = sm_clock()
    s.sync()
    out = s.fetch(spins=True, trace=True)
    tr = out["trace"]
    ctr = out.get("counters")
    sums = out["spins"].astype(np.int64).sum(1)
    print(json.dumps({
        "recipe": recipe, "R": R, "sweeps": sweeps, "kernel": s.kernel, "gen_s": round(tg, 2),
        "launches": s.launch_count, "ms": min(ts), "sm_mhz": clk, "ms_all": ts,
        "updates_per_s": R * g.num_nodes * sweeps / (min(ts) * 1e-3),
        "cut": out["cut"].tolist()[:8], "imbalance": out["imbalance"].tolist()[:8],
        "imb_trace_r0": tr[0, :, 2].tolist()[-10:], "ctr_r0": out["counters"][0].tolist()[-40:], "cut_trace_r0": tr[0, :, 1].tolist()[-5:],
        "final_sum_ok": bool((np.abs(sums) == out["imbalance"]).all()),
        "counter_ok": bool((out["balance_counter"] == sums).all()),
    }), flush=True)


args = sys.argv[1:]
for i in range(0, len(args), 3):
    run(args[i], int(args[i + 1]), int(args[i + 2]))
