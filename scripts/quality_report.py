"""Pooled (racy) mode vs exact mode quality over many seeds: mean / best
balanced cut and balanced fraction per BASELINE G-set config (4096 seeds),
the 1M-vertex config (K4, 8 seeds x 2 runs) and the hub graph (k2_chains, 8
blocks of 256). Writes one JSON document (profiles/r02_quality.json)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1908_00210_b200 as pi
from tests.helpers import golden_configs, product_graph


def run(prob, det, seeds, sweeps=1000):
    p = pi.AnnealParams()
    p.sweeps = sweeps
    if det:
        p.deterministic = True
    else:
        p.workers = 8
    s = pi.Session(prob, p, len(seeds))
    s.set_seeds(np.asarray(seeds, dtype=np.uint64))
    s.launch()
    s.sync()
    return s.kernel, s.fetch(spins=False)


def summary(out, floor):
    bal = out["imbalance"] <= floor
    return {"mean_cut": float(out["cut"].mean()), "best_balanced_cut": int(out["cut"][bal].min()) if bal.any() else None,
            "balanced_fraction": float(bal.mean())}


doc = {}
docs = golden_configs()
for name in ("G1", "G22", "G55", "G81pm1"):
    g = product_graph(docs[name]["recipe"])
    prob = pi.MinCutProblem.with_default_coefficients(g)
    seeds = np.arange(1, 4097)
    ke, ex = run(prob, True, seeds)
    kt, th = run(prob, False, seeds)
    floor = g.num_nodes % 2
    doc[name] = {"seeds": 4096, "sweeps": 1000, "exact": dict(kernel=ke, **summary(ex, floor)),
                 "pooled": dict(kernel=kt, **summary(th, floor))}
    print(name, json.dumps(doc[name]), flush=True)
g = product_graph(docs["M1"]["recipe"])
prob = pi.MinCutProblem.with_default_coefficients(g)
cuts, imbs = [], []
for seed in range(1, 9):
    for _ in range(2):
        k, o = run(prob, False, [seed], sweeps=20)
        cuts.append(int(o["cut"][0]))
        imbs.append(int(o["imbalance"][0]))
det = docs["M1"]["runs"][0]["cut"]
doc["M1"] = {"runs": 16, "sweeps": 20, "kernel": k, "deterministic_cut": det,
             "pooled_cut_rel": [round(c / det - 1, 5) for c in cuts], "mean_rel": round(float(np.mean(cuts)) / det - 1, 5),
             "imbalance_max": max(imbs)}
print("M1", json.dumps(doc["M1"]), flush=True)
from tests.test_gpu_hub import hub_graph
n, edges = hub_graph()
prob = pi.MinCutProblem.with_default_coefficients(pi.Graph.from_edges(n, edges))
fe, ft = [], []
for b in range(8):
    seeds = np.arange(1 + 256 * b, 257 + 256 * b)
    _, ex = run(prob, True, seeds, sweeps=200)
    k, th = run(prob, False, seeds, sweeps=200)
    fe.append(float((ex["imbalance"] == 0).mean()))
    ft.append(float((th["imbalance"] == 0).mean()))
doc["hub_12k_deg5000"] = {"seeds": 2048, "sweeps": 200, "pooled_kernel": k, "exact_balanced_fraction": float(np.mean(fe)),
                          "pooled_balanced_fraction": float(np.mean(ft))}
print("hub", json.dumps(doc["hub_12k_deg5000"]), flush=True)
json.dump(doc, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/r02_quality.json", "w"), indent=1)
