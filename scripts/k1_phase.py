"""Exact-kernel time per phase of the anneal (per-sweep device timestamps from the trace)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1908_00210_b200 as pi
from bench import build_graph, CONFIGS

name = sys.argv[1] if len(sys.argv) > 1 else "G22"
g = build_graph(pi, CONFIGS[name][0]); R, S = CONFIGS[name][1], CONFIGS[name][2]
prob = pi.MinCutProblem.with_default_coefficients(g)
p = pi.AnnealParams(); p.sweeps = S; p.deterministic = True
s = pi.Session(prob, p, R, trace=True)
s.set_seeds(np.arange(1, R + 1, dtype=np.uint64))
s.launch(); s.sync()
d = s.fetch(spins=False, trace=True)
sec = d["trace_seconds"].mean(axis=0)  # per sweep, mean over replicas
tot = sec.sum()
print(f"{name}: kernel {d['seconds']*1e3:.1f} ms, sum of mean sweep times {tot*1e3:.1f} ms")
for a in range(0, S, S // 10):
    b = a + S // 10
    print(f"  sweeps {a:4d}-{b:4d}: {sec[a:b].sum()*1e3:6.2f} ms ({sec[a:b].sum()/tot:5.1%}), {sec[a:b].mean()*1e6:6.1f} us/sweep, "
          f"{sec[a:b].mean()*1.965e9/g.num_nodes:5.1f} cycles/visit")
