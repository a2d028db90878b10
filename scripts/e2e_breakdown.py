import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1908_00210_b200 as pi
from bench import build_graph, CONFIGS
g = build_graph(pi, CONFIGS["G22"][0])
prob = pi.MinCutProblem.with_default_coefficients(g)
p = pi.AnnealParams(); p.sweeps = 1000; p.deterministic = True
seeds = np.arange(1, 1025, dtype=np.uint64)
for trace in (True, False):
    for i in range(3):
        t0 = time.perf_counter(); out = pi.anneal_batch_fresh(prob, p, seeds, trace); t1 = time.perf_counter()
        print(f"trace={trace} total {t1-t0:.3f}s kernel {out['seconds']:.3f}s")
t0 = time.perf_counter(); s = pi.Session(prob, p, 1024, trace=True); t1 = time.perf_counter()
s.set_seeds(seeds); s.launch(); s.sync(); t2 = time.perf_counter()
out = s.fetch(spins=True, trace=True); t3 = time.perf_counter()
print(f"session create {t1-t0:.3f} launch+sync {t2-t1:.3f} fetch(trace) {t3-t2:.3f}")
