import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1908_00210_b200 as pi
from bench import build_graph, CONFIGS
g = build_graph(pi, CONFIGS[sys.argv[1]][0])
prob = pi.MinCutProblem.with_default_coefficients(g)
p = pi.AnnealParams(); p.sweeps = int(sys.argv[2]); p.workers = 8
s = pi.Session(prob, p, 1024, trace=True)
s.set_seeds(np.arange(1, 1025, dtype=np.uint64)); s.launch(); s.sync()
print(s.kernel, s.fetch(spins=False)["seconds"])
