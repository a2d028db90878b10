"""acceptance.cpp criterion 5 in the pooled mode: best balanced cut of 10 seeds on torus(100, 20, 32) (bound 50)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1908_00210_b200 as pi
from tests.helpers import product_graph

g = product_graph(["torus", "100", "20", "32"])
prob = pi.MinCutProblem.with_default_coefficients(g)
for rep in range(3):
    p = pi.AnnealParams()
    p.sweeps, p.workers = 1000, 8
    s = pi.Session(prob, p, 10)
    s.set_seeds(np.arange(1, 11, dtype=np.uint64))
    s.launch()
    s.sync()
    o = s.fetch(spins=False)
    bal = o["imbalance"] == 0
    print(s.kernel, sorted(o["cut"][bal].tolist()), flush=True)
