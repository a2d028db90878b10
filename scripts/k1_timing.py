"""Time the exact kernel per config with CUDA events on the session stream."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1908_00210_b200 as pi
from bench import build_graph, CONFIGS

def run(name, R, sweeps, reps=3):
    recipe = CONFIGS[name][0]
    g = build_graph(pi, recipe)
    prob = pi.MinCutProblem.with_default_coefficients(g)
    p = pi.AnnealParams(); p.sweeps = sweeps; p.deterministic = True
    st = torch.cuda.Stream(); torch.cuda.set_stream(st)
    s = pi.Session(prob, p, R, stream=st.cuda_stream, trace=True)
    s.set_seeds(np.arange(1, R + 1, dtype=np.uint64))
    ts = []
    for i in range(reps + 1):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st); s.launch(); e1.record(st); torch.cuda.synchronize()
        if i: ts.append(e0.elapsed_time(e1))
    s.sync()
    ms = min(ts)
    ups = R * g.num_nodes * sweeps / (ms * 1e-3)
    print(json.dumps({"config": name, "R": R, "sweeps": sweeps, "ms": ms, "updates_per_s": ups,
                      "ns_per_visit_per_replica": ms * 1e6 / (g.num_nodes * sweeps), "kernel": s.kernel}), flush=True)

for name in sys.argv[1].split(","):
    for R in [int(x) for x in sys.argv[2].split(",")]:
        run(name, R, int(sys.argv[3]) if len(sys.argv) > 3 else 100)
