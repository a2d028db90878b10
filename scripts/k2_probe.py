"""K2 (throughput mode) timing + quality vs K1 exact on the BASELINE configs."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1908_00210_b200 as pi
from bench import build_graph, CONFIGS

def run(name, R, sweeps, det):
    g = build_graph(pi, CONFIGS[name][0])
    prob = pi.MinCutProblem.with_default_coefficients(g)
    p = pi.AnnealParams(); p.sweeps = sweeps
    if det: p.deterministic = True
    else: p.workers = 8
    st = torch.cuda.Stream(); torch.cuda.set_stream(st)
    s = pi.Session(prob, p, R, stream=st.cuda_stream, trace=True)
    s.set_seeds(np.arange(1, R + 1, dtype=np.uint64))
    ts = []
    for i in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st); s.launch(); e1.record(st); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    s.sync()
    out = s.fetch(spins=True, trace=True)
    cut, imb = out["cut"], out["imbalance"]
    bal = imb <= g.num_nodes % 2
    tr = out["trace"]
    consistent = bool((tr[:, -1, 1] == cut).all() and (tr[:, -1, 2] == imb).all())
    print(json.dumps({"config": name, "mode": "exact" if det else "throughput", "kernel": s.kernel, "R": R,
                      "sweeps": sweeps, "ms": min(ts), "updates_per_s": R * g.num_nodes * sweeps / (min(ts) * 1e-3),
                      "best_bal_cut": int(cut[bal].min()) if bal.any() else None, "mean_cut": float(cut.mean()),
                      "frac_balanced": float(bal.mean()), "max_imb": int(imb.max()), "trace_consistent": consistent}),
          flush=True)

for name in sys.argv[1].split(","):
    R = int(sys.argv[2]); sw = int(sys.argv[3])
    run(name, R, sw, True)
    run(name, R, sw, False)
