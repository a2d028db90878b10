"""Loader throughput: G-set text of the 1M-vertex graph ->
parse -> CSR, the reference's Graph::parse_gset (graph.cpp:81-128, compiled
from /root/reference by oracle/Makefile into oracle/_ref) against ours, on the
same text and host; then ours through gdi_graph_create + layouts (GPU box).

usage: python scripts/parse_bench.py [N M SEED]   (default: the M1 recipe)"""
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1908_00210_b200 as pi


REF_TIMER = """
import importlib.util, os, sys, time
path = sys.argv[1]
so = [f for f in os.listdir(path) if f.startswith("pyising") and f.endswith(".so")][0]
spec = importlib.util.spec_from_file_location("pyising", os.path.join(path, so))
ref = importlib.util.module_from_spec(spec); spec.loader.exec_module(ref)
text = open(sys.argv[2]).read()
ts = []
for _ in range(2):
    t0 = time.perf_counter(); g = ref.Graph.parse_gset(text); ts.append(time.perf_counter() - t0)
print(min(ts), g.num_nodes, g.num_edges)
"""


def time_reference(text):
    """The reference's pybind module in its own process (pybind type names clash)."""
    import subprocess
    import tempfile

    path = os.path.join(REPO, "oracle", "_ref")
    if not os.path.isdir(path) or not any(f.startswith("pyising") for f in os.listdir(path)):
        return None
    with tempfile.NamedTemporaryFile("w", suffix=".gset", delete=False) as f:
        f.write(text)
    try:
        out = subprocess.run([sys.executable, "-c", REF_TIMER, path, f.name], capture_output=True, text=True,
                             check=True).stdout.split()
        return float(out[0]), int(out[1]), int(out[2])
    finally:
        os.unlink(f.name)


def best(f, reps=3):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = f()
        ts.append(time.perf_counter() - t0)
    return min(ts), out


n, m, seed = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (1000000, 4000000, 1000001)
g = pi.random_graph(n, m, seed)
text = g.to_gset()
ours_s, gp = best(lambda: pi.Graph.parse_gset(text))
assert gp.num_nodes == n and gp.num_edges == m
res = {"graph": f"random_graph({n},{m},{seed})", "text_bytes": len(text), "host_threads": os.cpu_count(),
       "ours_parse_s": ours_s}
ref = time_reference(text)
if ref is not None:
    assert ref[1:] == (n, m)
    res["reference_parse_s"] = ref[0]
    res["speedup"] = ref[0] / ours_s
if pi.device_count() > 0:
    # parse -> gdi_graph_create (pinned staging, upload, device validation) ->
    # the K4 layouts (degree order, SELL rows, position rows), each on a fresh
    # Graph (the device copy is cached per Graph)
    def load():
        t0 = time.perf_counter()
        gg = pi.Graph.parse_gset(text)
        t1 = time.perf_counter()
        p = pi.AnnealParams()
        p.sweeps, p.workers = 20, 8
        s = pi.Session(pi.MinCutProblem.with_default_coefficients(gg), p, 1)
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1, s.kernel

    load()  # (CUDA context, first-touch of the pinned staging buffer)
    runs = [load() for _ in range(3)]
    k = min(range(3), key=lambda i: runs[i][0] + runs[i][1])
    res["parse_s"], res["upload_and_layouts_s"], res["kernel"] = runs[k]
    res["parse_to_device_ready_s"] = runs[k][0] + runs[k][1]
print(json.dumps(res), flush=True)
