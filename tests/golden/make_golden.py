"""Regenerate the golden vectors from the UNMODIFIED reference (TEST INFRASTRUCTURE).

Runs in the dev container only (needs /root/reference compiled into
oracle/_ref by `make -C oracle`). Produces:

  config_runs.json  BASELINE.json configs: per-seed final cut / imbalance /
                    h_scaled, FNV-1a of the final int8 spins and of the
                    (h_scaled, cut, imbalance) trace, via oracle/_ref/ref_tool
                    (reference anneal.cpp, deterministic mode).
  small_cases.json  small graphs (weighted, odd n, isolated nodes, n=1, custom
                    coefficients / schedules) with full spins, full trace and
                    the barrier counter, via the reference pybind module
                    oracle/_ref/pyising (proj/python/module.cpp).
  bench_rows.json   the reference's own run_benchmark rows (bench.cpp:64-202)
                    for BENCH_GRAPHS (G-set files written from the recipes by
                    the reference generators) plus one unreadable file, both
                    strategies, via ref_tool runbench.

Usage: python tests/golden/make_golden.py [--only bench]
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(REPO, "oracle", "_ref")
TOOL = os.path.join(REF, "ref_tool")

CONFIGS = {
    # name: (recipe args, seed range, sweeps, full spins/trace for first seed)
    "G1": (["random", "800", "19176", "1"], (1, 16), 1000),
    "G22": (["random", "2000", "19990", "22"], (1, 1024), 1000),
    "G55": (["random", "5000", "12498", "55"], (1, 64), 1000),
    "G81pm1": (["torus_pm1", "100", "200", "81"], (1, 16), 1000),
    "M1": (["random", "1000000", "4000000", "1000001"], (1, 1), 20),
    # acceptance criterion 5 known answers (acceptance.cpp:194-196)
    "G47": (["random", "1000", "9990", "47"], (1, 10), 1000),
    "G43": (["random", "1000", "9990", "43"], (1, 10), 1000),
    "G32": (["torus", "100", "20", "32"], (1, 10), 1000),
}


def run_tool(args):
    out = subprocess.run([TOOL, *args], check=True, capture_output=True, text=True).stdout
    return json.loads(out)


def golden_config(name):
    recipe, (lo, hi), sweeps = CONFIGS[name]
    chunks = []
    step = max(1, (hi - lo + 1) // 8)
    s = lo
    while s <= hi:
        e = min(hi, s + step - 1)
        chunks.append((s, e))
        s = e + 1
    with ThreadPoolExecutor(8) as ex:
        parts = list(ex.map(lambda c: run_tool(
            ["golden", *recipe, "--seeds", str(c[0]), str(c[1]), "--sweeps", str(sweeps)]), chunks))
    head = run_tool(["golden", *recipe, "--seeds", str(lo), str(lo), "--sweeps", str(sweeps),
                     "--full-spins", "--full-trace"]) if name in ("G1", "G22", "G81pm1") else None
    runs = [r for p in parts for r in p["runs"]]
    doc = {k: parts[0][k] for k in ("n", "m", "gset_fnv", "max_degree")}
    doc.update(recipe=recipe, sweeps=sweeps, runs=runs)
    if head:
        doc["first_full"] = head["runs"][0]
    return name, doc


SMALL_SCRIPT = r"""
import json, random, sys
sys.path.insert(0, sys.argv[1])
import pyising as pi

def weighted(n, m, rng):
    m = min(m, n * (n - 1) // 2)
    seen, edges = set(), []
    while len(edges) < m:
        u, v = rng.randrange(n), rng.randrange(n)
        if u == v: continue
        u, v = min(u, v), max(u, v)
        if (u, v) in seen: continue
        seen.add((u, v))
        w = 0
        while w == 0: w = rng.randint(-3, 5)
        edges.append((u, v, w))
    return edges

rng = random.Random(20261018)
cases = []
def add(name, n, edges, coeffs, sweeps, pf0, decay, seed, strategy="gdi"):
    g = pi.Graph.from_edges(n, [pi.Edge(u, v, w) for (u, v, w) in edges])
    prob = pi.MinCutProblem.make_unchecked(g, pi.Coefficients(*coeffs))
    p = pi.AnnealParams(); p.sweeps = sweeps; p.flip_fraction0 = pf0; p.decay_rate = decay
    p.deterministic = True; p.seed = seed
    p.strategy = pi.Strategy.standard if strategy == "standard" else pi.Strategy.gdi
    r = pi.anneal(prob, p)
    sc = pi.score(prob, r.state)
    cases.append(dict(name=name, n=n, edges=edges, coeffs=list(coeffs), sweeps=sweeps, pf0=pf0,
                      decay=decay, seed=seed, strategy=strategy, spins=list(r.state),
                      trace=[[t.hamiltonian_scaled, t.cut, t.imbalance] for t in r.trace],
                      pf=[t.flip_probability for t in r.trace],
                      cut=sc.cut, imbalance=sc.imbalance, h_scaled=sc.hamiltonian_scaled))

add("two_node", 2, [(0, 1, 1)], (1, 1, 1), 50, 0.2, 0.9, 2)
add("single_node", 1, [], (1, 4, 1), 5, 0.04, 0.99, 1)
add("c4_default", 4, [(0, 1, 1), (1, 2, 1), (2, 3, 1), (3, 0, 1)], (1, 4, 1), 100, 0.04, 0.99, 1)
add("isolated", 9, [(0, 1, 1), (2, 3, 1), (3, 4, 2)], (1, 4, 1), 40, 0.3, 0.9, 5)
for t in range(24):
    n = rng.randint(3, 90)
    m = rng.randint(0, 3 * n)
    edges = weighted(n, m, rng)
    coeffs = rng.choice([(1, 4, 1), (1, 1, 1), (3, 2, 1), (7, 3, 8), (2, 9, 4)])
    sweeps = rng.randint(1, 60)
    pf0 = rng.choice([0.0, 0.04, 0.2, 1.0, 0.5])
    decay = rng.choice([0.99, 0.9, 0.5])
    seed = rng.getrandbits(64)
    add(f"weighted_{t}", n, edges, coeffs, sweeps, pf0, decay, seed,
        "standard" if t % 5 == 4 else "gdi")
json.dump(cases, sys.stdout)
"""


def small_cases():
    out = subprocess.run([sys.executable, "-c", SMALL_SCRIPT, REF], check=True,
                         capture_output=True, text=True).stdout
    return json.loads(out)


# run_benchmark parity set: name -> recipe (written as <name>.txt G-set files)
BENCH_GRAPHS = {
    "rnd500": ["random", "500", "5000", "5"],
    "torus30x20": ["torus", "30", "20", "7"],
    "pm1_20x20": ["torus_pm1", "20", "20", "9"],
    "rnd200": ["random", "200", "600", "11"],
}
BENCH_ARGS = {"runs": 6, "base_seed": 21, "sweeps": 300}


def bench_rows():
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        paths = []
        for name, recipe in BENCH_GRAPHS.items():
            text = subprocess.run([TOOL, "gset", *recipe], check=True, capture_output=True, text=True).stdout
            path = os.path.join(d, name + ".txt")
            with open(path, "w") as f:
                f.write(text)
            paths.append(path)
        bad = os.path.join(d, "unreadable.txt")
        with open(bad, "w") as f:
            f.write("3 1\n1 9 1\n")
        paths.insert(1, bad)
        rows = run_tool(["runbench", *paths, "--replicas", str(BENCH_ARGS["runs"]), "--seeds",
                         str(BENCH_ARGS["base_seed"]), "0", "--strategy", "both", "--sweeps",
                         str(BENCH_ARGS["sweeps"])])
    return {"graphs": BENCH_GRAPHS, "args": BENCH_ARGS, "order": [os.path.basename(p)[:-4] for p in paths],
            "rows": rows}


def main():
    if not os.path.exists(TOOL):
        sys.exit("build the reference first: make -C oracle")
    with open(os.path.join(HERE, "bench_rows.json"), "w") as f:
        json.dump(bench_rows(), f, indent=1)
    if "--only" in sys.argv:
        print("wrote bench_rows.json")
        return
    docs = dict(golden_config(n) for n in CONFIGS)
    with open(os.path.join(HERE, "config_runs.json"), "w") as f:
        json.dump(docs, f, separators=(",", ":"))
    with open(os.path.join(HERE, "small_cases.json"), "w") as f:
        json.dump(small_cases(), f, separators=(",", ":"))
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
