"""A hub vertex (degree >= 4096) in an otherwise sparse graph: the row-length
extreme the reference handles uniformly (anneal.cpp:90-92, one loop over any
row). Exact mode bit for bit against the oracle (every exact kernel the
session picks); the pooled mode's exact invariants (counter == spin sum at
every barrier, trace == final score) and quality against the exact mode, on
both pooled kernels (k2_chains for many replicas, K4 for a single replica).
"""
import numpy as np
import pytest

import paper_1908_00210_b200 as pi
from oracle import oracle as o

pytestmark = pytest.mark.gpu


def hub_graph(n=12000, extra=30000, hub_deg=5000, seed=7):
    rng = np.random.default_rng(seed)
    seen, edges = set(), []
    for v in rng.choice(np.arange(1, n), hub_deg, replace=False):  # vertex 0: the hub
        seen.add((0, int(v)))
        edges.append((0, int(v), 1))
    while len(edges) < hub_deg + extra:
        u, v = sorted(int(x) for x in rng.integers(1, n, 2))
        if u == v or (u, v) in seen:
            continue
        seen.add((u, v))
        edges.append((u, v, 1))
    return n, edges


@pytest.fixture(scope="module")
def hub():
    n, edges = hub_graph()
    e = np.array(edges, dtype=np.int64)
    g = pi.Graph.from_edges(n, edges)
    assert g.max_degree >= 4096
    return g, o.csr_from_edges(n, e[:, 0], e[:, 1], e[:, 2])


def test_hub_exact_bit_exact_vs_oracle(hub):
    g, og = hub
    p = pi.AnnealParams()
    p.sweeps, p.deterministic = 40, True
    seeds = np.arange(1, 5, dtype=np.uint64)
    s = pi.Session(pi.MinCutProblem.with_default_coefficients(g), p, len(seeds), trace=True)
    s.set_seeds(seeds)
    s.launch()
    s.sync()
    out = s.fetch(spins=True, trace=True)
    for i, sd in enumerate(seeds.tolist()):
        ref = o.anneal(og, sd, sweeps=40)
        assert out["spins"][i].tolist() == ref["spins"].tolist(), (s.kernel, sd)
        assert out["trace"][i].tolist() == ref["trace"].tolist(), (s.kernel, sd)


@pytest.fixture(scope="module")
def big_hub():
    n, edges = hub_graph(n=100000, extra=400000, hub_deg=6000, seed=8)
    return pi.Graph.from_edges(n, edges)


@pytest.mark.parametrize("kernel,replicas", [("k2", 256), ("k4", 1)])
def test_hub_pooled_invariants_and_quality(hub, big_hub, kernel, replicas, monkeypatch):
    """The pooled kernels on hub graphs: k2_chains (12k vertices, 256
    replicas) and K4 (100k vertices, one replica: the kernel that visits a
    single replica's vertices from ~150 chains at once, so a graph much
    smaller than that in-flight window would be a Jacobi sweep and is left to
    K2). Exact invariants every run; mean cut within 2% of the exact mode's
    (3% for one replica); balanced runs no more than 10% below the exact
    mode's (measured: 81% vs 86% with k2_chains: concurrent chains' last flips
    leave residuals that this graph's stiff vertices do not absorb). K4 runs
    20 sweeps (the M1 schedule): late in a long anneal the hub's neighbours
    drift together faster than K4's per-chain counters and its low-degree tail
    correct (imbalance ~100 of 100k after 200 sweeps; K4)."""
    g = hub[0] if kernel == "k2" else big_hub
    prob = pi.MinCutProblem.with_default_coefficients(g)
    # k2: three sessions of 256 replicas (the shape that runs k2_chains),
    # seeds 1..768: the balanced fraction of 256 runs varies by +-2.5% from
    # run to run (racy chains), so the comparison pools 768
    blocks = 3 if kernel == "k2" else 1
    res = {}
    for det in (True, False):
        p = pi.AnnealParams()
        p.sweeps = 200 if kernel == "k2" else 20
        if det:
            p.deterministic = True
        else:
            p.workers = 8
        outs = []
        for b in range(blocks):
            s = pi.Session(prob, p, replicas, trace=True)
            s.set_seeds(np.arange(1 + b * replicas, 1 + (b + 1) * replicas, dtype=np.uint64))
            s.launch()
            s.sync()
            outs.append(s.fetch(spins=True, trace=True))
        res[det] = (s.kernel, {k: np.concatenate([o[k] for o in outs]) for k in outs[0] if np.ndim(outs[0][k]) > 0})
    kern, th = res[False]
    assert kern.startswith("k4_sweep" if kernel == "k4" else "k2_chains"), kern
    sums = th["spins"].astype(np.int64).sum(1)
    assert (th["balance_counter"] == sums).all() and (np.abs(sums) == th["imbalance"]).all()
    assert (th["trace"][:, -1, 1] == th["cut"]).all()
    assert (np.abs(th["counters"]) == th["trace"][:, :, 2]).all()
    ev = pi.evaluate_batch(prob, th["spins"])
    assert (ev["cut"] == th["cut"]).all()
    ex = res[True][1]
    tol = (0.02 if replicas > 1 else 0.03) * abs(ex["cut"].mean())
    assert th["cut"].mean() <= ex["cut"].mean() + tol, (th["cut"].mean(), ex["cut"].mean())
    if replicas > 1:
        assert (th["imbalance"] == 0).mean() >= (ex["imbalance"] == 0).mean() - 0.10
    else:
        assert th["imbalance"].max() <= 4
