"""k1_block's rows variant (row records in global memory, degree <= 4): bit for
bit against the C restatement of the reference's deterministic anneal
(anneal.cpp:86-202), forced (GDI_BLOCK_ROWS=1) on small graphs of every
shape the variant accepts, and chosen automatically on G81+-1 (whose CSR does
not fit shared memory next to 7 replicas) against the golden vectors."""
import numpy as np
import pytest

import paper_1908_00210_b200 as pi
from oracle import oracle as o
from tests.helpers import fnv_rows, golden_configs, product_graph

pytestmark = pytest.mark.gpu


def det_params(sweeps):
    p = pi.AnnealParams()
    p.sweeps, p.deterministic = sweeps, True
    return p


def sparse_edges(n, m, maxdeg, signed, seed):
    rng = np.random.default_rng(seed)
    deg = np.zeros(n, int)
    seen, edges = set(), []
    while len(edges) < m:
        u, v = sorted(int(x) for x in rng.integers(0, n, 2))
        if u == v or (u, v) in seen or deg[u] >= maxdeg or deg[v] >= maxdeg:
            continue
        seen.add((u, v))
        deg[u] += 1
        deg[v] += 1
        edges.append((u, v, int(rng.choice([-1, 1])) if signed else 1))
    return edges


@pytest.mark.parametrize("n,m,signed", [(33, 40, False), (100, 150, True), (257, 400, False), (1000, 1900, True)])
def test_rows_variant_forced_bit_exact(n, m, signed, monkeypatch):
    monkeypatch.setenv("GDI_BLOCK_ROWS", "1")
    edges = sparse_edges(n, m, 4, signed, n)
    e = np.array(edges, dtype=np.int64)
    g = pi.Graph.from_edges(n, edges)
    og = o.csr_from_edges(n, e[:, 0], e[:, 1], e[:, 2])
    seeds = np.arange(3, 3 + 20, dtype=np.uint64)
    s = pi.Session(pi.MinCutProblem.with_default_coefficients(g), det_params(60), len(seeds), trace=True)
    s.set_seeds(seeds)
    s.launch()
    s.sync()
    out = s.fetch(spins=True, trace=True)
    assert s.kernel.endswith(",rows>"), s.kernel
    for i, sd in enumerate(seeds.tolist()):
        ref = o.anneal(og, sd, sweeps=60)
        assert out["spins"][i].tolist() == ref["spins"].tolist(), (n, sd)
        assert out["trace"][i].tolist() == ref["trace"].tolist(), (n, sd)


def test_rows_variant_torus_forced_bit_exact(monkeypatch):
    monkeypatch.setenv("GDI_BLOCK_ROWS", "1")
    for recipe in (["torus", "10", "13", "5"], ["torus_pm1", "20", "20", "9"]):
        g = product_graph(recipe)
        og = o.recipe(":".join(recipe))
        out = pi.anneal_batch(pi.MinCutProblem.with_default_coefficients(g), det_params(80),
                              np.arange(1, 9, dtype=np.uint64), trace=True)
        for i in range(8):
            ref = o.anneal(og, i + 1, sweeps=80)
            assert out["spins"][i].tolist() == ref["spins"].tolist()
            assert out["trace"][i].tolist() == ref["trace"].tolist()


def test_rows_variant_chosen_for_g81_golden():
    doc = golden_configs()["G81pm1"]
    g = product_graph(doc["recipe"])
    seeds = np.array([int(r["seed"]) for r in doc["runs"]], dtype=np.uint64)
    s = pi.Session(pi.MinCutProblem.with_default_coefficients(g), det_params(int(doc["sweeps"])), len(seeds))
    s.set_seeds(seeds)
    s.launch()
    s.sync()
    assert s.kernel.endswith(",rows>"), s.kernel
    out = s.fetch(spins=True)
    fnv = fnv_rows(out["spins"])
    for i, r in enumerate(doc["runs"]):
        assert int(out["cut"][i]) == int(r["cut"]) and int(out["imbalance"][i]) == int(r["imbalance"])
        assert f"{fnv[i]:016x}" == r["spins_fnv"]
