"""The reference annealer contract, run through the product path on the GPU.

Ports of reference proj/tests/test_anneal.cpp (cited per test) and the
anneal cases of proj/python/tests/test_smoke.py, plus the hook-based
acceptance criteria 3 and 4 (proj/tests/acceptance.cpp:124-183).
"""
import numpy as np
import pytest

import paper_1908_00210_b200 as pi

pytestmark = pytest.mark.gpu


def params(**kw):
    p = pi.AnnealParams()
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def naive_h(g, coeffs, s):
    s = np.asarray(s, dtype=np.int64)
    cut = sum(e.weight for e in g.edges() if s[e.u] != s[e.v])
    return coeffs.a_num * int(s.sum()) ** 2 + coeffs.b_num * cut


def test_two_node_optimum():  # test_anneal.cpp:60-75
    g = pi.Graph.parse_gset("2 1\n1 2 1")
    p = pi.MinCutProblem.make_unchecked(g, pi.Coefficients(1, 1, 1))
    for seed in (1, 2, 3, 4, 5):
        r = pi.anneal(p, params(sweeps=50, flip_fraction0=0.2, decay_rate=0.9, deterministic=True, seed=seed))
        assert pi.cut_value(g, r.state) == 1 and pi.imbalance(r.state) == 0
        assert len(r.trace) == 50


def test_four_cycle_optimum():  # test_anneal.cpp:77-103
    c4 = pi.Graph.parse_gset("4 4\n1 2 1\n2 3 1\n3 4 1\n4 1 1")
    p = pi.MinCutProblem.make_unchecked(c4, pi.Coefficients(1, 1, 1))
    hits = 0
    for seed in range(1, 11):
        r = pi.anneal(p, params(sweeps=100, flip_fraction0=0.2, decay_rate=0.9, deterministic=True, seed=seed))
        hits += pi.cut_value(c4, r.state) == 2 and pi.imbalance(r.state) == 0
    assert hits >= 6
    tuned = pi.MinCutProblem.with_default_coefficients(c4)
    for seed in range(1, 6):
        r = pi.anneal(tuned, params(sweeps=100, flip_fraction0=0.2, decay_rate=0.9, deterministic=True, seed=seed))
        assert pi.cut_value(c4, r.state) == 2 and pi.imbalance(r.state) == 0


def _random_weighted(n, m, rng):
    m = min(m, n * (n - 1) // 2)
    seen, edges = set(), []
    while len(edges) < m:
        u, v = sorted(int(x) for x in rng.integers(0, n, 2))
        if u == v or (u, v) in seen:
            continue
        seen.add((u, v))
        w = 0
        while w == 0:
            w = int(rng.integers(-3, 6))
        edges.append((u, v, w))
    return pi.Graph.from_edges(n, edges)


def test_greedy_descent_never_increases_h():  # test_anneal.cpp:105-131, acceptance crit. 3
    rng = np.random.default_rng(1234)
    for _ in range(8):
        n = int(8 + rng.integers(0, 30))
        g = _random_weighted(n, int(rng.integers(0, 3 * n + 1)), rng)
        c = pi.Coefficients(1, 4, 1)
        p = pi.MinCutProblem.make_unchecked(g, c)
        state = {"prev": None, "viol": 0, "n": 0}

        def on_update(node, spins):
            h = naive_h(g, c, spins)
            if state["prev"] is not None and h > state["prev"]:
                state["viol"] += 1
            state["prev"] = h
            state["n"] += 1

        pi.anneal(p, params(sweeps=20, flip_fraction0=0.0, deterministic=True, seed=int(rng.integers(1, 2**62))),
                  on_update=on_update)
        assert state["viol"] == 0 and state["n"] == 20 * n


def test_every_node_visited_once_per_sweep():  # test_anneal.cpp:133-144
    g = pi.random_graph(37, 60, 3)
    p = pi.MinCutProblem.with_default_coefficients(g)
    seen = []
    pi.anneal(p, params(sweeps=11, deterministic=True), on_update=lambda i, s: seen.append(i))
    assert len(seen) == 11 * 37
    assert seen[:37] == list(range(37)) and seen[-37:] == list(range(37))


@pytest.mark.parametrize("workers", [1, 4])
def test_counter_matches_spin_sum_at_every_barrier(workers):  # test_anneal.cpp:146-170, crit. 4
    g = pi.random_graph(1000, 3000, 17)
    p = pi.MinCutProblem.with_default_coefficients(g)
    rec = []
    pi.anneal(p, params(sweeps=50, workers=workers, flip_fraction0=0.2, decay_rate=0.99, seed=7),
              on_sweep_end=lambda k, s, c: rec.append((k, sum(s), c)))
    assert [k for k, _, _ in rec] == list(range(50))
    assert all(total == counter for _, total, counter in rec)


def test_deterministic_bit_reproducible():  # test_anneal.cpp:172-190
    g = pi.random_graph(200, 800, 9)
    p = pi.MinCutProblem.with_default_coefficients(g)
    a = pi.anneal(p, params(sweeps=60, deterministic=True, seed=42))
    b = pi.anneal(p, params(sweeps=60, deterministic=True, seed=42))
    assert a.state == b.state
    assert [(t.hamiltonian_scaled, t.cut, t.imbalance, t.flip_probability) for t in a.trace] == \
           [(t.hamiltonian_scaled, t.cut, t.imbalance, t.flip_probability) for t in b.trace]


def test_one_worker_equals_deterministic():  # test_anneal.cpp:192-207
    g = pi.random_graph(300, 900, 21)
    p = pi.MinCutProblem.with_default_coefficients(g)
    det = pi.anneal(p, params(sweeps=40, seed=13, deterministic=True))
    one = pi.anneal(p, params(sweeps=40, seed=13, workers=1))
    assert det.state == one.state
    assert [t.hamiltonian_scaled for t in det.trace] == [t.hamiltonian_scaled for t in one.trace]


def test_standard_equals_gdi_deterministic():  # test_anneal.cpp:209-226, acceptance crit. 8
    rng = pi.Rng(88)
    for _ in range(5):
        n = 10 + rng.next_below(40)
        g = pi.random_graph(n, 2 * n, rng.next())
        p = pi.MinCutProblem.with_default_coefficients(g)
        seed = rng.next()
        s = pi.anneal(p, params(sweeps=40, deterministic=True, seed=seed, strategy=pi.Strategy.standard))
        d = pi.anneal(p, params(sweeps=40, deterministic=True, seed=seed, strategy=pi.Strategy.gdi))
        assert s.state == d.state


def test_trace_flip_probability_schedule():  # test_anneal.cpp:228-244
    g = pi.random_graph(50, 100, 5)
    p = pi.MinCutProblem.with_default_coefficients(g)
    pa = params(sweeps=30, flip_fraction0=0.3, decay_rate=0.95, deterministic=True)
    r = pi.anneal(p, pa)
    assert len(r.trace) == 30
    assert [t.flip_probability for t in r.trace] == [pi.flip_probability(pa, k) for k in range(30)]
    assert all(r.trace[k].flip_probability <= r.trace[k - 1].flip_probability for k in range(1, 30))
    assert all(t.seconds >= 0 for t in r.trace) and r.seconds >= 0


def test_single_node_graph():  # test_anneal.cpp:246-255
    g = pi.Graph.from_edges(1, [])
    r = pi.anneal(pi.MinCutProblem.with_default_coefficients(g), params(sweeps=5, deterministic=True))
    assert len(r.state) == 1 and pi.imbalance(r.state) == 1


def test_smoke_c4_and_reproducibility():  # test_smoke.py:58-81
    c4 = pi.Graph.parse_gset("4 4\n1 2 1\n2 3 1\n3 4 1\n4 1 1")
    r = pi.anneal(pi.MinCutProblem.with_default_coefficients(c4), params(sweeps=100, deterministic=True, seed=1))
    assert pi.cut_value(c4, r.state) == 2 and pi.imbalance(r.state) == 0 and len(r.trace) == 100
    g = pi.random_graph(120, 400, 11)
    p = pi.MinCutProblem.with_default_coefficients(g)
    a = pi.anneal(p, params(sweeps=50, deterministic=True, seed=9))
    b = pi.anneal(p, params(sweeps=50, deterministic=True, seed=9))
    assert a.state == b.state and [t.cut for t in a.trace] == [t.cut for t in b.trace]


def test_smoke_oracle_agreement():  # test_smoke.py:84-99, acceptance crit. 2 in miniature
    g = pi.random_connected_gnp(10, 0.4, 5)
    oracle = pi.brute_force_balanced_mincut(g, 0)
    p = pi.MinCutProblem.with_default_coefficients(g)
    seeds = np.arange(100, 110, dtype=np.uint64)
    out = pi.anneal_batch(p, params(sweeps=300, deterministic=True), seeds)
    bal = out["imbalance"] == 0
    assert (out["cut"][bal] >= oracle.cut).all()
    assert int(out["cut"][bal].min()) == oracle.cut


def test_invalid_params_raise_config_error():
    g = pi.random_graph(20, 30, 1)
    p = pi.MinCutProblem.with_default_coefficients(g)
    with pytest.raises(pi.ConfigError):
        pi.anneal(p, params(sweeps=0))
    with pytest.raises(pi.ConfigError):
        pi.anneal(p, params(decay_rate=1.0))
