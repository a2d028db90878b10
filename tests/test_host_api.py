"""Host-side solver API on CPU (no GPU needed).

Ports of reference proj/tests/test_graph.cpp, test_model.cpp and
test_evaluate.cpp cases and the non-anneal parts of
proj/python/tests/test_smoke.py, run against the product's C++ host code
through pyising. Generators are checked bit-for-bit against the reference
(golden G-set hashes) and the RNG against the C restatement.
"""
import numpy as np
import pytest

import paper_1908_00210_b200 as pi
from oracle import oracle as o
from tests.helpers import fnv_bytes, golden_configs, product_graph


# ---------------------------------------------------------------- graph I/O

def test_parse_smallest_graph():  # test_graph.cpp:10-19
    g = pi.Graph.parse_gset("2 1\n1 2 1")
    assert (g.num_nodes, g.num_edges, g.max_degree) == (2, 1, 1)
    assert g.neighbors(0) == [(1, 1)] and g.neighbors(1) == [(0, 1)]


@pytest.mark.parametrize("text", ["3 1\n1 4 1", "2 1\n1 1 1", "2 1\n1 2", "2 1\nx y z", "2 2\n1 2 1",
                                  "2 1\n1 2 1\n2 1 3", "", "0 0", "2 1\n1 2 99999999999", "-1 0"])
def test_parse_errors(text):  # test_graph.cpp:32-49
    with pytest.raises(pi.ParseError):
        pi.Graph.parse_gset(text)


def test_parse_error_line_numbers():
    with pytest.raises(pi.ParseError, match="line 2"):
        pi.Graph.parse_gset("2 1\n1 4 1")
    with pytest.raises(pi.ParseError, match="line 5"):
        pi.Graph.parse_gset("% c\n\n3 2\n1 2 1\n1 2 1\n")


def test_comments_blanks_negative_weights_isolated():  # test_graph.cpp:51-63
    g = pi.Graph.parse_gset("% mirror header\n# another comment\n\n4 2\n1 2 -1\n\n2 3 5\n")
    assert (g.num_nodes, g.num_edges) == (4, 2)
    assert not g.all_unit_weights and g.degree(3) == 0
    u = g.with_unit_weights()
    assert u.all_unit_weights and u.neighbors(0)[0][1] == 1 and g.neighbors(0)[0][1] == -1


def test_density():  # test_graph.cpp:65-75
    k4 = pi.Graph.parse_gset("4 6\n1 2 1\n1 3 1\n1 4 1\n2 3 1\n2 4 1\n3 4 1")
    assert pi.density(k4) == 1.0
    assert pi.density(pi.Graph.parse_gset("2 0\n")) == 0.0
    with pytest.raises(pi.DomainError):
        pi.density(pi.Graph.from_edges(1, []))


def test_roundtrip_and_degree_sum():  # test_graph.cpp:77-108
    rng = pi.Rng(123)
    for _ in range(20):
        n = 5 + rng.next_below(40)
        m = rng.next_below(n * (n - 1) // 2 + 1)
        g = pi.random_graph(n, m, rng.next())
        h = pi.Graph.parse_gset(g.to_gset())
        assert h.to_gset() == g.to_gset()
        assert [(e.u, e.v, e.weight) for e in h.edges()] == [(e.u, e.v, e.weight) for e in g.edges()]
        assert sum(g.degree(v) for v in range(n)) == 2 * g.num_edges


def test_from_edges_validation():
    with pytest.raises(pi.DomainError):
        pi.Graph.from_edges(0, [])
    with pytest.raises(pi.DomainError):
        pi.Graph.from_edges(3, [(0, 3, 1)])
    with pytest.raises(pi.DomainError):
        pi.Graph.from_edges(3, [(1, 1, 1)])
    with pytest.raises(pi.DomainError):
        pi.Graph.from_edges(3, [(0, 1, 1), (1, 0, 2)])


# ---------------------------------------------------------------- generators

@pytest.mark.parametrize("name", ["G1", "G22", "G55", "G81pm1", "G47", "G43", "G32"])
def test_product_generators_match_reference(name):
    doc = golden_configs()[name]
    g = product_graph(doc["recipe"])
    assert (g.num_nodes, g.num_edges, g.max_degree) == (doc["n"], doc["m"], doc["max_degree"])
    assert f"{fnv_bytes(g.to_gset().encode()):016x}" == doc["gset_fnv"]


def test_generator_shapes():  # test_graph.cpp:120-133
    t = pi.torus_graph(100, 20, 32)
    assert (t.num_nodes, t.num_edges, t.max_degree) == (2000, 4000, 4)
    assert pi.random_tree(10000, 70).num_edges == 9999
    assert pi.random_connected_gnp(12, 0.3, 9).num_nodes == 12
    with pytest.raises(pi.DomainError):
        pi.random_graph(1, 0, 1)
    with pytest.raises(pi.DomainError):
        pi.torus_graph(2, 5, 1)


def test_product_rng_matches_restatement():
    r = pi.Rng.stream(7, 1)
    assert [r.next() for _ in range(64)] == o.draws(7, 1, 64).tolist()


# ---------------------------------------------------------------- model

def test_coefficient_rule():  # test_model.cpp:23-57, test_smoke.py:34-44
    star = pi.Graph.from_edges(2000, [pi.Edge(0, v, 1) for v in range(1, 5)])
    c = pi.coefficients_for(star)
    assert c.a == 1.0 and c.b == 1.0
    with pytest.raises(pi.ConfigError):
        pi.MinCutProblem.make(star, pi.Coefficients(1, 4, 1))
    pi.MinCutProblem.make_unchecked(star, pi.Coefficients(1, 4, 1))
    c2 = pi.coefficients_for(pi.Graph.parse_gset("2 1\n1 2 1"), 2, 1)
    assert c2.a == 0.5 and c2.b == 2.0
    with pytest.raises(pi.ConfigError):
        pi.MinCutProblem.make_unchecked(star, pi.Coefficients(0, 4, 1))


def test_hamiltonian_identity_and_candidates():  # test_model.cpp:94-185, test_smoke.py:47-55
    rng = np.random.default_rng(5)
    for _ in range(30):
        g = pi.random_graph(40, 90, int(rng.integers(1, 1 << 30)))
        c = pi.Coefficients(int(rng.integers(1, 5)), int(rng.integers(1, 5)), 1)
        p = pi.MinCutProblem.make_unchecked(g, c)
        s = [1 if x else -1 for x in rng.integers(0, 2, 40)]
        h = pi.global_hamiltonian_scaled(p, s)
        assert h == c.a_num * sum(s) ** 2 + c.b_num * pi.cut_value(g, s)
        i = int(rng.integers(0, 40))
        ce = pi.candidate_energies_mincut(p, s, sum(s) - s[i], i)
        # flip-delta consistency: E(-s_i) - E(s_i) == H(flipped) - H(s)
        t = list(s)
        t[i] = -s[i]
        e_own, e_flip = (ce.at_plus_scaled, ce.at_minus_scaled) if s[i] > 0 else (ce.at_minus_scaled, ce.at_plus_scaled)
        assert e_flip - e_own == pi.global_hamiltonian_scaled(p, t) - h


def test_local_field_examples():  # test_model.cpp:59-92
    g = pi.Graph.parse_gset("2 1\n1 2 1")
    p = pi.MinCutProblem.make_unchecked(g, pi.Coefficients(1, 2, 1))
    assert pi.local_field(p, [1, 1], 0) == 1.0
    with pytest.raises(pi.DomainError):
        pi.local_field(p, [1, 1], 5)


# ---------------------------------------------------------------- evaluation

def test_cut_imbalance_score():  # test_evaluate.cpp
    c4 = pi.Graph.parse_gset("4 4\n1 2 1\n2 3 1\n3 4 1\n4 1 1")
    assert pi.cut_value(c4, [1, 1, -1, -1]) == 2
    assert pi.imbalance([1, 1, -1]) == 1 and pi.imbalance([1] * 5) == 5
    p = pi.MinCutProblem.with_default_coefficients(c4)
    sc = pi.score(p, [1, 1, -1, -1])
    assert (sc.cut, sc.imbalance, sc.hamiltonian_scaled) == (2, 0, 8)
    with pytest.raises(pi.DomainError):
        pi.cut_value(c4, [1, 1])


def test_brute_force_oracle():  # test_smoke.py:58-66, test_evaluate.cpp:58-81
    p4 = pi.Graph.parse_gset("4 3\n1 2 1\n2 3 1\n3 4 1")
    r = pi.brute_force_balanced_mincut(p4, 0)
    assert r.cut == 1 and r.witness == [1, 1, -1, -1]
    k4 = pi.Graph.parse_gset("4 6\n1 2 1\n1 3 1\n1 4 1\n2 3 1\n2 4 1\n3 4 1")
    assert pi.brute_force_balanced_mincut(k4, 0).cut == 4
    with pytest.raises(pi.CapacityError):
        pi.brute_force_balanced_mincut(pi.random_tree(30, 1), 0)
    with pytest.raises(pi.DomainError):
        pi.brute_force_balanced_mincut(pi.Graph.parse_gset("3 1\n1 2 1"), 0)
    # exhaustive cross-check on small random graphs (test_support.hpp:36-51)
    rng = np.random.default_rng(9)
    for _ in range(10):
        n = int(rng.integers(4, 11))
        g = pi.random_graph(n, int(rng.integers(0, n * (n - 1) // 2 + 1)), int(rng.integers(1, 1 << 30)))
        best = min(pi.cut_value(g, [1 if (mask >> i) & 1 else -1 for i in range(n)])
                   for mask in range(1 << n) if abs(2 * bin(mask).count("1") - n) <= n % 2)
        assert pi.brute_force_balanced_mincut(g, n % 2).cut == best


# ---------------------------------------------------------------- annealer params

def test_params_validation_and_schedule():  # test_anneal.cpp:14-58
    p = pi.AnnealParams()
    p.sweeps, p.flip_fraction0, p.decay_rate = 1000, 0.20, 0.99
    assert pi.flip_probability(p, 0) == 0.20
    assert abs(pi.flip_probability(p, 999) - 0.20 * 0.99 ** 999) < 1e-9
    with pytest.raises(pi.ConfigError):
        pi.flip_probability(p, 1000)
    d = pi.default_params_for(pi.Strategy.gdi, pi.random_graph(100, 200, 1))
    s = pi.default_params_for(pi.Strategy.standard, pi.random_graph(100, 200, 1))
    assert d.flip_fraction0 == 0.04 and s.flip_fraction0 == 5 * d.flip_fraction0
    assert (d.decay_rate, d.sweeps) == (0.99, 1000)
    d.deterministic, d.workers = True, 8
    assert d.validated().workers == 1
    bad = pi.AnnealParams()
    bad.sweeps = 0
    with pytest.raises(pi.ConfigError):
        bad.validated()
    bad.sweeps, bad.flip_fraction0 = 10, 1.5
    with pytest.raises(pi.ConfigError):
        bad.validated()
    assert pi.strategy_from_string("gdi") == pi.Strategy.gdi
    with pytest.raises(pi.ConfigError):
        pi.strategy_from_string("metropolis")


def test_anneal_fails_loudly_without_gpu():
    """No CPU fallback: without a CUDA device the product path raises."""
    if pi.device_count() > 0:
        pytest.skip("a GPU is visible")
    p = pi.MinCutProblem.with_default_coefficients(pi.random_graph(20, 30, 1))
    params = pi.AnnealParams()
    params.deterministic = True
    with pytest.raises(RuntimeError, match="no CUDA device"):
        pi.anneal(p, params)
    with pytest.raises(RuntimeError):
        pi.anneal_batch(p, params, np.arange(1, 4, dtype=np.uint64))
