"""K3 (k3_eval.cu) — fused exact cut + spin sum, against the C restatement of
evaluate.cpp:10-32 (oracle.cut) on the same spins, for both kernel shapes:
bit-sliced over 32 replicas (k3_sliced: R >= 16, |w| == 1, 4n bytes of
shared memory) and bit-packed per replica (k3_pack + k3_bits: few replicas,
general weights, the 1M-vertex graph, int2 edges beyond 65536 vertices).
Integer results: bit-exact."""
import numpy as np
import pytest

import paper_1908_00210_b200 as pi
from oracle import oracle as o
from tests.helpers import product_graph

pytestmark = pytest.mark.gpu


def _spins(R, n, seed, p=0.5):
    rng = np.random.default_rng(seed)
    return np.where(rng.random((R, n)) < p, 1, -1).astype(np.int8)


def _graph_pair(n, edges):
    g = pi.Graph.from_edges(n, [(u, v, w) for u, v, w in edges])
    eu, ev, ew = (np.array(x, np.int32) for x in zip(*edges))
    return g, o.csr_from_edges(n, eu, ev, ew)


def _check(g, og, spins, a_num=1, b_num=4):
    prob = pi.MinCutProblem.with_default_coefficients(g)
    sc = pi.evaluate_batch(prob, spins)
    for r in range(spins.shape[0]):
        cut = o.cut(og, spins[r])
        bal = int(spins[r].astype(np.int64).sum())
        assert sc["cut"][r] == cut, (r, sc["cut"][r], cut)
        assert sc["imbalance"][r] == abs(bal)
    return sc


@pytest.mark.parametrize("R", [1, 5, 16, 31, 32, 33, 100, 1024])
def test_k3_unit_graph_all_replica_counts(R):
    # G22 shape: R < 16 -> pack + bits, R >= 16 -> bit-sliced (partial last group for 31, 33, 100)
    g = product_graph(["random", "2000", "19990", "22"])
    og = o.recipe("random:2000:19990:22")
    _check(g, og, _spins(R, 2000, R))


@pytest.mark.parametrize("R", [3, 64])
def test_k3_pm1_torus(R):
    g = product_graph(["torus_pm1", "100", "200", "81"])
    og = o.recipe("torus_pm1:100:200:81")
    _check(g, og, _spins(R, g.num_nodes, 11 + R))


@pytest.mark.parametrize("R", [2, 40])
def test_k3_general_weights_and_odd_n(R):
    # weights in [-5, 5] \ {0}, n = 1001 (rows not 4-byte aligned, last word partial)
    rng = np.random.default_rng(5)
    n, seen, edges = 1001, set(), []
    while len(edges) < 6000:
        u, v = sorted(rng.integers(0, n, 2).tolist())
        if u == v or (u, v) in seen:
            continue
        seen.add((u, v))
        w = int(rng.integers(1, 6)) * (1 if rng.random() < 0.5 else -1)
        edges.append((u, v, w))
    g, og = _graph_pair(n, edges)
    _check(g, og, _spins(R, n, 7))


@pytest.mark.parametrize("R", [1, 48])
def test_k3_pm1_odd_n_sliced_and_bits(R):
    rng = np.random.default_rng(9)
    n, seen, edges = 333, set(), []
    while len(edges) < 1500:
        u, v = sorted(rng.integers(0, n, 2).tolist())
        if u == v or (u, v) in seen:
            continue
        seen.add((u, v))
        edges.append((u, v, 1 if rng.random() < 0.6 else -1))
    g, og = _graph_pair(n, edges)
    _check(g, og, _spins(R, n, 13, p=0.3))


def test_k3_wide_edges_beyond_65536_vertices():
    # n = 100000: int2 edge list; a few replicas (bits path) and 20 (sliced needs 4n <= 200 KB: 400 KB -> bits)
    g = product_graph(["random", "100000", "400000", "77"])
    og = o.recipe("random:100000:400000:77")
    for R in (1, 20):
        _check(g, og, _spins(R, 100000, 17 + R))


def test_k3_edge_cases_all_equal_and_empty_graph():
    g = product_graph(["random", "2000", "19990", "22"])
    og = o.recipe("random:2000:19990:22")
    for val in (1, -1):
        for R in (2, 32):
            sc = _check(g, og, np.full((R, 2000), val, np.int8))
            assert (sc["cut"] == 0).all()
    g0, og0 = pi.Graph.from_edges(40, []), o.csr_from_edges(40, [], [], [])
    _check(g0, og0, _spins(33, 40, 3))


def test_k3_rejects_non_spin_bytes():
    g = product_graph(["random", "2000", "19990", "22"])
    prob = pi.MinCutProblem.with_default_coefficients(g)
    for R in (3, 40):
        s = _spins(R, 2000, 1)
        s[R - 1, 1234] = 0
        with pytest.raises(pi.DomainError):
            pi.evaluate_batch(prob, s)
        s[R - 1, 1234] = 2
        with pytest.raises(pi.DomainError):
            pi.evaluate_batch(prob, s)


def test_k3_device_entry_point_matches_host():
    """gdi_evaluate_device on device-resident spins (the bench's K3 leg) equals
    the host path, on the same stream, with the bad flag left clear."""
    import torch

    g = product_graph(["random", "2000", "19990", "22"])
    prob = pi.MinCutProblem.with_default_coefficients(g)
    ev = pi.Evaluator(prob)
    spins = _spins(1024, 2000, 21)
    ref = ev.evaluate(spins)
    d = torch.from_numpy(spins).cuda()
    out = torch.zeros((1024, 2), dtype=torch.int64, device="cuda")
    bad = torch.ones(1, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(2):  # (scratch reused between calls)
        ev.evaluate_device(d.data_ptr(), 1024, out.data_ptr(), bad.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert got[:, 0].tolist() == ref["cut"].tolist()
    assert np.abs(got[:, 1]).tolist() == ref["imbalance"].tolist()
    assert int(bad.item()) == 0
