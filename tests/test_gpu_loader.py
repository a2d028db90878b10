"""Device-side loader (csrc/layout.cu): statistics of the validation pass and
the lazily built kernel layouts, checked against host-side numpy on the same
CSR through the C ABI (gdi_graph_create / gdi_graph_query)."""
import ctypes

import numpy as np
import pytest

import paper_1908_00210_b200 as pi

pytestmark = pytest.mark.gpu


class Info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int64), ("max_degree", ctypes.c_int32),
                ("device", ctypes.c_int32), ("all_unit_weights", ctypes.c_int32), ("device_bytes", ctypes.c_int64)]


@pytest.fixture(scope="module")
def lib():
    lib = ctypes.CDLL(pi.LIBGDI)
    lib.gdi_last_error.restype = ctypes.c_char_p
    VP = ctypes.c_void_p  # pointers must be declared (bare Python ints pass as 32-bit ints)
    lib.gdi_graph_create.argtypes = [ctypes.c_int, ctypes.c_int32, VP, VP, VP, ctypes.POINTER(VP)]
    lib.gdi_graph_query.argtypes = [VP, ctypes.POINTER(Info)]
    lib.gdi_graph_destroy.argtypes = [VP]
    return lib


def query(lib, g, weighted):
    off, nbr, w = g.csr()
    off = np.ascontiguousarray(off, np.int64)
    nbr = np.ascontiguousarray(nbr, np.int32)
    w = np.ascontiguousarray(w, np.int32)
    h = ctypes.c_void_p()
    rc = lib.gdi_graph_create(0, g.num_nodes, off.ctypes.data, nbr.ctypes.data,
                              w.ctypes.data if weighted else None, ctypes.byref(h))
    assert rc == 0, lib.gdi_last_error()
    info = Info()
    assert lib.gdi_graph_query(h, ctypes.byref(info)) == 0
    lib.gdi_graph_destroy(h)
    return info, np.diff(off)


@pytest.mark.parametrize("n,m,seed", [(1000, 9990, 47), (300000, 1200000, 3)])
def test_device_validation_statistics_unit(lib, n, m, seed):
    g = pi.random_graph(n, m, seed)
    info, deg = query(lib, g, weighted=False)
    assert (info.n, info.m) == (n, m)
    assert info.max_degree == int(deg.max()) == g.max_degree
    assert info.all_unit_weights == 1 and info.device_bytes > 0


def test_device_validation_statistics_weighted(lib):
    t = pi.torus_graph(60, 50, 9)
    rng = pi.Rng(9)
    g = pi.Graph.from_edges(t.num_nodes, [(e.u, e.v, 1 if rng.coin() else -1) for e in t.edges()])
    info, deg = query(lib, g, weighted=True)
    assert info.all_unit_weights == 0 and info.max_degree == int(deg.max())
    # weights given but all 1: recognised as unit
    info1, _ = query(lib, pi.random_graph(500, 2000, 1), weighted=True)
    assert info1.all_unit_weights == 1


@pytest.mark.gpu
@pytest.mark.parametrize("mode_workers", [1, 8])
def test_one_shot_trace_columns_match_records(mode_workers, monkeypatch):
    """anneal_batch_fresh (gdi_anneal_batch_columns: the trace written straight
    into numpy columns) returns what anneal_batch (records, then columns)
    does: same spins, scores, trace and flip probabilities; positive sweep
    times. Exact mode and the pooled mode (its run-to-run reproducible
    one-warp-per-replica kernel: k2_chains races its chains)."""
    from tests.helpers import golden_configs, product_graph

    monkeypatch.setenv("GDI_FORCE_KERNEL", "k2_gather" if mode_workers > 1 else "auto")
    g = product_graph(golden_configs()["G22"]["recipe"])
    prob = pi.MinCutProblem.with_default_coefficients(g)
    p = pi.AnnealParams()
    p.sweeps = 50
    p.workers = mode_workers
    p.deterministic = mode_workers == 1
    seeds = np.arange(1, 33, dtype=np.uint64)
    a = pi.anneal_batch(prob, p, seeds, True)
    b = pi.anneal_batch_fresh(prob, p, seeds, True)
    assert np.array_equal(a["spins"], b["spins"])
    assert np.array_equal(a["cut"], b["cut"]) and np.array_equal(a["imbalance"], b["imbalance"])
    assert np.array_equal(a["trace"], b["trace"])
    assert np.array_equal(a["flip_probability"], b["flip_probability"])
    assert b["trace_seconds"].shape == (32, 50) and (b["trace_seconds"] > 0).all()
    c = pi.anneal_batch_fresh(prob, p, seeds, False)
    assert "trace" not in c and np.array_equal(c["spins"], b["spins"])
