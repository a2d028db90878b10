"""Vertex-partitioned throughput anneal (the 1M-vertex
config) with W ranks emulated on one GPU (sharding.emulate_partitioned: W
device sessions in one process, the per-sweep all-gather done as a device
copy; the ranks' kernels never wait on each other, so the semantics are those
of W GPUs). Statistical parity with the tolerances stated in each test."""
import numpy as np
import pytest

import paper_1908_00210_b200 as pi
from paper_1908_00210_b200 import sharding as sh
from tests.helpers import golden_configs, product_graph

pytestmark = pytest.mark.gpu


def tparams(sweeps):
    p = pi.AnnealParams()
    p.sweeps, p.workers = sweeps, 8
    return p


@pytest.fixture(scope="module")
def m1():
    doc = golden_configs()["M1"]
    g = product_graph(doc["recipe"])
    return doc, g, pi.MinCutProblem.with_default_coefficients(g)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_partitioned_m1_quality_and_consistency(m1, world):
    """Remote spins are one sweep stale on every rank, so the cut grows with
    W on this short (20-sweep) schedule: measured +0.3% (W=1) to +6% (W=8)
    over the reference's deterministic cut 1252631. Tolerance: no worse than
    the reference's own pooled mode on this graph (1.342M with 16 workers,
    i.e. 7.1% over the deterministic cut); imbalance <= 2 (the global tail is
    replayed identically on every rank); identical spins on every rank; exact
    counter and cut."""
    doc, g, prob = m1
    out = sh.emulate_partitioned(prob, tparams(20), 1, world)
    assert out["rank_spins_agree"]
    det = doc["runs"][0]["cut"]
    assert out["cut"] <= 1.071 * det, (out["cut"], det)
    assert out["imbalance"] <= 2
    s = out["spins"].astype(np.int64)
    assert int(s.sum()) == out["balance_counter"] and abs(int(s.sum())) == out["imbalance"]
    ev = pi.evaluate_batch(prob, out["spins"].reshape(1, -1))
    assert int(ev["cut"][0]) == out["cut"]  # partial cuts sum to the exact cut
    assert (np.abs(out["counters"]) == out["trace_imbalance"]).all()


def test_partitioned_world1_matches_single_device_quality(m1):
    doc, g, prob = m1
    a = sh.emulate_partitioned(prob, tparams(20), 1, 1)
    s = pi.Session(prob, tparams(20), 1, trace=True)
    s.set_seeds(np.array([1], dtype=np.uint64))
    s.launch()
    s.sync()
    b = s.fetch(spins=True, trace=True)
    assert abs(a["cut"] - int(b["cut"][0])) <= 0.01 * int(b["cut"][0])
