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


@pytest.mark.parametrize("world", [2, 4, 8])
def test_fused_partition_quality_and_consistency(m1, world):
    """Fused exchange (spin changes stored into every rank's copy during the
    sweep, only the counter deltas collected per sweep): remote spins are no
    longer a sweep stale, so the cut stays within 2% of the reference's
    deterministic cut at every W; ranks end identical; exact counter and cut."""
    doc, g, prob = m1
    out = sh.emulate_partitioned(prob, tparams(20), 1, world, fused=True)
    assert out["rank_spins_agree"]
    det = doc["runs"][0]["cut"]
    assert out["cut"] <= 1.02 * det, (out["cut"], det)
    assert out["imbalance"] <= 2
    s = out["spins"].astype(np.int64)
    assert int(s.sum()) == out["balance_counter"]
    assert int(pi.evaluate_batch(prob, out["spins"].reshape(1, -1))["cut"][0]) == out["cut"]


def _ipc_rank(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        pi.set_device(0)
        g = pi.random_graph(100000, 400000, 77)
        prob = pi.MinCutProblem.with_default_coefficients(g)
        out = sh.anneal_partitioned(prob, tparams(30), 5, dist, 0, fused=True)
        ev = int(pi.evaluate_batch(prob, out["spins"].reshape(1, -1))["cut"][0])
        q.put((rank, out["spins"].tobytes(), out["cut"], ev, out["imbalance"], out["balance_counter"],
               int(out["spins"].astype(np.int64).sum())))
    finally:
        dist.destroy_process_group()


def test_fused_partition_two_processes_cuda_ipc():
    """Two ranks as two processes (the real code path: CUDA IPC handles of the
    spin copies exchanged through torch.distributed, peer stores from the sweep
    kernels, gloo for the per-sweep deltas). They share one GPU here; all
    waiting happens on the host between launches, so no kernel waits on
    another rank's kernel."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    (_, sp0, cut0, ev0, imb0, ctr0, sum0), (_, sp1, cut1, ev1, imb1, ctr1, sum1) = got
    assert sp0 == sp1  # identical global spins on both ranks
    assert cut0 == cut1 == ev0 == ev1  # partial cuts sum to the exact cut
    assert imb0 == imb1 <= 2 and ctr0 == ctr1 == sum0 == sum1


def _nccl_graph_rank(port, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        pi.set_device(0)
        g = pi.random_graph(100000, 400000, 77)
        prob = pi.MinCutProblem.with_default_coefficients(g)
        pa = sh.PartitionedAnneal(prob, tparams(30), 5, dist, 0)
        a = pa.run()
        b = pa.run()  # a replay of the captured anneal
        graphed, err = pa.graph is not None, pa.graph_error
        pa.close()
        ev = [int(pi.evaluate_batch(prob, r["spins"].reshape(1, -1))["cut"][0]) for r in (a, b)]
        q.put((graphed, err, [r["cut"] for r in (a, b)], ev, [r["imbalance"] for r in (a, b)],
               [r["balance_counter"] == int(r["spins"].astype(np.int64).sum()) for r in (a, b)]))
    finally:
        dist.destroy_process_group()


def test_partitioned_anneal_nccl_cuda_graph():
    """The multi-rank driver's anneal (init + per sweep: sweep kernel, NCCL
    all-gather, finishing kernel) captured as one CUDA graph and replayed, here
    with a world of one NCCL rank: the capture succeeds and a replay gives an
    exact cut, an exact counter and a balanced result."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_graph_rank, args=(port, q))
    p.start()
    graphed, err, cuts, ev, imb, ctr_ok = q.get(timeout=600)
    p.join(timeout=120)
    assert graphed, err
    assert cuts == ev and all(i <= 2 for i in imb) and all(ctr_ok), (cuts, ev, imb, ctr_ok)
