"""Multi-rank host logic on the CPU (gloo, world_size 2): replica sharding and
the vertex-partition exchange driver (paper_1908_00210_b200/sharding.py).

The device kernels are replaced by a numpy stand-in with the same exchange
format (int64 delta + one uint32 per owned chunk), so what is checked here is
the plumbing that the GPU path uses unchanged: seed blocks, rank-major
all-gathers, partial-cut all-reduce, and that every rank ends with the same
global state.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1908_00210_b200 import sharding as sh


def test_replica_seed_blocks_partition_the_seed_range():
    blocks = [sh.replica_seeds(r, 4, 256) for r in range(4)]
    allseeds = np.concatenate(blocks)
    assert np.array_equal(allseeds, np.arange(1, 1 + 4 * 256, dtype=np.uint64))
    with pytest.raises(ValueError):
        sh.replica_seeds(4, 4, 1)


def test_solve_selection_lowest_h_first_seed_on_ties():  # ising_cli.cpp:160
    sc = np.array([[40, 10, 0, 7], [36, 9, 0, 9], [36, 9, 0, 3], [50, 8, 2, 1]])
    assert sh.select_solve(sc) == 2
    s = sh.summarize(sc, parity=0)
    assert s["cut"] == 9 and s["seed"] == 3 and s["best_balanced_cut"] == 9 and s["min_cut"] == 8


def test_owned_chunks_cover_every_chunk_once():
    n = 1000003
    seen = np.concatenate([sh.owned_chunks(n, r, 8) for r in range(8)])
    assert np.array_equal(np.sort(seen), np.arange((n + 31) // 32))
    assert sh.exchange_bytes(n, 8) % 16 == 0 and sh.exchange_bytes(n, 8) >= 8 + 4 * len(sh.owned_chunks(n, 0, 8))


class FakePartSession:
    """numpy stand-in for pyising.PartSession: owned chunks c = rank (mod W) of
    an identity order; a 'sweep' flips owned spins by a seeded rule."""

    def __init__(self, n, edges, world, rank, seed, sweeps):
        self.n, self.edges, self.W, self.r, self.S = n, edges, world, rank, sweeps
        self.rng = np.random.default_rng(seed)  # same seed on every rank -> same init
        self.s = np.where(self.rng.random(n) < 0.5, 1, -1).astype(np.int8)
        self.nb = sh.exchange_bytes(n, world)
        self.trace_cut, self.trace_imb, self.ctr = [], [], []
        self.G = int(self.s.sum())

    def init(self):
        pass

    def _owned(self):
        nck = (self.n + 31) // 32
        return [c for c in range(self.r, nck, self.W)]

    def sweep(self, k, send):
        delta = 0
        words = []
        for c in self._owned():
            lo, hi = 32 * c, min(32 * c + 32, self.n)
            flip = (np.arange(lo, hi) * 7 + k * 13 + self.r) % 5 == 0
            old = self.s[lo:hi].copy()
            self.s[lo:hi][flip] *= -1
            delta += int(self.s[lo:hi].sum() - old.sum())
            words.append(int(sum(1 << l for l in range(hi - lo) if self.s[lo + l] > 0)))
        buf = np.zeros(self.nb, np.uint8)
        buf[:8] = np.frombuffer(np.int64(delta).tobytes(), np.uint8)
        buf[8:8 + 4 * len(words)] = np.frombuffer(np.array(words, np.uint32).tobytes(), np.uint8)
        send[:] = torch.from_numpy(buf)

    def finish(self, k, recv):
        r = recv.numpy()
        tot = 0
        nck = (self.n + 31) // 32
        for q in range(self.W):
            part = r[q * self.nb:(q + 1) * self.nb]
            tot += int(np.frombuffer(part[:8].tobytes(), np.int64)[0])
            words = np.frombuffer(part[8:].tobytes(), np.uint32)
            if q == self.r:
                continue
            for i, c in enumerate(range(q, nck, self.W)):
                for l in range(min(32, self.n - 32 * c)):
                    self.s[32 * c + l] = 1 if (int(words[i]) >> l) & 1 else -1
        self.G += tot
        lo, hi = len(self.edges) * self.r // self.W, len(self.edges) * (self.r + 1) // self.W
        e = self.edges[lo:hi]
        self.trace_cut.append(int((self.s[e[:, 0]] != self.s[e[:, 1]]).sum()))
        self.trace_imb.append(abs(int(self.s.sum())))
        self.ctr.append(self.G)

    def fetch(self):
        return {"spins": self.s.copy(), "imbalance": self.trace_imb[-1], "balance_counter": self.ctr[-1],
                "trace_cut_part": np.array(self.trace_cut), "trace_imbalance": np.array(self.trace_imb),
                "counters": np.array(self.ctr), "seconds": 0.0}


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # replica sharding: rank-major gather of score rows, same summary everywhere
        seeds = sh.replica_seeds(rank, world, 3)
        res = {"hamiltonian_scaled": np.array([30, 20, 25]) + rank, "cut": np.array([7, 5, 6]) + rank,
               "imbalance": np.array([0, 0, 2]), }
        allsc = sh.gather_scores(sh.score_rows(res, seeds), dist)
        summ = sh.summarize(allsc, parity=0)
        # vertex partitioning through the real driver with the numpy stand-in
        n, S = 300, 4
        rng = np.random.default_rng(5)
        edges = np.unique(np.sort(rng.integers(0, n, size=(900, 2)), 1), axis=0)
        edges = edges[edges[:, 0] != edges[:, 1]]
        fs = FakePartSession(n, edges, world, rank, 11, S)
        send = torch.zeros(fs.nb, dtype=torch.uint8)
        recv = torch.zeros(world * fs.nb, dtype=torch.uint8)
        out = sh.run_partitioned([fs], S, lambda: dist.all_gather_into_tensor(recv, send),
                                 lambda i: (send, recv))

        def ar(a):
            t = torch.as_tensor(a)
            dist.all_reduce(t)
            return t.numpy()

        comb = sh.combine(out, ar)
        full_cut = int((comb["spins"][edges[:, 0]] != comb["spins"][edges[:, 1]]).sum())
        q.put((rank, allsc.tolist(), summ, comb["spins"].tolist(), comb["cut"], full_cut,
               int(comb["spins"].astype(np.int64).sum()), comb["balance_counter"]))
    finally:
        dist.destroy_process_group()


class _RecSession:
    """Stands in for a PartSession: records the driver's call order."""

    def __init__(self, log, name):
        self.log, self.name = log, name

    def init(self):
        self.log.append(("init", self.name))

    def sweep(self, k, send):
        self.log.append(("sweep", self.name, k))

    def finish(self, k, recv):
        self.log.append(("finish", self.name, k))

    def fetch(self):
        return {}


def test_run_partitioned_fused_barrier_order():
    """Fused exchange (sweep kernels store into the other ranks' spin copies):
    no rank may start sweep 0 before every rank initialised its copy, nor
    sweep k+1 before every rank finished sweep k (tail replay, cut) on its
    copy. run_partitioned calls the barrier after init and between sweeps."""
    log = []
    ss = [_RecSession(log, r) for r in range(2)]
    sh.run_partitioned(ss, 3, lambda: log.append(("exchange",)), lambda i: (0, 0),
                       barrier=lambda: log.append(("barrier",)))
    kinds = [e[0] for e in log]
    assert kinds == ["init", "init", "barrier",
                     "sweep", "sweep", "exchange", "finish", "finish", "barrier",
                     "sweep", "sweep", "exchange", "finish", "finish", "barrier",
                     "sweep", "sweep", "exchange", "finish", "finish"]
    # unfused: no barrier at all
    log.clear()
    sh.run_partitioned(ss, 2, lambda: log.append(("exchange",)), lambda i: (0, 0))
    assert ("barrier",) not in log and [e[0] for e in log].count("sweep") == 4


def test_gloo_world2_sharding_and_partition_exchange():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    (r0, sc0, su0, sp0, cut0, full0, sum0, ctr0), (r1, sc1, su1, sp1, cut1, full1, sum1, ctr1) = got
    assert sc0 == sc1 and len(sc0) == 6 and [row[3] for row in sc0] == [1, 2, 3, 4, 5, 6]
    assert su0 == su1 and su0["seed"] == 2 and su0["cut"] == 5
    assert sp0 == sp1  # every rank ends with the same global spins
    assert cut0 == cut1 == full0 == full1  # partial cuts sum to the full cut
    assert sum0 == ctr0 == sum1 == ctr1  # counter = sum of spins on every rank
