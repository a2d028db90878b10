"""Multi-GPU drivers: one process per GPU, torch.distributed
(NCCL) for the plumbing, libgdi kernels for the work.

* Replica sharding (G1/G22/G55/G81): replicas are independent, so each rank
  anneals its own contiguous block of seeds with no data-path collective;
  one small all-gather of per-replica scores after the run selects the result
  with the reference's rules (solve: lowest H_scaled, first seed on ties,
  ising_cli.cpp:160; bench: best balanced cut, bench.cpp:181-193).
* Vertex partitioning (the 1M-vertex graph): one replica over W ranks. Rank r
  owns the chunks c = r (mod W) of the degree-binned order (K4 chains
  r, r + W, ...) and keeps a full spin copy. Fused (default): every spin
  change is stored by the sweep kernel itself into the other ranks' copies
  through peer memory (NVLink; CUDA IPC handles exchanged once), and the
  per-sweep collective only sums the counter deltas. Unfused: once per sweep,
  all-gather the spin word of every owned chunk plus the delta (include/gdi.h
  gdi_part_*). Each rank counts the cut over the rows of its own chunks;
  partial cuts are summed at the end with one all-reduce.

`emulate_partitioned` runs the W ranks as W sessions in one process on one
device, the exchange being a device-side concatenation: the ranks' kernels
never wait on each other (the exchange happens between launches), so this
reproduces the multi-GPU semantics exactly on one GPU for testing.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np


# ---------------------------------------------------------------- replica sharding


def replica_seeds(rank: int, world: int, per_rank: int, seed0: int = 1) -> np.ndarray:
    """Contiguous seed block of `rank` (weak scaling: per_rank seeds each)."""
    if not (0 <= rank < world) or per_rank < 1:
        raise ValueError("bad rank/world/per_rank")
    return np.arange(seed0 + rank * per_rank, seed0 + (rank + 1) * per_rank, dtype=np.uint64)


def select_solve(scores: np.ndarray) -> int:
    """Row index of the solve winner in an (R, 4) array of
    {hamiltonian_scaled, cut, imbalance, seed}: lowest H, first seed on ties
    (reference ising_cli.cpp:160)."""
    return int(np.lexsort((scores[:, 3], scores[:, 0]))[0])


def summarize(scores: np.ndarray, parity: int) -> dict:
    """Bench-style summary (bench.cpp:181-193) + the solve winner."""
    win = select_solve(scores)
    bal = scores[scores[:, 2] <= parity]
    return {"cut": int(scores[win, 1]), "imbalance": int(scores[win, 2]), "seed": int(scores[win, 3]),
            "best_balanced_cut": int(bal[:, 1].min()) if len(bal) else None,
            "min_cut": int(scores[:, 1].min()), "min_imbalance": int(scores[:, 2].min()),
            "mean_cut": float(scores[:, 1].mean())}


def gather_scores(local: np.ndarray, dist=None, device=None) -> np.ndarray:
    """All-gather the (R, 4) int64 score rows of every rank (rank-major)."""
    import torch

    t = torch.as_tensor(np.ascontiguousarray(local, dtype=np.int64), device=device)
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return t.cpu().numpy()
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return torch.cat(parts).cpu().numpy()


def score_rows(res: dict, seeds: np.ndarray) -> np.ndarray:
    return np.stack([res["hamiltonian_scaled"], res["cut"], res["imbalance"], seeds.astype(np.int64)], 1)


# ---------------------------------------------------------------- vertex partitioning


def owned_chunks(n: int, rank: int, world: int) -> np.ndarray:
    """Chunks (32 vertices of the degree-binned order) owned by `rank`."""
    nck = (n + 31) // 32
    return np.arange(rank, nck, world)


def exchange_bytes(n: int, world: int) -> int:
    """Per-rank send buffer: int64 delta + one uint32 per owned chunk (rank 0
    owns the most), padded to 16 bytes (matches part_exchange_bytes)."""
    nck = (n + 31) // 32
    words = (nck + world - 1) // world
    return (8 + 4 * words + 15) & ~15


def run_partitioned(sessions: Sequence, sweeps: int, exchange: Callable, buffers: Callable,
                    barrier: Callable | None = None):
    """Drive W' local sessions (W' = 1 per process on real GPUs, W on one GPU
    when emulating) through init + per-sweep sweep / exchange / finish.

    buffers(i) -> (send_ptr, recv_ptr) for local session i; exchange() moves
    every rank's send buffer into every rank's recv buffer (rank-major).
    barrier(), with the fused exchange: no rank may start sweep k+1 (whose
    kernel stores into the other ranks' spin copies) before every rank has
    finished sweep k's barrier work on its copy (tail replay, cut), nor sweep 0
    before every rank has initialised its copy."""
    for s in sessions:
        s.init()  # writes the whole local copy: peers must not store into it before this
    if barrier is not None:
        barrier()
    for k in range(sweeps):
        for i, s in enumerate(sessions):
            s.sweep(k, buffers(i)[0])
        exchange()
        for i, s in enumerate(sessions):
            s.finish(k, buffers(i)[1])
        if barrier is not None and k + 1 < sweeps:
            barrier()
    return [s.fetch() for s in sessions]


def combine(results: Sequence[dict], all_reduce_sum: Callable | None = None) -> dict:
    """Global result from per-rank fetches: cuts are summed over ranks (local
    list, plus all_reduce_sum over processes when given); spins, imbalance and
    counters are global on every rank."""
    tc = np.sum([r["trace_cut_part"] for r in results], axis=0).astype(np.int64)
    if all_reduce_sum is not None:
        tc = all_reduce_sum(tc)
    r0 = results[0]
    return {"spins": r0["spins"], "cut": int(tc[-1]), "imbalance": int(r0["imbalance"]),
            "trace_cut": tc, "trace_imbalance": r0["trace_imbalance"], "counters": r0["counters"],
            "balance_counter": int(r0["balance_counter"]), "seconds": max(r["seconds"] for r in results)}


class PartitionedAnneal:
    """One rank's reusable vertex-partitioned anneal (call collectively on every
    rank; process group initialised, one GPU per rank). The session, the peer
    mappings (fused: CUDA IPC handles exchanged once) and the exchange buffers
    are set up here, outside any timed region; run() is one whole anneal
    (init + all sweeps). Under NCCL the anneal's launch sequence - per sweep the
    sweep kernel, the all-gather of the send buffers, the finishing kernel and
    (fused) the barrier all-reduce - is captured once as a CUDA graph and each
    run() replays it: 2 of our launches + 1-2 collectives per sweep, no host
    work between them. close() tears the peer mappings down in the order
    gdi.h gdi_part_detach asks for."""

    def __init__(self, problem, params, seed: int, dist, device: int, stream=None, fused: bool = True,
                 graph: bool = True):
        import torch

        import paper_1908_00210_b200 as pi

        self.dist, self.sweeps = dist, params.sweeps
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        self.dev = torch.device("cuda", device)
        self.stream = stream or torch.cuda.Stream(self.dev)
        self.ps = pi.PartSession(problem, params, self.world, self.rank, int(seed), stream=self.stream.cuda_stream,
                                 device=device)
        self.fused = fused and self.world > 1
        if self.fused:
            handles = [None] * self.world
            dist.all_gather_object(handles, self.ps.ipc_handle())
            self.ps.attach_peers(b"".join(handles))
        nb = self.ps.exchange_bytes
        self.nccl = dist.get_backend() == "nccl"
        self.cdev = self.dev if self.nccl else torch.device("cpu")
        self.send = torch.zeros(nb, dtype=torch.uint8, device=self.dev)
        self.recv = torch.zeros(self.world * nb, dtype=torch.uint8, device=self.dev)
        self.token = torch.zeros(1, dtype=torch.int32, device=self.cdev)
        self.graph = None
        self.use_graph = graph and self.nccl
        self.graph_error = None

    def _exchange(self):
        import torch

        if self.nccl:
            self.dist.all_gather_into_tensor(self.recv, self.send)
        else:  # gloo (multi-rank rehearsal on fewer GPUs): host-staged
            self.stream.synchronize()
            out = torch.empty(self.recv.numel(), dtype=torch.uint8)
            self.dist.all_gather_into_tensor(out, self.send.cpu())
            self.recv.copy_(out)

    def _barrier(self):  # stream-ordered under NCCL: a device-side barrier, no host round trip
        if not self.nccl:
            self.stream.synchronize()
        self.dist.all_reduce(self.token)

    def _enqueue(self):
        """The anneal's launch sequence (run_partitioned's order)."""
        ps = self.ps
        ps.init()  # writes the whole local copy: peers must not store into it before this
        if self.fused:
            self._barrier()
        sp, rp = self.send.data_ptr(), self.recv.data_ptr()
        for k in range(self.sweeps):
            ps.sweep(k, sp)
            self._exchange()
            ps.finish(k, rp)
            if self.fused and k + 1 < self.sweeps:
                self._barrier()

    def launch(self):
        """Enqueue one anneal on the stream (graph replay under NCCL)."""
        import torch

        with torch.cuda.stream(self.stream):
            if self.use_graph and self.graph is None:
                try:
                    self._enqueue()  # warm-up run: NCCL communicators and kernels initialised before capture
                    self.stream.synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=self.stream):
                        self._enqueue()
                    self.graph = g
                except RuntimeError as e:  # capture unsupported here: stay eager
                    self.use_graph, self.graph_error = False, str(e)
                    self.stream.synchronize()
            if self.graph is not None:
                self.graph.replay()
            else:
                self._enqueue()

    @property
    def launches_per_anneal(self) -> int:
        return 1 + 2 * self.sweeps  # init + (sweep, finish) per sweep; collectives not counted

    def result(self) -> dict:
        import torch

        res = [self.ps.fetch()]

        def all_reduce_sum(a):
            t = torch.as_tensor(a, device=self.cdev)
            self.dist.all_reduce(t)
            return t.cpu().numpy()

        return combine(res, all_reduce_sum)

    def run(self) -> dict:
        self.launch()
        return self.result()

    def close(self):
        if self.fused:
            # teardown order (gdi.h gdi_part_detach): close the peers' mappings on
            # every rank, barrier, and only then free the exported copies
            self.ps.detach()
            self.dist.barrier()
        self.graph = None
        self.ps = None


def anneal_partitioned(problem, params, seed: int, dist, device: int, stream=None, fused: bool = True,
                       graph: bool = True) -> dict:
    """One rank of a W-rank vertex-partitioned anneal (call on every rank;
    process group already initialised, one GPU per rank). fused: spin changes
    go straight into the other ranks' copies over peer memory (CUDA IPC
    handles exchanged once), and the per-sweep collective carries only the
    counter deltas; otherwise the owned chunks' spin words are all-gathered
    every sweep. graph: under NCCL, the anneal is one CUDA graph replay."""
    pa = PartitionedAnneal(problem, params, seed, dist, device, stream, fused, graph)
    try:
        return pa.run()
    finally:
        pa.close()


def emulate_partitioned(problem, params, seed: int, world: int, device: int = 0, fused: bool = False) -> dict:
    """All W ranks in this process on one device (see module docstring);
    fused: the ranks' sweep kernels store into each other's spin copies."""
    import torch

    import paper_1908_00210_b200 as pi

    dev = torch.device("cuda", device)
    stream = torch.cuda.current_stream(dev)
    ss = [pi.PartSession(problem, params, world, r, int(seed), stream=stream.cuda_stream, device=device)
          for r in range(world)]
    if fused and world > 1:
        for s_ in ss:
            s_.attach_local(ss)
    nb = ss[0].exchange_bytes
    sends = [torch.zeros(nb, dtype=torch.uint8, device=dev) for _ in range(world)]
    recv = torch.zeros(world * nb, dtype=torch.uint8, device=dev)

    def exchange():
        torch.cat(sends, out=recv)

    res = run_partitioned(ss, params.sweeps, exchange, lambda i: (sends[i].data_ptr(), recv.data_ptr()))
    out = combine(res)
    out["rank_spins_agree"] = all(np.array_equal(r["spins"], res[0]["spins"]) for r in res)
    return out
