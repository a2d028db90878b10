#!/usr/bin/env python3
"""gdi-b200 benchmark — spin-updates/s of the GDI annealing hot path.

Workload (BASELINE.json configs[1]): G22-shape random graph
random_graph(2000, 19990, 22), 1024 replicas per GPU (seeds 1 + rank*1024 ...),
1000 sweeps, A=1 B=4, pf0=0.04, decay 0.99, deterministic (exact, bit-for-bit
the reference's single-worker anneal per replica). One step = one full anneal
of all replicas (= R * n * M spin updates) in one kernel launch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config G22|G1|G55|G81pm1]
  python bench.py --impl reference ...   # reference CPU arm (oracle/_ref)

Multi-GPU (torchrun, one rank per GPU): replicas are independent, so each
rank anneals its own 1024 (weak scaling, no data-path collective); after the
timed region one tiny NCCL all-gather collects per-replica scores for the
best-cut selection (solve rule: lowest H, first seed wins ties).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    # name: (recipe, replicas per GPU, sweeps, mean degree for §8(d) bytes)
    "G1": (["random", "800", "19176", "1"], 1024, 1000),
    "G22": (["random", "2000", "19990", "22"], 1024, 1000),
    "G55": (["random", "5000", "12498", "55"], 1024, 1000),
    "G81pm1": (["torus_pm1", "100", "200", "81"], 1024, 1000),
    # BASELINE configs[4]: one replica of the 1M-vertex rudy graph, 20 sweeps
    # (the reference's CPU probe); run with --mode throughput
    "M1": (["random", "1000000", "4000000", "1000001"], 1, 20),
}
METRIC = "spin-updates/sec at 1/2/4/8 B200 and best balanced cut on G-set vs CPU ref"


def algorithmic_bytes_per_update(n: int, m: int, weighted: bool) -> float:
    """B_logical = 4 + 4*d + [weighted]*d + d + 2 (d = 2m/n)."""
    d = 2.0 * m / n
    return 4 + 4 * d + (d if weighted else 0) + d + 2


def build_graph(pi, recipe):
    kind, *a = recipe
    if kind == "random":
        return pi.random_graph(int(a[0]), int(a[1]), int(a[2]))
    if kind == "torus_pm1":
        t = pi.torus_graph(int(a[0]), int(a[1]), int(a[2]))
        rng = pi.Rng(int(a[2]))
        return pi.Graph.from_edges(t.num_nodes, [(e.u, e.v, 1 if rng.coin() else -1) for e in t.edges()])
    raise ValueError(recipe)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_traffic(config: str, kernel: str):
    """Per-launch traffic of the dominant kernel from the committed ncu
    --set full capture (profiles/roofline_traffic.json): DRAM bytes
    (dram__bytes_read.sum + dram__bytes_write.sum), L2 bytes (lts__t_bytes.sum)
    and shared-memory wavefronts, or None when no capture of this kernel is
    committed."""
    try:
        with open(os.path.join(REPO, "profiles", "roofline_traffic.json")) as f:
            doc = json.load(f)
    except OSError:
        return None
    return doc.get(f"{config}:{kernel}")


def roofline(bpu: float, updates: float, ms: float, l2: float, hbm: float, peaks_src: str,
             traffic, working_set: int, l2_size: int, note: str, smem_gbs: float = None):
    """SURVEY.md 8(d) accounting: achieved = updates/s x B_logical against the
    peak of the level that holds the working set (L2 when the CSR + spins fit
    in L2, HBM otherwise)."""
    achieved = bpu * updates / (ms * 1e-3) / 1e9
    in_l2 = working_set <= l2_size
    peak = l2 if in_l2 else hbm
    rec = {"bound": "l2" if in_l2 else "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
           "frac": achieved / peak,
           "traffic": None, "bytes_per_update": bpu, "working_set_bytes": working_set,
           "l2_bytes": l2_size,
           "peak_source": ("live L2 read probe (probe.cu: 16-byte __ldcg loads of a 48 MB L2-resident "
                           "buffer, 4 CTAs/SM x 512 threads, 50 passes; profiles/r02_l2_peak.json)") if in_l2
                          else peaks_src,
           "hbm_peak_gbs": hbm, "frac_of_hbm": achieved / hbm, "l2_peak_gbs": l2, "note": note}
    if smem_gbs:
        # the exact / pooled kernels stage the CSR and the replica state in
        # shared memory, so the logical bytes are served from there: a dense
        # graph (G1, degree 48) can exceed the L2 figure (frac > 1)
        rec["smem_peak_gbs"] = smem_gbs
        rec["frac_of_smem"] = achieved / smem_gbs
        rec["smem_peak_source"] = "148 SMs x 128 B/cycle x the sampled SM clock (nominal shared-memory bandwidth)"
    if traffic:
        units = traffic.get("updates_per_launch")
        lps = traffic.get("launches_per_step", 1)
        # per step, like `achieved` (M1: one k4_sweep launch per sweep)
        rec["traffic"] = traffic["dram_bytes_per_launch"] * lps if traffic.get("dram_bytes_per_launch") else None
        if traffic.get("lts_bytes_per_launch"):
            rec["l2_traffic"] = traffic["lts_bytes_per_launch"] * lps
        rec["traffic_source"] = traffic.get("source")
        if units:
            rec["measured_per_update"] = {
                k: traffic[k] / units for k in ("dram_bytes_per_launch", "lts_bytes_per_launch",
                                                "smem_wavefronts_per_launch") if traffic.get(k) is not None}
    return rec


def l2_probe_gbs(pi) -> float:
    """Measured L2-resident read bandwidth (library probe, 48 MB buffer)."""
    return pi.probe_l2_bandwidth(48 << 20, 50)


def ref_tool_path():
    p = os.path.join(REPO, "oracle", "_ref", "ref_tool")
    return p if os.path.exists(p) else None


def cpu_reference_bench(recipe, sweeps, replicas, threads, seed0=1):
    tool = ref_tool_path()
    if tool is None:
        return None
    out = subprocess.run([tool, "bench", *recipe, "--replicas", str(replicas), "--threads", str(threads),
                          "--sweeps", str(sweeps), "--seeds", str(seed0), str(seed0)],
                         check=True, capture_output=True, text=True).stdout
    return json.loads(out)


def cpu_port_bench(recipe, sweeps, replicas, seed0=1):
    """Fallback CPU baseline: the C restatement, single core (kind 'port')."""
    from oracle import oracle as o

    g = o.recipe(":".join(recipe))
    t0 = time.perf_counter()
    for r in range(replicas):
        o.anneal(g, seed0 + r, sweeps)
    s = time.perf_counter() - t0
    return {"seconds": s, "updates_per_s": replicas * g.n * sweeps / s, "threads": 1, "replicas": replicas}


def host_cpu():
    return {"cpu_model": cpu_model(), "nproc": os.cpu_count()}


def cpu_baseline(recipe, n, sweeps):
    threads = os.cpu_count() or 1
    # bounded sample: ~20 CPU-seconds of reference work (one G22 replica is
    # ~0.35 s on one core), rounded to whole waves of the thread pool
    per_rep = 0.35 * (n * sweeps) / 2.0e6
    reps = max(threads, int(round(20.0 / max(per_rep, 1e-3) / threads)) * threads)
    res = cpu_reference_bench(recipe, sweeps, reps, threads)
    if res is not None:
        return {"value": res["updates_per_s"], "unit": "spin-updates/s", "cores": res["threads"],
                "kind": "reference", **host_cpu(),
                "sample": f"{reps} deterministic single-worker anneals ({sweeps} sweeps) on a "
                          f"{res['threads']}-thread pool, oracle/_ref/ref_tool (bench.cpp:158-175 scheduling)"}
    reps = 2
    res = cpu_port_bench(recipe, sweeps, reps)
    return {"value": res["updates_per_s"], "unit": "spin-updates/s", "cores": 1, "kind": "port", **host_cpu(),
            "sample": f"{reps} anneals ({sweeps} sweeps) with the C restatement, 1 core"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    recipe, _, sweeps = CONFIGS[args.config]
    n = int(recipe[1]) if recipe[0] == "random" else int(recipe[1]) * int(recipe[2])
    threads = os.cpu_count() or 1
    per_rep = 0.35 * (n * sweeps) / 2.0e6
    reps = max(threads, int(round(15.0 / max(per_rep, 1e-3) / threads)) * threads)
    vals, times = [], []
    kind = "reference" if ref_tool_path() else "port"
    for i in range(args.warmup + args.steps):
        if kind == "reference":
            res = cpu_reference_bench(recipe, sweeps, reps, threads, seed0=1 + i * reps)
        else:
            res = cpu_port_bench(recipe, sweeps, 1, seed0=1 + i)
        if i >= args.warmup:
            vals.append(res["updates_per_s"])
            times.append(res["seconds"])
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "spin-updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int8/int64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {' '.join(recipe)}, deterministic replicas, {sweeps} sweeps",
                   "replicas_per_step": reps if kind == "reference" else 1},
        "cpu_baseline": {"value": value, "unit": "spin-updates/s", "cores": threads if kind == "reference" else 1,
                         "kind": kind, **host_cpu(), "sample": f"{reps if kind == 'reference' else 1} replicas per step"},
        "e2e": {"value": value, "unit": "spin-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def topology_only(args):
    """Process-group plumbing of the multi-rank bench without any GPU work:
    every rank joins (BENCH_DIST_BACKEND, default nccl), rank 0 prints the
    world it saw (tests/test_bench_launch.py runs this with gloo on CPU)."""
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if world > 1:
        dist.init_process_group(backend)
        import torch

        t = torch.tensor([rank], dtype=torch.int64)
        dist.all_reduce(t)
        ranks_sum = int(t.item())
        dist.destroy_process_group()
    else:
        ranks_sum = 0
    if rank == 0:
        print(json.dumps({"n_gpus": world, "ranks_sum": ranks_sum, "requested": args.gpus,
                          "backend": backend if world > 1 else None}), flush=True)
    return 0


def run_partition_bench(args, pi, torch, dist, world, rank, local, dev, recipe, g, prob, params):
    """BASELINE configs[4] on N GPUs: ONE replica of the 1M-vertex graph,
    vertex-partitioned (sharding.PartitionedAnneal: K4 chains per rank; spin
    changes stored into the peers' copies during the sweep, the counter deltas
    all-gathered per sweep). Strong scaling: the total work is fixed. The
    session, peer mappings and buffers are set up once, outside the timed
    region; a step = one full anneal (init + all sweeps), replayed as one CUDA
    graph under NCCL."""
    from paper_1908_00210_b200 import sharding as sh

    n, m, sweeps = g.num_nodes, g.num_edges, params.sweeps
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    pa = sh.PartitionedAnneal(prob, params, 1, dist, local, stream)

    def step():
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pa.launch()
        e1.record(stream)
        return e0, e1

    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        dist.barrier()
        runs = [step() for _ in range(args.steps)]
        torch.cuda.synchronize(dev)
    ms = sum(a.elapsed_time(b) for a, b in runs) / len(runs)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out = pa.result()
    graphed = pa.graph is not None
    pa.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": n * sweeps / (float(t.item()) * 1e-3), "unit": "spin-updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(t.item()),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int8 spins / int64 energies", "data": "synthetic",
            "config": {"workload": f"M1: {' '.join(recipe)}, one replica vertex-partitioned over {world} GPUs, "
                                   f"{sweeps} sweeps, pooled throughput mode",
                       "n": n, "m": m, "replicas": 1, "sweeps": sweeps,
                       "parallelism": f"vertex partition x{world}: chunks c = rank (mod {world}); changed chunk "
                                      "spin words stored into the other ranks' copies over peer memory during the "
                                      "sweep (CUDA IPC), per sweep a 16-byte counter all-gather + a barrier all-reduce",
                       "cuda_graph": graphed,
                       "l2": "flushed between steps (256 MB write)", "kernel": "k4_sweep + k4_finish (partitioned)"},
            "clocks": clocks.summary(),
            "gpu_launches": args.steps * pa.launches_per_anneal,
            "result": {"cut": out["cut"], "imbalance": out["imbalance"]},
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def eval_leg(pi, torch, prob, g, spins, stream, flush, dev, hbm, hbm_src, reps=20):
    """K3 (k3_eval.cu, north_star (4)): the fused exact cut + spin sum of the
    step's final spins, device-resident, timed alone with CUDA events (L2
    flushed before every call); plus the same spins tiled to 16x the batch,
    where the int8 spin stream dominates. Roofline: algorithmic bytes = the
    int8 spins (R * n) + the canonical edge list (4 B per edge up to 65536
    vertices, else 8 B; +4 B weights if general) per call, against HBM."""
    ev = pi.Evaluator(prob, dev.index or 0)
    n, m = g.num_nodes, g.num_edges
    eb = (4 if n <= 65536 else 8) + (4 if not g.all_unit_weights and not _pm1(g) else 0)
    out = {}
    for label, tile in (("batch", 1), ("batch_x16", 16)):
        sp = np.ascontiguousarray(np.tile(spins, (tile, 1)))
        R = sp.shape[0]
        d = torch.from_numpy(sp).to(dev)
        res = torch.zeros((R, 2), dtype=torch.int64, device=dev)
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        ts = []
        for i in range(reps + 3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ev.evaluate_device(d.data_ptr(), R, res.data_ptr(), bad.data_ptr(), stream.cuda_stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
        ref = ev.evaluate(sp[:1])  # host path on the first row (its own upload) as a spot check
        got = res.cpu().numpy()
        ms = statistics.median(ts)
        algo = R * n + m * eb
        out[label] = {
            "replicas": R, "ms": ms, "evals_per_s": R / (ms * 1e-3), "edge_checks_per_s": R * m / (ms * 1e-3),
            "kernel": "k3_slice + k3_sliced" if (R >= 16 and n * 4 <= 200 * 1024 and (g.all_unit_weights or _pm1(g)))
                      else "k3_pack + k3_bits",
            "launches": 4, "note": "timed region = 2 memsets + 2 kernels of gdi_evaluate_device",
            "roofline": {"bound": "hbm", "achieved": algo / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": algo / (ms * 1e-3) / 1e9 / hbm, "algorithmic_bytes": algo, "peak_source": hbm_src},
            "check": bool(int(got[0, 0]) == int(ref["cut"][0]) and abs(int(got[0, 1])) == int(ref["imbalance"][0])
                          and int(bad.item()) == 0)}
    return out


def _pm1(g) -> bool:
    return not g.all_unit_weights and all(abs(w) == 1 for _, _, w in _edge_weights(g))


def _edge_weights(g):
    for u in range(g.num_nodes):
        for v, w in g.neighbors(u):
            yield u, v, w


def free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(nproc: int) -> int:
    """`bench.py --gpus N` without a launcher: re-run this command under
    torch.distributed.run, one rank per GPU on this node (rendezvous on
    127.0.0.1), and return its exit code. Rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    # NCCL's init lines on stderr (one per rank: the ranks can be counted from
    # the log); the JSON line stays alone on stdout
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.TimeoutExpired):
        pass
    return "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="G22", choices=sorted(CONFIGS))
    ap.add_argument("--replicas", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-throughput", action="store_true")
    ap.add_argument("--no-eval", action="store_true", help="skip the K3 evaluation leg")
    ap.add_argument("--mode", default="exact", choices=["exact", "throughput"],
                    help="headline mode: exact (bit-exact, default) or throughput (pooled racy mode)")
    ap.add_argument("--topology-only", action="store_true",
                    help="initialise the ranks, print the rank/world line and exit (launcher test)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # the driver runs `bench.py --gpus N` directly: launch N ranks here
        return spawn_ranks(args.gpus)
    if args.topology_only:
        return topology_only(args)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_1908_00210_b200 as pi
    from paper_1908_00210_b200 import sharding as sh

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # NCCL, one GPU per rank (the driver's scaling runs). BENCH_DIST_BACKEND=gloo
    # lets several ranks share fewer GPUs to rehearse the multi-rank plumbing
    # (replica sharding has no kernels that wait across ranks; the numbers of
    # such a run are not measurements).
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = dev if backend == "nccl" else torch.device("cpu")  # where collective tensors live
    pi.set_device(local)

    recipe, R, sweeps = CONFIGS[args.config]
    R = args.replicas or R
    g = build_graph(pi, recipe)
    n, m = g.num_nodes, g.num_edges
    prob = pi.MinCutProblem.with_default_coefficients(g)
    params = pi.AnnealParams()
    if args.mode == "exact":
        params.sweeps, params.deterministic = sweeps, True
    else:
        params.sweeps, params.workers = sweeps, 8
        args.no_throughput = True  # the headline already is the throughput mode
    seeds = sh.replica_seeds(rank, world, R)
    if args.config == "M1" and args.mode == "throughput" and world > 1:
        return run_partition_bench(args, pi, torch, dist, world, rank, local, dev, recipe, g, prob, params)

    # a real (non-legacy) stream: the session launches on it and the torch
    # events below are recorded on the same stream
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sess = pi.Session(prob, params, R, stream=stream.cuda_stream, trace=True, device=local)
    sess.set_seeds(seeds)
    # L2 flush buffer (> 126 MB L2) rewritten between timed steps
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step_on(session):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        session.launch()
        e1.record(stream)
        return e0, e1

    def one_step():
        return step_on(sess)

    # nvidia-smi samples every 100 ms and needs ~0.3 s to start: the sampler
    # runs from the warm-up on, and short steps (1M config: ~2 ms) keep the
    # GPU busy with extra untimed warm-up steps until it has samples, so the
    # clocks below are those of the loaded GPU around the timed region
    with ClockSampler(local) as clocks:
        tw0 = time.perf_counter()
        nw = 0
        while nw < args.warmup or (time.perf_counter() - tw0 < 1.0 and len(clocks.rows) < 3):
            one_step()
            torch.cuda.synchronize(dev)
            nw += 1
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t_wall0 = time.perf_counter()
        evs = [one_step() for _ in range(args.steps)]
        torch.cuda.synchronize(dev)
        t_wall = time.perf_counter() - t_wall0
    if world > 1:
        dist.barrier()
    kernel_ms = [a.elapsed_time(b) for a, b in evs]
    step_ms = sum(kernel_ms) / len(kernel_ms)
    t_local = torch.tensor([step_ms], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    step_ms_max = float(t_local.item())
    updates_per_step = world * R * n * sweeps
    value = updates_per_step / (step_ms_max * 1e-3)

    # results of the last step: best balanced cut across all replicas of all ranks
    res = sess.fetch(spins=False, trace=False)
    sc = sh.gather_scores(sh.score_rows(res, seeds), dist if world > 1 else None, device=cdev)
    summ = sh.summarize(sc, n % 2)
    best = {k: summ[k] for k in ("cut", "imbalance", "seed", "best_balanced_cut")}

    line = None
    if rank == 0:
        weighted = not g.all_unit_weights
        bpu = algorithmic_bytes_per_update(n, m, weighted)
        peaks = {}
        try:
            with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
        except OSError:
            pass
        hbm = peaks.get("hbm_gbs", 6650.0)
        hbm_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
        l2 = l2_probe_gbs(pi)
        l2_size = torch.cuda.get_device_properties(dev).L2_cache_size
        ws = (n + 1) * 4 + 2 * m * 4 + (2 * m if weighted else 0) + R * n  # compact CSR + int8 spins
        clk = clocks.summary()
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        smem_gbs = sms * 128 * clk["sm_mhz"] * 1e6 / 1e9 if clk.get("sm_mhz") else None
        onchip = not sess.kernel.startswith(("k4_", "k1_window")) and ",rows" not in sess.kernel  # CSR in smem
        rl = roofline(bpu, R * n * sweeps, step_ms, l2, hbm, hbm_src, measured_traffic(args.config, sess.kernel),
                      ws, l2_size,
                      ("exact mode: each replica is one serial decision chain (SURVEY 8(d): K1 is latency-bound, "
                       "see cycles_per_visit); " if args.mode == "exact" else "") +
                      "logical bytes per SURVEY 8(d); the CSR and spins are smem/L2 resident",
                      smem_gbs if onchip else None)
        if args.mode == "exact" and clk.get("sm_mhz"):
            # SM cycles per visit of one replica chain (all chains run concurrently)
            rl["cycles_per_visit"] = step_ms * 1e-3 * clk["sm_mhz"] * 1e6 / (n * sweeps)
        line = {
            "metric": METRIC, "value": value, "unit": "spin-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int8 spins / int64 energies", "data": "synthetic",
            "config": {"workload": f"{args.config}: random_graph/torus recipe {' '.join(recipe)}, "
                                   f"{R} replicas per GPU, {sweeps} sweeps, "
                                   + ("deterministic exact mode" if args.mode == "exact" else "pooled throughput mode"),
                       "n": n, "m": m, "replicas_per_gpu": R, "sweeps": sweeps,
                       "mode": "exact (bit-identical to reference single-worker anneal)" if args.mode == "exact"
                               else "throughput (reference pooled racy mode, statistically equivalent)",
                       "parallelism": f"replicas x{world} (weak)", "l2": "flushed between steps (256 MB write)",
                       "kernel": sess.kernel},
            "roofline": rl,
            "clocks": clk,
            "gpu_launches": args.steps * sess.launch_count,
            "wall_s_timed": t_wall,
            "result": best,
        }
    sess.sync()
    if rank == 0 and not args.no_eval:
        fin = sess.fetch(spins=True, trace=False)
        line["evaluation"] = eval_leg(pi, torch, prob, g, fin["spins"], stream, flush, dev, hbm, hbm_src)
    del sess

    # Throughput mode (K2, the reference's pooled racy mode) on the same
    # workload and seeds: reported beside the exact-mode headline.
    if not args.no_throughput:
        tparams = pi.AnnealParams()
        tparams.sweeps, tparams.workers = sweeps, 8
        tsess = pi.Session(prob, tparams, R, stream=stream.cuda_stream, trace=True, device=local)
        tsess.set_seeds(seeds)
        for _ in range(args.warmup):
            step_on(tsess)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        tev = [step_on(tsess) for _ in range(args.steps)]
        torch.cuda.synchronize(dev)
        t_ms = sum(a.elapsed_time(b) for a, b in tev) / len(tev)
        tt = torch.tensor([t_ms], dtype=torch.float64, device=cdev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tsess.sync()
        tres = tsess.fetch(spins=False, trace=False)
        if rank == 0:
            tbal = tres["imbalance"] <= n % 2
            line["throughput_mode"] = {
                "value": updates_per_step / (float(tt.item()) * 1e-3), "unit": "spin-updates/s",
                "ms_per_step": float(tt.item()), "kernel": tsess.kernel,
                "mode": "racy pooled mode (reference workers>1), Philox4x32-10, statistically equivalent",
                "best_balanced_cut": int(tres["cut"][tbal].min()) if tbal.any() else None,
                "mean_cut": float(tres["cut"].mean()), "frac_balanced": float(tbal.mean()),
                "gpu_launches": args.steps * tsess.launch_count,
                "roofline": roofline(bpu, R * n * sweeps, t_ms, l2, hbm, hbm_src,
                                     measured_traffic(args.config, tsess.kernel), ws, l2_size,
                                     "logical bytes per SURVEY 8(d); the CSR and spins are smem/L2 resident",
                                     smem_gbs if not tsess.kernel.startswith(("k4_", "k1_window"))
                                     and ",rows" not in tsess.kernel else None)}
        del tsess

    # e2e: the public batched call with host buffers (fresh CSR upload, seeds
    # H2D, full spins + trace + scores D2H) every step
    if not args.no_e2e:
        if world > 1:
            dist.barrier()
        e2e_times = []
        for i in range(2 + max(1, args.steps // 2)):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            pi.anneal_batch_fresh(prob, params, seeds, True)
            torch.cuda.synchronize(dev)
            if i >= 2:
                e2e_times.append(time.perf_counter() - t0)
        t_e2e = torch.tensor([statistics.median(e2e_times)], dtype=torch.float64, device=cdev)
        if world > 1:
            dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
        if rank == 0:
            h2d = (n + 1) * 4 + 2 * m * 4 + (0 if g.all_unit_weights else 2 * m * 4) + R * 8 + sweeps * 8
            d2h = R * n + R * sweeps * (24 + 8) + R * 8 + R * 24
            line["e2e"] = {"value": updates_per_step / float(t_e2e.item()), "unit": "spin-updates/s",
                           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                           "seconds_per_step": float(t_e2e.item()),
                           "path": "pyising.anneal_batch_fresh -> gdi_graph_create + gdi_anneal_batch (C ABI)"}
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(recipe, n, sweeps)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
