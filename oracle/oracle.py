"""TEST INFRASTRUCTURE — ctypes front-end of the C restatement (gdi_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module, and only as the checker. The product library never loads it.
Parity of the restatement itself is pinned by tests/test_oracle_golden.py
against vectors produced by the unmodified reference (oracle/_ref).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

I8P = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
I64P = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
U64P = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
F64P = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            import subprocess

            subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)
        L = ctypes.CDLL(path)
        c = ctypes
        L.orc_rng_draws.argtypes = [c.c_uint64, c.c_uint64, c.c_int64, U64P]
        L.orc_rng_draws.restype = None
        for name in ("orc_gen_random",):
            getattr(L, name).argtypes = [c.c_int32, c.c_int64, c.c_uint64, I32P, I32P, I32P]
            getattr(L, name).restype = c.c_int
        for name in ("orc_gen_torus", "orc_gen_torus_pm1"):
            getattr(L, name).argtypes = [c.c_int32, c.c_int32, c.c_uint64, I32P, I32P, I32P]
            getattr(L, name).restype = c.c_int
        L.orc_csr_from_edges.argtypes = [c.c_int32, c.c_int64, I32P, I32P, I32P, I64P, I32P, I32P]
        L.orc_csr_from_edges.restype = c.c_int32
        L.orc_canonical_edges.argtypes = [c.c_int32, I64P, I32P, I32P, I32P, I32P, I32P]
        L.orc_canonical_edges.restype = c.c_int64
        L.orc_cut.argtypes = [c.c_int32, I64P, I32P, I32P, I8P]
        L.orc_cut.restype = c.c_int64
        L.orc_anneal_det.argtypes = [
            c.c_int32, I64P, I32P, I32P, c.c_int64, c.c_int64, c.c_int64, c.c_int32,
            c.c_double, c.c_double, c.c_uint64, I8P, I64P, I64P, F64P, I64P,
        ]
        L.orc_anneal_det.restype = c.c_int
        U8P = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
        L.orc_fnv1a_rows.argtypes = [U8P, c.c_int64, c.c_int64, U64P]
        L.orc_fnv1a_rows.restype = None
        _LIB = L
    return _LIB


def fnv1a_rows(rows: np.ndarray) -> list[int]:
    """FNV-1a 64 of each row's raw bytes."""
    b = np.ascontiguousarray(rows).view(np.uint8).reshape(rows.shape[0], -1)
    out = np.empty(b.shape[0], np.uint64)
    lib().orc_fnv1a_rows(b, b.shape[0], b.shape[1], out)
    return [int(x) for x in out]


def fnv1a(data: bytes) -> int:
    return fnv1a_rows(np.frombuffer(data, np.uint8).reshape(1, -1))[0]


def draws(seed: int, stream: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().orc_rng_draws(seed, stream, count, out)
    return out


@dataclass
class Csr:
    n: int
    offsets: np.ndarray  # int64[n+1]
    nbr: np.ndarray  # int32[2m]
    w: np.ndarray  # int32[2m]
    max_degree: int

    @property
    def m(self) -> int:
        return int(self.offsets[-1]) // 2

    def canonical_edges(self):
        m = self.m
        eu = np.empty(m, np.int32)
        ev = np.empty(m, np.int32)
        ew = np.empty(m, np.int32)
        lib().orc_canonical_edges(self.n, self.offsets, self.nbr, self.w, eu, ev, ew)
        return eu, ev, ew

    def to_gset(self) -> str:
        eu, ev, ew = self.canonical_edges()
        lines = [f"{self.n} {self.m}"]
        lines += [f"{u + 1} {v + 1} {w}" for u, v, w in zip(eu.tolist(), ev.tolist(), ew.tolist())]
        return "\n".join(lines) + "\n"


def csr_from_edges(n: int, eu, ev, ew=None) -> Csr:
    eu = np.ascontiguousarray(eu, np.int32)
    ev = np.ascontiguousarray(ev, np.int32)
    ew = np.ones_like(eu) if ew is None else np.ascontiguousarray(ew, np.int32)
    m = len(eu)
    off = np.empty(n + 1, np.int64)
    nbr = np.empty(max(2 * m, 1), np.int32)
    w = np.empty(max(2 * m, 1), np.int32)
    rc = lib().orc_csr_from_edges(n, m, eu, ev, ew, off, nbr, w)
    if rc < 0:
        raise ValueError(f"orc_csr_from_edges failed ({rc})")
    return Csr(n, off, nbr[: 2 * m], w[: 2 * m], int(rc))


def random_graph(n: int, m: int, seed: int) -> Csr:
    eu, ev, ew = (np.empty(m, np.int32) for _ in range(3))
    if lib().orc_gen_random(n, m, seed, eu, ev, ew):
        raise ValueError("bad random_graph args")
    return csr_from_edges(n, eu, ev, ew)


def torus_graph(rows: int, cols: int, seed: int, pm1: bool = False) -> Csr:
    m = 2 * rows * cols
    eu, ev, ew = (np.empty(m, np.int32) for _ in range(3))
    fn = lib().orc_gen_torus_pm1 if pm1 else lib().orc_gen_torus
    if fn(rows, cols, seed, eu, ev, ew):
        raise ValueError("bad torus args")
    return csr_from_edges(rows * cols, eu, ev, ew)


def recipe(spec: str) -> Csr:
    """'random:N:M:SEED' | 'torus:R:C:SEED' | 'torus_pm1:R:C:SEED'."""
    kind, *a = spec.split(":")
    a = [int(x) for x in a]
    if kind == "random":
        return random_graph(*a)
    if kind == "torus":
        return torus_graph(*a)
    if kind == "torus_pm1":
        return torus_graph(*a, pm1=True)
    raise ValueError(spec)


def cut(g: Csr, spins) -> int:
    return int(lib().orc_cut(g.n, g.offsets, g.nbr, g.w, np.ascontiguousarray(spins, np.int8)))


def anneal(g: Csr, seed: int, sweeps: int = 1000, pf0: float = 0.04, decay: float = 0.99,
           a: int = 1, b: int = 4, denom: int = 1) -> dict:
    spins = np.empty(g.n, np.int8)
    trace = np.empty((sweeps, 3), np.int64)
    counter = np.empty(sweeps, np.int64)
    pf = np.empty(sweeps, np.float64)
    stats = np.empty(2, np.int64)
    rc = lib().orc_anneal_det(g.n, g.offsets, g.nbr, g.w, a, b, denom, sweeps, pf0, decay, seed,
                              spins, trace, counter, pf, stats)
    if rc:
        raise ValueError("bad anneal params")
    return {"spins": spins, "trace": trace, "counter": counter, "pf": pf,
            "ties": int(stats[0]), "draws": int(stats[1])}
