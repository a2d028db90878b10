"""Shared test helpers: golden vectors, hashing, recipe graphs (product side)."""
from __future__ import annotations

import functools
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
FNV_OFFSET = 1469598103934665603
FNV_PRIME = 1099511628211


def fnv_rows(rows: np.ndarray) -> list[int]:
    """FNV-1a 64 of each row's raw bytes (C helper in the test-only oracle lib)."""
    from oracle import oracle as o

    return o.fnv1a_rows(rows)


def fnv_bytes(data: bytes) -> int:
    return fnv_rows(np.frombuffer(data, np.uint8).reshape(1, -1))[0]


@functools.lru_cache(None)
def golden_configs() -> dict:
    with open(os.path.join(GOLDEN, "config_runs.json")) as f:
        return json.load(f)


@functools.lru_cache(None)
def small_cases() -> list:
    with open(os.path.join(GOLDEN, "small_cases.json")) as f:
        return json.load(f)


def product_graph(recipe: list[str]):
    """Build a recipe graph with the PRODUCT generators (pyising)."""
    import paper_1908_00210_b200 as pi

    kind, *a = recipe
    if kind == "random":
        return pi.random_graph(int(a[0]), int(a[1]), int(a[2]))
    if kind == "torus":
        return pi.torus_graph(int(a[0]), int(a[1]), int(a[2]))
    if kind == "torus_pm1":
        t = pi.torus_graph(int(a[0]), int(a[1]), int(a[2]))
        rng = pi.Rng(int(a[2]))
        edges = [(e.u, e.v, 1 if rng.coin() else -1) for e in t.edges()]
        return pi.Graph.from_edges(t.num_nodes, edges)
    raise ValueError(recipe)


def oracle_graph(recipe: list[str]):
    from oracle import oracle as o

    kind, *a = recipe
    return o.recipe(":".join([kind, *a]))
