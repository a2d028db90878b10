"""gdi-b200 — GDI Ising annealing (arXiv 1908.00210) for balanced min-cut on B200.

The compute path is native: `pyising` (pybind11) -> libising.so (C++ solver
API, source-compatible with the reference headers) -> libgdi.so (C ABI in
include/gdi.h) -> sm_100a kernels. Importing this package fails loudly when
the extension has not been built (`make`); there is no Python or CPU fallback.
"""
from __future__ import annotations

import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIBDIR = os.path.join(_HERE, "lib")
LIBGDI = os.path.join(LIBDIR, "libgdi.so")
LIBISING = os.path.join(LIBDIR, "libising.so")

try:
    from . import pyising  # noqa: F401
except ImportError as exc:  # pragma: no cover - exercised only on a broken build
    raise ImportError(
        "paper_1908_00210_b200: native extension not built; run `make` at the repo root "
        f"(or __graft_entry__.build()). Original error: {exc}"
    ) from exc

from .pyising import *  # noqa: F401,F403,E402

__all__ = [name for name in dir(pyising) if not name.startswith("_")]
