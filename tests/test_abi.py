"""The C-ABI boundary (include/gdi.h) on CPU: the library loads, exports every
declared entry point, validates inputs before touching a device, and fails
loudly (GDI_ERR_RUNTIME) when no device is present. No compute calls."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1908_00210_b200 as pkg

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "gdi.h")

GDI_ERR_CONFIG, GDI_ERR_DOMAIN, GDI_ERR_RUNTIME = -1, -2, -4


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(gdi_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    L = ctypes.CDLL(pkg.LIBGDI)
    L.gdi_last_error.restype = ctypes.c_char_p
    # pointers must be declared: ctypes passes bare Python ints as 32-bit ints
    VP = ctypes.c_void_p
    L.gdi_graph_create.argtypes = [ctypes.c_int, ctypes.c_int32, VP, VP, VP, ctypes.POINTER(VP)]
    return L


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert missing == []


def test_libising_links_libgdi_and_no_cpu_annealer():
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", pkg.LIBISING], capture_output=True, text=True).stdout
    assert "anneal" in out
    deps = subprocess.run(["ldd", pkg.LIBISING], capture_output=True, text=True).stdout
    assert "libgdi.so" in deps


def test_abi_version(lib):
    assert lib.gdi_abi_version() == 1


def test_graph_create_validates_before_device(lib):
    out = ctypes.c_void_p()
    off = np.array([0, 1, 2], dtype=np.int64)
    self_loop = np.array([0, 1], dtype=np.int32)
    rc = lib.gdi_graph_create(0, 2, off.ctypes.data, self_loop.ctypes.data, None, ctypes.byref(out))
    assert rc == GDI_ERR_DOMAIN and b"self-loop" in lib.gdi_last_error()
    bad_range = np.array([5, 0], dtype=np.int32)
    rc = lib.gdi_graph_create(0, 2, off.ctypes.data, bad_range.ctypes.data, None, ctypes.byref(out))
    assert rc == GDI_ERR_DOMAIN
    rc = lib.gdi_graph_create(0, 0, off.ctypes.data, bad_range.ctypes.data, None, ctypes.byref(out))
    assert rc == GDI_ERR_DOMAIN
    rc = lib.gdi_graph_create(0, 2, off.ctypes.data, self_loop.ctypes.data, None, None)
    assert rc == GDI_ERR_CONFIG


def test_no_device_is_a_runtime_error(lib):
    count = ctypes.c_int(-1)
    lib.gdi_device_count(ctypes.byref(count))
    if count.value > 0:
        pytest.skip("a GPU is visible")
    out = ctypes.c_void_p()
    off = np.array([0, 1, 2], dtype=np.int64)
    nbr = np.array([1, 0], dtype=np.int32)
    rc = lib.gdi_graph_create(0, 2, off.ctypes.data, nbr.ctypes.data, None, ctypes.byref(out))
    assert rc == GDI_ERR_RUNTIME and b"no CUDA device" in lib.gdi_last_error()


def test_session_rejects_null_graph(lib):
    class Params(ctypes.Structure):
        _fields_ = [("sweeps", ctypes.c_int32), ("strategy", ctypes.c_int32), ("mode", ctypes.c_int32),
                    ("flags", ctypes.c_uint32), ("flip_fraction0", ctypes.c_double), ("decay_rate", ctypes.c_double),
                    ("a_num", ctypes.c_int64), ("b_num", ctypes.c_int64), ("denom", ctypes.c_int64)]

    p = Params(10, 1, 0, 0, 0.04, 0.99, 1, 4, 1)
    out = ctypes.c_void_p()
    assert lib.gdi_session_create(None, ctypes.byref(p), 4, None, ctypes.byref(out)) == GDI_ERR_CONFIG
