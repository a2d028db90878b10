"""Where the e2e time goes: each C-ABI step of one fresh anneal_batch timed (ctypes)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1908_00210_b200 as pi
from bench import build_graph, CONFIGS

lib = ctypes.CDLL(pi.LIBGDI)
lib.gdi_last_error.restype = ctypes.c_char_p


class Params(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int32), ("strategy", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("flip_fraction0", ctypes.c_double), ("decay_rate", ctypes.c_double),
                ("a_num", ctypes.c_int64), ("b_num", ctypes.c_int64), ("denom", ctypes.c_int64)]


class Outputs(ctypes.Structure):
    _fields_ = [("spins", ctypes.c_void_p), ("trace", ctypes.c_void_p), ("scores", ctypes.c_void_p),
                ("snapshots", ctypes.c_void_p), ("counters", ctypes.c_void_p), ("seconds", ctypes.c_double)]


VP = ctypes.c_void_p  # pointer arguments must be declared (bare ints pass as 32-bit)
lib.gdi_graph_create.argtypes = [ctypes.c_int, ctypes.c_int32, VP, VP, VP, ctypes.POINTER(VP)]
lib.gdi_graph_destroy.argtypes = [VP]
lib.gdi_session_create.argtypes = [VP, ctypes.POINTER(Params), ctypes.c_int32, VP, ctypes.POINTER(VP)]
lib.gdi_session_set_seeds.argtypes = [VP, VP]
lib.gdi_session_launch.argtypes = [VP]
lib.gdi_session_sync.argtypes = [VP]
lib.gdi_session_fetch.argtypes = [VP, ctypes.POINTER(Outputs)]
lib.gdi_session_destroy.argtypes = [VP]


def ck(rc):
    if rc:
        raise RuntimeError(lib.gdi_last_error())


name = sys.argv[1] if len(sys.argv) > 1 else "G22"
mode = 1 if (len(sys.argv) > 2 and sys.argv[2] == "throughput") else 0
g = build_graph(pi, CONFIGS[name][0])
R, S = CONFIGS[name][1], CONFIGS[name][2]
off, nbr, _w = g.csr()
off = np.ascontiguousarray(off, np.int64)
nbr = np.ascontiguousarray(nbr, np.int32)
n = g.num_nodes
seeds = np.arange(1, R + 1, dtype=np.uint64)
spins = np.empty((R, n), np.int8)
scores = np.empty((R, 5), np.int64)
trace = np.empty((R, S, 6), np.float64)
for it in range(3):
    t = [time.perf_counter()]
    gr = ctypes.c_void_p()
    ck(lib.gdi_graph_create(0, n, off.ctypes.data, nbr.ctypes.data, None, ctypes.byref(gr)))
    t.append(time.perf_counter())
    p = Params(S, 1, mode, 1, 0.04, 0.99, 1, 4, 1)
    s = ctypes.c_void_p()
    ck(lib.gdi_session_create(gr, ctypes.byref(p), R, None, ctypes.byref(s)))
    t.append(time.perf_counter())
    ck(lib.gdi_session_set_seeds(s, seeds.ctypes.data))
    ck(lib.gdi_session_launch(s))
    ck(lib.gdi_session_sync(s))
    t.append(time.perf_counter())
    o = Outputs(spins.ctypes.data, None, scores.ctypes.data, None, None, 0.0)
    ck(lib.gdi_session_fetch(s, ctypes.byref(o)))
    t.append(time.perf_counter())
    o = Outputs(None, trace.ctypes.data, None, None, None, 0.0)
    ck(lib.gdi_session_fetch(s, ctypes.byref(o)))
    t.append(time.perf_counter())
    lib.gdi_session_destroy(s)
    lib.gdi_graph_destroy(gr)
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"{name} it{it}: graph_create {d[0]:.1f} ms | session_create {d[1]:.1f} | launch+sync {d[2]:.1f} "
          f"(kernel {o.seconds*1e3:.1f}) | fetch spins+scores {d[3]:.1f} | fetch trace {d[4]:.1f} | destroy {d[5]:.1f}")
