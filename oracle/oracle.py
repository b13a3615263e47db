"""ctypes binding of oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

May be imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg.  Shares no code with the CUDA path.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")

OK, INFEASIBLE, INVALID_ARG = 0, 1, -1

# orc_window -- declared independently of the library's coop_window
ORC_WINDOW = np.dtype([("first", "<i4"), ("last", "<i4"), ("span", "<u8"), ("cost", "<f8"),
                       ("n_evict", "<i4"), ("status", "<i4")])

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            here = os.path.dirname(_HERE)
            import sys
            sys.path.insert(0, here)
            from paper_2311_00591_b200 import _build  # builds only; does not load libcoop
            _build.build_oracle()
        L = ctypes.CDLL(LIB_PATH)
        L.orc_window_search.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
        L.orc_window_search.restype = ctypes.c_int
        L.orc_window_search_many.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int64,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p]
        L.orc_window_search_many.restype = ctypes.c_int
        L.orc_fsum.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        L.orc_fsum.restype = ctypes.c_double
        _lib = L
    return _lib


def search(size_state, cost, stale, request: int) -> np.void:
    """O1 on one pool -> orc_window record"""
    ss = np.ascontiguousarray(size_state, np.uint64)
    c = np.ascontiguousarray(cost, np.float64)
    s = np.ascontiguousarray(stale, np.float64)
    out = np.zeros(1, ORC_WINDOW)
    lib().orc_window_search(len(ss), ss.ctypes.data, c.ctypes.data, s.ctypes.data,
                            int(request), out.ctypes.data)
    return out[0]


def search_many(size_state, cost, stale, requests, n_pools: int, n: int, stride: int) -> np.ndarray:
    ss = np.ascontiguousarray(size_state, np.uint64)
    c = np.ascontiguousarray(cost, np.float64)
    s = np.ascontiguousarray(stale, np.float64)
    r = np.ascontiguousarray(requests, np.uint64)
    out = np.zeros(n_pools, ORC_WINDOW)
    lib().orc_window_search_many(n_pools, n, stride, ss.ctypes.data, c.ctypes.data,
                                 s.ctypes.data, r.ctypes.data, out.ctypes.data)
    return out


def fsum(x) -> float:
    x = np.ascontiguousarray(x, np.float64)
    return float(lib().orc_fsum(x.ctypes.data, x.size))
