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
            from oracle import build as _ob  # the oracle's own gcc build (no product code)
            _ob.build_oracle()
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


# ----------------------------------------------------------------------------- O2 replay
class _OrcTrace(ctypes.Structure):
    _fields_ = [("n_tensors", ctypes.c_int32), ("n_ops", ctypes.c_int32),
                ("size", ctypes.c_void_p), ("is_param", ctypes.c_void_p),
                ("producer", ctypes.c_void_p), ("cost_us", ctypes.c_void_p),
                ("out", ctypes.c_void_p), ("inplace_src", ctypes.c_void_p),
                ("phase", ctypes.c_void_p), ("in_ptr", ctypes.c_void_p),
                ("in_idx", ctypes.c_void_p)]


class _OrcCfg(ctypes.Structure):
    _fields_ = [("budget", ctypes.c_uint64), ("flags", ctypes.c_uint32),
                ("class_threshold", ctypes.c_uint32), ("max_depth", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


F_PARTITION, F_INPLACE, F_PARTITION_ALL_PHASES, F_DTR, F_DTE = 1, 2, 4, 8, 16
UNSATISFIABLE, THRASHED = -3, -4
EV_PARAM, EV_ALLOC, EV_INPLACE, EV_EVICT, EV_FREE, EV_REMAT, EV_EXEC, EV_REXEC = range(8)

ORC_RESULT = np.dtype([("status", "<i4"), ("fail_op", "<i4"), ("base_us", "<i8"),
                       ("total_us", "<i8"), ("evictions", "<i8"), ("remat", "<i8"),
                       ("pressure", "<i8"), ("frag_fail", "<i8"), ("inplace_reuse", "<i8"),
                       ("heuristic_evals", "<i8"), ("sum_free_bytes_after", "<u8"),
                       ("sum_free_blocks_after", "<i8"), ("digest", "<u8"),
                       ("max_depth", "<i4"), ("max_blocks", "<i4"), ("budget", "<u8"),
                       ("n_events", "<i8")])
ORC_EVENT = np.dtype([("kind", "<i4"), ("op", "<i4"), ("tensor", "<i4"), ("pad", "<i4"),
                      ("addr", "<u8")])


def _trace_struct(tr):
    arrs = dict(size=np.ascontiguousarray(tr.size, np.uint64),
                is_param=np.ascontiguousarray(tr.is_param, np.uint8),
                producer=np.ascontiguousarray(tr.producer, np.int32),
                cost_us=np.ascontiguousarray(tr.cost_us, np.int64),
                out=np.ascontiguousarray(tr.out, np.int32),
                inplace_src=np.ascontiguousarray(tr.inplace_src, np.int32),
                phase=np.ascontiguousarray(tr.phase, np.uint8),
                in_ptr=np.ascontiguousarray(tr.in_ptr, np.int32),
                in_idx=np.ascontiguousarray(tr.in_idx if len(tr.in_idx) else np.zeros(1, np.int32), np.int32))
    st = _OrcTrace(len(arrs["size"]), len(arrs["out"]), *[arrs[k].ctypes.data for k in
                   ("size", "is_param", "producer", "cost_us", "out", "inplace_src", "phase",
                    "in_ptr", "in_idx")])
    return st, arrs


def _replay_lib():
    L = lib()
    if not getattr(L, "_replay_ready", False):
        L.orc_replay.argtypes = [ctypes.POINTER(_OrcTrace), ctypes.POINTER(_OrcCfg),
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        L.orc_replay.restype = ctypes.c_int
        L.orc_peak_live.argtypes = [ctypes.POINTER(_OrcTrace), ctypes.c_uint32]
        L.orc_peak_live.restype = ctypes.c_uint64
        L._replay_ready = True
    return L


def replay(tr, budget: int, flags: int = F_PARTITION | F_INPLACE, class_threshold: int = 15,
           max_depth: int = 512, log_cap: int = 0):
    """O2 -> (result record, event log array or None)"""
    L = _replay_lib()
    st, keep = _trace_struct(tr)
    cfg = _OrcCfg(int(budget), int(flags), int(class_threshold), int(max_depth), 0)
    res = np.zeros(1, ORC_RESULT)
    log = np.zeros(max(log_cap, 1), ORC_EVENT) if log_cap else None
    L.orc_replay(ctypes.byref(st), ctypes.byref(cfg), res.ctypes.data,
                 log.ctypes.data if log is not None else None, int(log_cap))
    r = res[0]
    if log is not None:
        log = log[:min(int(r["n_events"]), log_cap)]
    return r, log


def peak_live(tr, flags: int = F_PARTITION | F_INPLACE) -> int:
    L = _replay_lib()
    st, keep = _trace_struct(tr)
    return int(L.orc_peak_live(ctypes.byref(st), int(flags)))


# ----------------------------------------------------------------------------- O3 online
NEEDS_REMAT, UNKNOWN_ID, NOMEM, BAD_STATE = 1, -2, -6, -7
OP_EXPENSIVE, OP_CHEAP, OP_INPLACE, OP_UNEVICTABLE, OP_PHASE_FWD = 1, 2, 4, 8, 16
ORC_ALLOC = np.dtype([("tensor_id", "<i8"), ("addr", "<u8"), ("size", "<u8"),
                      ("n_evicted", "<i4"), ("window_first", "<i4"), ("window_last", "<i4"),
                      ("reserved", "<i4"), ("window_span", "<u8"), ("window_cost", "<f8")])


def _pool_lib():
    L = lib()
    if not getattr(L, "_pool_ready", False):
        vp, i32, u32, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64
        L.orc_pool_create.argtypes = [u64, u32, u32, i32, i32]
        L.orc_pool_create.restype = vp
        L.orc_pool_destroy.argtypes = [vp]
        L.orc_pool_destroy.restype = None
        L.orc_pool_alloc.argtypes = [vp, u64, u64, u32, i32, vp, i32, vp, vp, i32]
        L.orc_pool_free.argtypes = [vp, i32]
        L.orc_pool_access.argtypes = [vp, i32, u64]
        L.orc_pool_remat.argtypes = [vp, i32, vp, vp, i32]
        L.orc_pool_stats.argtypes = [vp, vp]
        L.orc_pool_layout.argtypes = [vp, vp, vp, vp, i32]
        for f in ("orc_pool_alloc", "orc_pool_free", "orc_pool_access", "orc_pool_remat",
                  "orc_pool_stats", "orc_pool_layout"):
            getattr(L, f).restype = ctypes.c_int
        L._pool_ready = True
    return L


class Pool:
    """O3: the online single-pool calls (alloc / free / access / remat), plain C."""

    def __init__(self, budget: int, flags: int = F_PARTITION | F_INPLACE, class_threshold: int = 15,
                 max_tensors: int = 4096, max_edges: int = 16384):
        self._L = _pool_lib()
        self._p = self._L.orc_pool_create(int(budget), int(flags), int(class_threshold),
                                          int(max_tensors), int(max_edges))
        if not self._p:
            raise ValueError("orc_pool_create: bad arguments")

    def __del__(self):
        if getattr(self, "_p", None):
            self._L.orc_pool_destroy(self._p)
            self._p = None

    def _res(self, st, out, ev, cap):
        o = out[0]
        n = min(int(o["n_evicted"]), cap) if st == OK else 0
        return st, o, [int(x) for x in ev[:n]]

    def alloc(self, size, cost_us, op_flags=0, inplace_src=-1, parents=(), evicted_cap=8192):
        par = np.ascontiguousarray(list(parents) or [0], np.int32)
        out = np.zeros(1, ORC_ALLOC)
        ev = np.zeros(max(evicted_cap, 1), np.int32)
        st = self._L.orc_pool_alloc(self._p, int(size), int(cost_us), int(op_flags), int(inplace_src),
                                    par.ctypes.data, len(parents), out.ctypes.data, ev.ctypes.data,
                                    int(evicted_cap))
        return self._res(st, out, ev, evicted_cap)

    def free(self, t):
        return self._L.orc_pool_free(self._p, int(t))

    def access(self, t, advance_us=0):
        return self._L.orc_pool_access(self._p, int(t), int(advance_us))

    def remat(self, t, evicted_cap=8192):
        out = np.zeros(1, ORC_ALLOC)
        ev = np.zeros(max(evicted_cap, 1), np.int32)
        st = self._L.orc_pool_remat(self._p, int(t), out.ctypes.data, ev.ctypes.data, int(evicted_cap))
        return self._res(st, out, ev, evicted_cap)

    def stats(self):
        res = np.zeros(1, ORC_RESULT)
        self._L.orc_pool_stats(self._p, res.ctypes.data)
        return res[0]

    def layout(self, cap=8192):
        a = np.zeros(cap, np.uint64)
        z = np.zeros(cap, np.uint64)
        o = np.zeros(cap, np.int32)
        n = self._L.orc_pool_layout(self._p, a.ctypes.data, z.ctypes.data, o.ctypes.data, cap)
        n = min(n, cap)
        return a[:n].copy(), z[:n].copy(), o[:n].copy()


# ----------------------------------------------------------------------------- O4 budgets
ORC_BUDGET = np.dtype([("peak", "<u8"), ("min_budget", "<u8"), ("cutoff_budget", "<u8"),
                       ("min_status", "<i4"), ("cutoff_status", "<i4"), ("replays", "<i4"),
                       ("reserved", "<i4")])


def budget_search(tr, flags: int = F_PARTITION | F_INPLACE, class_threshold: int = 15,
                  max_depth: int = 512, coarse: int = 64, fine: int = 64):
    """O4 -> orc_budget_result record (min / cutoff budgets on the R45 grids)"""
    L = _replay_lib()
    if not getattr(L, "_budget_ready", False):
        L.orc_budget_search.argtypes = [ctypes.POINTER(_OrcTrace), ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
        L.orc_budget_search.restype = ctypes.c_int
        L._budget_ready = True
    st, keep = _trace_struct(tr)
    out = np.zeros(1, ORC_BUDGET)
    L.orc_budget_search(ctypes.byref(st), int(flags), int(class_threshold), int(max_depth),
                        int(coarse), int(fine), out.ctypes.data)
    return out[0]
