"""Thin ctypes binding of libcoop (include/coop.h): argument marshalling only.

Every step of the search / replay runs in libcoop's CUDA kernels.  There is no Python or
CPU fallback: if libcoop.so is missing or cannot load, import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("COOP_LIB_OVERRIDE") or os.path.join(_HERE, "libcoop.so")  # override: A/B kernel builds

OK = 0
INFEASIBLE = 1
ERR_INVALID_ARG = -1
ERR_UNKNOWN_ID = -2
ERR_UNSATISFIABLE = -3
ERR_THRASHED = -4
ERR_CUDA = -5
ERR_NOMEM = -6
ERR_BAD_STATE = -7
ERR_UNIMPLEMENTED = -8

FREE, EVICTABLE, PINNED = 0, 1, 2
MAX_BLOCKS = 8192

# struct coop_window (32 bytes)
WINDOW_DTYPE = np.dtype([("first", "<i4"), ("last", "<i4"), ("span", "<u8"),
                         ("cost", "<f8"), ("n_evict", "<i4"), ("status", "<i4")])
assert WINDOW_DTYPE.itemsize == 32


class CoopError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {status_string(status)} ({status})")
        self.status = status


class TablesSoA(ctypes.Structure):
    _fields_ = [("size_state", ctypes.c_void_p), ("cost", ctypes.c_void_p),
                ("stale", ctypes.c_void_p), ("n_pools", ctypes.c_int64),
                ("n_blocks", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("pool_stride", ctypes.c_int64)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libcoop.so not built at {LIB_PATH}; run __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    lib.coop_status_string.restype = ctypes.c_char_p
    lib.coop_status_string.argtypes = [ctypes.c_int]
    lib.coop_version.restype = ctypes.c_char_p
    lib.coop_window_search_batched.restype = ctypes.c_int
    lib.coop_window_search_batched.argtypes = [ctypes.POINTER(TablesSoA), ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_void_p]
    lib.coop_window_search_batched_host.restype = ctypes.c_int
    lib.coop_window_search_batched_host.argtypes = [ctypes.POINTER(TablesSoA), ctypes.c_void_p,
                                                    ctypes.c_void_p, ctypes.c_int64]
    lib.coop__fixed_round_sum_host.restype = ctypes.c_double
    lib.coop__fixed_round_sum_host.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    return lib


lib = _load()


def status_string(status: int) -> str:
    return lib.coop_status_string(int(status)).decode()


def version() -> str:
    return lib.coop_version().decode()


def _ptr(x) -> int:
    """data pointer of a torch tensor or numpy array"""
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    return int(x.ctypes.data)


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        return int(torch.cuda.current_stream().cuda_stream)
    if hasattr(stream, "cuda_stream"):
        return int(stream.cuda_stream)
    return int(stream)


def window_search_batched(size_state, cost, stale, requests, out, n_pools: int, n_blocks: int,
                          pool_stride: int, stream=None) -> int:
    """coop_window_search_batched on device buffers (torch CUDA tensors or raw pointers).

    `out` must hold n_pools * 32 bytes (e.g. torch.empty(n_pools * 4, dtype=torch.int64)).
    Asynchronous on `stream` (default: torch's current stream).  Raises on error status.
    """
    t = TablesSoA(_ptr(size_state) if not isinstance(size_state, int) else size_state,
                  _ptr(cost) if not isinstance(cost, int) else cost,
                  _ptr(stale) if not isinstance(stale, int) else stale,
                  int(n_pools), int(n_blocks), 0, int(pool_stride))
    rc = lib.coop_window_search_batched(
        ctypes.byref(t), _ptr(requests) if not isinstance(requests, int) else requests,
        _ptr(out) if not isinstance(out, int) else out, _stream_handle(stream))
    if rc < 0:
        raise CoopError(rc, "coop_window_search_batched")
    return rc


def window_search_batched_host(size_state, cost, stale, requests, n_pools: int, n_blocks: int,
                               pool_stride: int, out=None, chunk_pools: int = 0) -> np.ndarray:
    """coop_window_search_batched_host on host arrays (numpy or CPU torch, ideally pinned)."""
    if out is None:
        out = np.empty(n_pools, dtype=WINDOW_DTYPE)
    t = TablesSoA(_ptr(size_state), _ptr(cost), _ptr(stale), int(n_pools), int(n_blocks), 0,
                  int(pool_stride))
    rc = lib.coop_window_search_batched_host(ctypes.byref(t), _ptr(requests), _ptr(out),
                                             int(chunk_pools))
    if rc < 0:
        raise CoopError(rc, "coop_window_search_batched_host")
    return out


def windows_from_device(out_tensor) -> np.ndarray:
    """copy a device result buffer to a numpy structured array of coop_window"""
    raw = out_tensor.cpu().numpy().view(np.uint8)
    return raw.view(WINDOW_DTYPE)


def _fixed_round_sum_host(h: np.ndarray) -> float:
    """test hook: the CUDA path's 192-bit exact-sum + RN, compiled for the host"""
    h = np.ascontiguousarray(h, dtype=np.float64)
    return float(lib.coop__fixed_round_sum_host(h.ctypes.data, h.size))


# ----------------------------------------------------------------------------- replay
class TraceDesc(ctypes.Structure):
    _fields_ = [("n_tensors", ctypes.c_int32), ("n_ops", ctypes.c_int32),
                ("size", ctypes.c_void_p), ("is_param", ctypes.c_void_p),
                ("producer", ctypes.c_void_p), ("cost_us", ctypes.c_void_p),
                ("out", ctypes.c_void_p), ("inplace_src", ctypes.c_void_p),
                ("phase", ctypes.c_void_p), ("in_ptr", ctypes.c_void_p),
                ("in_idx", ctypes.c_void_p)]


F_PARTITION, F_INPLACE, F_PARTITION_ALL_PHASES = 1, 2, 4
F_POLICY_DTR, F_POLICY_DTE = 8, 16  # the paper's baseline eviction policies (R46)

REPLAY_RESULT_DTYPE = np.dtype([
    ("status", "<i4"), ("fail_op", "<i4"), ("base_us", "<i8"), ("total_us", "<i8"),
    ("evictions", "<i8"), ("remat", "<i8"), ("pressure", "<i8"), ("frag_fail", "<i8"),
    ("inplace_reuse", "<i8"), ("heuristic_evals", "<i8"), ("sum_free_bytes_after", "<u8"),
    ("sum_free_blocks_after", "<i8"), ("digest", "<u8"), ("max_depth", "<i4"),
    ("max_blocks", "<i4"), ("budget", "<u8"), ("n_events", "<i8"),
    ("search_ns_total", "<i8"), ("search_ns_max", "<i8")])
assert REPLAY_RESULT_DTYPE.itemsize == 136
EVENT_DTYPE = np.dtype([("kind", "<i4"), ("op", "<i4"), ("tensor", "<i4"), ("pad", "<i4"),
                        ("addr", "<u8")])

lib.coop_trace_create.argtypes = [ctypes.POINTER(TraceDesc), ctypes.POINTER(ctypes.c_void_p)]
lib.coop_trace_create.restype = ctypes.c_int
lib.coop_trace_destroy.argtypes = [ctypes.c_void_p]
lib.coop_trace_destroy.restype = ctypes.c_int
lib.coop_trace_peak_live.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64)]
lib.coop_trace_peak_live.restype = ctypes.c_int
lib.coop_replay_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32,
                                  ctypes.c_uint32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_int64, ctypes.c_void_p]
lib.coop_replay_trace.restype = ctypes.c_int
lib.coop_replay_snapshots.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_int32, ctypes.c_int32, ctypes.c_int64] + [ctypes.c_void_p] * 8
lib.coop_replay_snapshots.restype = ctypes.c_int


class Trace:
    """A trace uploaded to the device (coop_trace_create); `tr` has the SoA fields of
    gen.traces.Trace."""

    def __init__(self, tr):
        arrs = dict(size=np.ascontiguousarray(tr.size, np.uint64),
                    is_param=np.ascontiguousarray(tr.is_param, np.uint8),
                    producer=np.ascontiguousarray(tr.producer, np.int32),
                    cost_us=np.ascontiguousarray(tr.cost_us, np.int64),
                    out=np.ascontiguousarray(tr.out, np.int32),
                    inplace_src=np.ascontiguousarray(tr.inplace_src, np.int32),
                    phase=np.ascontiguousarray(tr.phase, np.uint8),
                    in_ptr=np.ascontiguousarray(tr.in_ptr, np.int32),
                    in_idx=np.ascontiguousarray(tr.in_idx if len(tr.in_idx) else np.zeros(1, np.int32), np.int32))
        d = TraceDesc(len(arrs["size"]), len(arrs["out"]), *[arrs[k].ctypes.data for k in
                      ("size", "is_param", "producer", "cost_us", "out", "inplace_src", "phase",
                       "in_ptr", "in_idx")])
        h = ctypes.c_void_p()
        rc = lib.coop_trace_create(ctypes.byref(d), ctypes.byref(h))
        if rc != OK:
            raise CoopError(rc, "coop_trace_create")
        self.handle = h
        self.n_tensors = len(arrs["size"])
        self.n_ops = len(arrs["out"])

    def close(self):
        if self.handle:
            lib.coop_trace_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def peak_live(self, flags: int) -> int:
        v = ctypes.c_uint64()
        rc = lib.coop_trace_peak_live(self.handle, int(flags), ctypes.byref(v))
        if rc != OK:
            raise CoopError(rc, "coop_trace_peak_live")
        return int(v.value)

    def replay_device(self, budgets, flags, out, log=None, log_cap: int = 0, class_threshold: int = 0,
                      max_depth: int = 0, stream=None) -> None:
        """coop_replay_trace into device buffers (torch tensors); asynchronous."""
        b = np.ascontiguousarray(budgets, np.uint64)
        rc = lib.coop_replay_trace(self.handle, b.ctypes.data, len(b), int(flags),
                                   int(class_threshold), int(max_depth), _ptr(out),
                                   _ptr(log) if log is not None else None, int(log_cap),
                                   _stream_handle(stream))
        if rc != OK:
            raise CoopError(rc, "coop_replay_trace")

    def snapshots_device(self, budget: int, flags: int, n_max: int, ss, cost, stale, requests, windows,
                         count, out, cap: int, class_threshold: int = 0, max_depth: int = 0, stream=None) -> None:
        """coop_replay_snapshots into device buffers (torch tensors); asynchronous."""
        rc = lib.coop_replay_snapshots(self.handle, int(budget), int(flags), int(class_threshold),
                                       int(max_depth), int(n_max), int(cap), _ptr(ss), _ptr(cost),
                                       _ptr(stale), _ptr(requests), _ptr(windows), _ptr(count), _ptr(out),
                                       _stream_handle(stream))
        if rc != OK:
            raise CoopError(rc, "coop_replay_snapshots")

    def snapshots(self, budget: int, flags: int, n_max: int, cap: int):
        """Synchronous: -> dict of device tensors ss / cost / stale [cap * n_max], requests [cap],
        windows (raw int64 [cap * 4]), plus count (int) and the replay result record."""
        import torch
        d = dict(ss=torch.empty(cap * n_max, dtype=torch.int64, device="cuda"),
                 cost=torch.empty(cap * n_max, dtype=torch.float64, device="cuda"),
                 stale=torch.empty(cap * n_max, dtype=torch.float64, device="cuda"),
                 requests=torch.empty(cap, dtype=torch.int64, device="cuda"),
                 windows=torch.empty(cap * 4, dtype=torch.int64, device="cuda"))
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        out = torch.empty(REPLAY_RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
        self.snapshots_device(budget, flags, n_max, d["ss"], d["cost"], d["stale"], d["requests"],
                              d["windows"], cnt, out, cap)
        torch.cuda.synchronize()
        d["count"] = int(cnt.item())
        d["result"] = out.cpu().numpy().view(REPLAY_RESULT_DTYPE)[0]
        return d

    def replay(self, budgets, flags, log_cap: int = 0, class_threshold: int = 0, max_depth: int = 0):
        """Synchronous convenience wrapper -> (results [n], events [n, log_cap] or None)."""
        import torch
        n = len(budgets)
        out = torch.empty(n * REPLAY_RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
        log = (torch.empty(max(1, n * log_cap) * EVENT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
               if log_cap else None)
        self.replay_device(budgets, flags, out, log, log_cap, class_threshold, max_depth)
        torch.cuda.synchronize()
        res = out.cpu().numpy().view(REPLAY_RESULT_DTYPE)
        ev = log.cpu().numpy().view(EVENT_DTYPE).reshape(n, log_cap) if log is not None else None
        return res, ev


# ----------------------------------------------------------------------------- online pool
NEEDS_REMAT = 1
OP_EXPENSIVE, OP_CHEAP, OP_INPLACE, OP_UNEVICTABLE, OP_PHASE_FWD = 1, 2, 4, 8, 16

# struct coop_alloc_result (56 bytes)
ALLOC_RESULT_DTYPE = np.dtype([("tensor_id", "<i8"), ("addr", "<u8"), ("size", "<u8"),
                               ("n_evicted", "<i4"), ("window_first", "<i4"),
                               ("window_last", "<i4"), ("reserved", "<i4"),
                               ("window_span", "<u8"), ("window_cost", "<f8")])
assert ALLOC_RESULT_DTYPE.itemsize == 56


class PoolConfig(ctypes.Structure):
    _fields_ = [("budget", ctypes.c_uint64), ("flags", ctypes.c_uint32),
                ("class_threshold", ctypes.c_uint32), ("max_tensors", ctypes.c_int32),
                ("max_edges", ctypes.c_int32)]


_vp = ctypes.c_void_p
lib.coop_pool_init.argtypes = [ctypes.POINTER(PoolConfig), ctypes.POINTER(_vp)]
lib.coop_pool_destroy.argtypes = [_vp]
lib.coop_alloc.argtypes = [_vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64,
                           _vp, ctypes.c_int32, _vp, _vp, ctypes.c_int32]
lib.coop_free.argtypes = [_vp, ctypes.c_int64]
lib.coop_access.argtypes = [_vp, ctypes.c_int64, ctypes.c_uint64]
lib.coop_rematerialize.argtypes = [_vp, ctypes.c_int64, _vp, _vp, ctypes.c_int32]
lib.coop_pool_stats.argtypes = [_vp, _vp]
lib.coop_pool_layout.argtypes = [_vp, _vp, _vp, _vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
lib.coop_pool_service.argtypes = [_vp, ctypes.c_uint32]
for _f in ("coop_pool_init", "coop_pool_destroy", "coop_alloc", "coop_free", "coop_access",
           "coop_rematerialize", "coop_pool_stats", "coop_pool_layout", "coop_pool_service"):
    getattr(lib, _f).restype = ctypes.c_int


class Pool:
    """One device-resident pool driven call by call (coop_pool_init and friends).  Calls
    return the library status (errors are returned, not raised, like the C API):
    alloc / remat -> (status, coop_alloc_result record, evicted ids); free / access ->
    status."""

    def __init__(self, budget: int, flags: int = F_PARTITION | F_INPLACE, class_threshold: int = 15,
                 max_tensors: int = 4096, max_edges: int = 16384, service_idle_us: int = 0):
        cfg = PoolConfig(int(budget), int(flags), int(class_threshold), int(max_tensors), int(max_edges))
        h = _vp()
        rc = lib.coop_pool_init(ctypes.byref(cfg), ctypes.byref(h))
        if rc != OK:
            raise CoopError(rc, "coop_pool_init")
        self.handle = h
        self._ev = np.zeros(8192, np.int64)
        if service_idle_us:
            self.service(service_idle_us)

    def service(self, idle_timeout_us: int):
        """coop_pool_service: resident polling CTA (idle_timeout_us > 0) or one launch per call (0)."""
        rc = lib.coop_pool_service(self.handle, int(idle_timeout_us))
        if rc != OK:
            raise CoopError(rc, "coop_pool_service")

    def close(self):
        if self.handle:
            lib.coop_pool_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _res(self, st, out, cap):
        n = min(int(out[0]["n_evicted"]), cap) if st == OK else 0
        return st, out[0], [int(x) for x in self._ev[:n]]

    def alloc(self, size, cost_us, op_flags=0, inplace_src=-1, parents=(), evicted_cap=8192):
        par = np.ascontiguousarray(list(parents) or [0], np.int64)
        out = np.zeros(1, ALLOC_RESULT_DTYPE)
        cap = min(evicted_cap, len(self._ev))
        st = lib.coop_alloc(self.handle, int(size), int(cost_us), int(op_flags), int(inplace_src),
                            par.ctypes.data, len(parents), out.ctypes.data, self._ev.ctypes.data, cap)
        return self._res(st, out, cap)

    def free(self, t):
        return lib.coop_free(self.handle, int(t))

    def access(self, t, advance_us=0):
        return lib.coop_access(self.handle, int(t), int(advance_us))

    def remat(self, t, evicted_cap=8192):
        out = np.zeros(1, ALLOC_RESULT_DTYPE)
        cap = min(evicted_cap, len(self._ev))
        st = lib.coop_rematerialize(self.handle, int(t), out.ctypes.data, self._ev.ctypes.data, cap)
        return self._res(st, out, cap)

    def stats(self):
        res = np.zeros(1, REPLAY_RESULT_DTYPE)
        rc = lib.coop_pool_stats(self.handle, res.ctypes.data)
        if rc != OK:
            raise CoopError(rc, "coop_pool_stats")
        return res[0]

    def layout(self, cap=8192):
        a = np.zeros(cap, np.uint64)
        z = np.zeros(cap, np.uint64)
        o = np.zeros(cap, np.int64)
        n = ctypes.c_int32()
        rc = lib.coop_pool_layout(self.handle, a.ctypes.data, z.ctypes.data, o.ctypes.data, cap,
                                  ctypes.byref(n))
        if rc != OK:
            raise CoopError(rc, "coop_pool_layout")
        k = min(n.value, cap)
        return a[:k].copy(), z[:k].copy(), o[:k].copy()


# ----------------------------------------------------------------------------- budget searches
BUDGET_RESULT_DTYPE = np.dtype([("peak", "<u8"), ("min_budget", "<u8"), ("cutoff_budget", "<u8"),
                                ("min_status", "<i4"), ("cutoff_status", "<i4"), ("replays", "<i4"),
                                ("reserved", "<i4")])
assert BUDGET_RESULT_DTYPE.itemsize == 40
lib.coop_budget_search.argtypes = [_vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int32, ctypes.c_int32,
                                   ctypes.c_int32, _vp]
lib.coop_budget_search.restype = ctypes.c_int


def budget_search(trace: "Trace", flags: int, coarse: int = 64, fine: int = 64, class_threshold: int = 0,
                  max_depth: int = 0):
    """coop_budget_search -> coop_budget_result record (min / cutoff budgets, R45)."""
    out = np.zeros(1, BUDGET_RESULT_DTYPE)
    rc = lib.coop_budget_search(trace.handle, int(flags), int(class_threshold), int(max_depth),
                                int(coarse), int(fine), out.ctypes.data)
    if rc != OK:
        raise CoopError(rc, "coop_budget_search")
    return out[0]
