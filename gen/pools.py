"""Seeded block-table generators.

* `bench_pools_host` / `bench_pools_device` -- the counter-based generator of gen/coop_gen.cu
  (config 1 "small" and config 4 "bench" laws), host and device, bit-identical.
* `random_pool` and friends -- numpy generators for parity tests (ties, barriers,
  cancellation, ragged sizes).  They only draw inputs; no search arithmetic lives here.

Block-table encoding: size_state = size | state << 62,
state 0 FREE / 1 EVICTABLE / 2 PINNED; cost c (us), stale s (us).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIBGEN_PATH = os.path.join(_HERE, "libcoopgen.so")

MODE_BENCH = 0
MODE_SMALL = 1
FREE, EVICTABLE, PINNED = 0, 1, 2

_lib = None


def _gen_lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIBGEN_PATH):
            raise ImportError(f"{LIBGEN_PATH} missing; run __graft_entry__.build()")
        lib = ctypes.CDLL(LIBGEN_PATH)
        args = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                ctypes.c_void_p]
        lib.coopgen_pools_host.argtypes = args
        lib.coopgen_pools_host.restype = ctypes.c_int
        lib.coopgen_pools_device.argtypes = args + [ctypes.c_void_p]
        lib.coopgen_pools_device.restype = ctypes.c_int
        _lib = lib
    return _lib


def bench_pools_host(mode: int, seed: int, p0: int, n_pools: int, n: int, stride: int | None = None):
    """Host arrays (size_state u64, cost f64, stale f64 [n_pools*stride]; requests u64)."""
    stride = n if stride is None else stride
    ss = np.zeros(n_pools * stride, np.uint64)
    c = np.zeros(n_pools * stride, np.float64)
    s = np.ones(n_pools * stride, np.float64)
    r = np.zeros(n_pools, np.uint64)
    rc = _gen_lib().coopgen_pools_host(mode, seed, p0, n_pools, n, stride, ss.ctypes.data,
                                       c.ctypes.data, s.ctypes.data, r.ctypes.data)
    if rc != 0:
        raise ValueError(f"coopgen_pools_host failed ({rc})")
    return ss, c, s, r


def bench_pools_device(mode: int, seed: int, p0: int, n_pools: int, n: int, stride: int,
                       ss, c, s, r, stream: int = 0) -> None:
    """Fill device buffers (torch CUDA tensors) asynchronously."""
    rc = _gen_lib().coopgen_pools_device(mode, seed, p0, n_pools, n, stride, ss.data_ptr(),
                                         c.data_ptr(), s.data_ptr(), r.data_ptr(), stream)
    if rc != 0:
        raise RuntimeError(f"coopgen_pools_device failed ({rc})")


def pack(sizes, states) -> np.ndarray:
    sizes = np.asarray(sizes, dtype=np.uint64)
    states = np.asarray(states, dtype=np.uint64)
    return sizes | (states << np.uint64(62))


def random_pool(rng: np.random.Generator, n: int, p_free=0.12, p_pinned=0.05, max_size=64,
                h_choices=None, coalesced=True, cost_scale=1.0):
    """One random pool: (size_state, cost, stale).  With h_choices, EVICTABLE items get
    h exactly from the given list (c = h * s with s a power of two => c/s == h exactly)."""
    st = np.full(n, EVICTABLE, np.uint64)
    u = rng.random(n)
    st[u < p_free] = FREE
    st[(u >= p_free) & (u < p_free + p_pinned)] = PINNED
    if coalesced:
        for k in range(1, n):
            if st[k] == FREE and st[k - 1] == FREE:
                st[k] = EVICTABLE
    sizes = rng.integers(1, max_size + 1, n).astype(np.uint64)
    if h_choices is not None:
        s = (2.0 ** rng.integers(0, 8, n)).astype(np.float64)
        h = np.asarray(h_choices, np.float64)[rng.integers(0, len(h_choices), n)]
        c = h * s
    else:
        s = rng.integers(1, 10**6, n).astype(np.float64)
        c = rng.random(n) * 1000.0 * cost_scale
    return pack(sizes, st), c, s


def stack_pools(pools, stride: int | None = None):
    """Stack same-length pools into SoA pool-major arrays with the given stride."""
    n = len(pools[0][0])
    stride = n if stride is None else stride
    P = len(pools)
    ss = np.zeros(P * stride, np.uint64)
    c = np.zeros(P * stride, np.float64)
    s = np.ones(P * stride, np.float64)
    for p, (a, b, d) in enumerate(pools):
        ss[p * stride:p * stride + n] = a
        c[p * stride:p * stride + n] = b
        s[p * stride:p * stride + n] = d
    return ss, c, s
