"""The C ABI (include/*.h): every declared symbol is exported by the built library, status
codes and argument checks behave as documented.  CPU-only (no compute calls)."""
import ctypes
import math
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions(header):
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(coop_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    from paper_2311_00591_b200 import coop
    names = declared_functions(os.path.join(ROOT, "include", "coop.h"))
    assert "coop_window_search_batched" in names
    lib = ctypes.CDLL(coop.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_status_strings_and_version():
    from paper_2311_00591_b200 import coop
    assert coop.status_string(0) == "COOP_OK"
    assert coop.status_string(-1) == "COOP_ERR_INVALID_ARG"
    assert coop.status_string(12345) == "COOP_ERR_UNKNOWN_STATUS"
    assert "sm_100a" in coop.version()


def test_argument_checks_without_gpu():
    from paper_2311_00591_b200 import coop
    lib = coop.lib
    assert lib.coop_window_search_batched(None, None, None, None) == coop.ERR_INVALID_ARG
    bad = [coop.TablesSoA(1, 1, 1, 1, 0, 0, 16), coop.TablesSoA(1, 1, 1, 1, 8193, 0, 9000),
           coop.TablesSoA(1, 1, 1, 1, 16, 0, 8), coop.TablesSoA(1, 1, 1, -1, 16, 0, 16),
           coop.TablesSoA(1, 1, 1, 1, 16, 7, 16), coop.TablesSoA(0, 1, 1, 1, 16, 0, 16)]
    for t in bad:
        assert lib.coop_window_search_batched(ctypes.byref(t), 1, 1, None) == coop.ERR_INVALID_ARG
    empty = coop.TablesSoA(0, 0, 0, 0, 16, 0, 16)
    assert lib.coop_window_search_batched(ctypes.byref(empty), 0, 0, None) == coop.OK


def test_cuda_exact_sum_arithmetic_on_host():
    """The CUDA path's 192-bit fixed-point sum + ties-to-even rounding (fixed192.cuh),
    compiled for the host, equals math.fsum (correctly rounded) on admissible values."""
    from paper_2311_00591_b200 import coop
    rng = np.random.default_rng(0)
    cases = [[1.0, 2.0 ** -53], [1.0, 2.0 ** -53, 2.0 ** -64], [1.0 + 2.0 ** -52, 2.0 ** -53],
             [2.0 ** 59, 2.0 ** 59, 2.0 ** -64], [2.0 ** -64] * 3, [], [0.0, 0.0],
             [1e-3, 2e-3, 1e-3], [2.0 ** 60 - 2.0 ** 7] * 8192]
    for _ in range(5000):
        k = int(rng.integers(1, 64))
        e = rng.integers(-64, 60, k)
        x = np.ldexp(1.0 + rng.random(k), e)
        x = np.where(x >= 2.0 ** 60, 2.0 ** 59, x)
        if rng.random() < 0.3:
            x[rng.random(k) < 0.3] = 0.0
        cases.append(list(x))
    for _ in range(2000):  # near-midpoint constructions: big + half-ulp pieces
        b = math.ldexp(1.0 + rng.integers(0, 2 ** 52) * 2.0 ** -52, int(rng.integers(-10, 50)))
        half = math.ulp(b) / 2
        extra = [half] if rng.random() < 0.5 else [half / 2, half / 2]
        if rng.random() < 0.5 and half / 4 >= 2.0 ** -64:
            extra.append(half / 4)
        cases.append([b] + [v for v in extra if v >= 2.0 ** -64])
    for xs in cases:
        assert coop._fixed_round_sum_host(np.array(xs, np.float64)) == math.fsum(xs), xs


def test_pool_argument_checks_without_gpu():
    """coop_pool_init validates its config, and every online call rejects a NULL pool,
    before touching the device."""
    from paper_2311_00591_b200 import coop
    lib = coop.lib
    h = ctypes.c_void_p()
    assert lib.coop_pool_init(None, ctypes.byref(h)) == coop.ERR_INVALID_ARG
    for cfg in [coop.PoolConfig(0, 0, 0, 16, 16), coop.PoolConfig(100, 32, 0, 16, 16),
                coop.PoolConfig(100, 24, 0, 16, 16),
                coop.PoolConfig(100, 0, 0, 0, 16), coop.PoolConfig(100, 0, 0, 16385, 16),
                coop.PoolConfig(100, 0, 0, 16, -1)]:
        assert lib.coop_pool_init(ctypes.byref(cfg), ctypes.byref(h)) == coop.ERR_INVALID_ARG
    assert lib.coop_alloc(None, 1, 1, 0, -1, None, 0, None, None, 0) == coop.ERR_INVALID_ARG
    assert lib.coop_free(None, 0) == coop.ERR_INVALID_ARG
    assert lib.coop_access(None, 0, 0) == coop.ERR_INVALID_ARG
    assert lib.coop_rematerialize(None, 0, None, None, 0) == coop.ERR_INVALID_ARG
    assert lib.coop_pool_stats(None, None) == coop.ERR_INVALID_ARG
    n = ctypes.c_int32()
    assert lib.coop_pool_layout(None, None, None, None, 0, ctypes.byref(n)) == coop.ERR_INVALID_ARG
    assert lib.coop_pool_destroy(None) == coop.ERR_INVALID_ARG
    assert lib.coop_pool_service(None, 0) == coop.ERR_INVALID_ARG
    assert coop.ALLOC_RESULT_DTYPE.itemsize == 56
