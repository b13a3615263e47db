"""GPU parity of the online single-pool calls (libcoop coop_pool_* / coop_alloc / coop_free /
coop_access / coop_rematerialize) with the oracle O3: call-by-call statuses, placements,
evicted windows (items, span, cost bits) and evicted ids; then counters (incl. the eviction
digest) and the block table.  Seeded random sessions from tests/pool_model.py plus the
SPEC.md worked examples replayed through the CUDA path."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import pool_model as PM  # noqa: E402
from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

STATS = ("fail_op", "base_us", "total_us", "evictions", "remat", "pressure", "frag_fail",
         "inplace_reuse", "heuristic_evals", "sum_free_bytes_after", "sum_free_blocks_after",
         "digest", "max_blocks", "budget", "n_events")


def _coop():
    from paper_2311_00591_b200 import coop
    return coop


def _same_state(g, o):
    sg, so = g.stats(), o.stats()
    for k in STATS:
        assert sg[k].item() == so[k].item(), k
    ag, zg, og = g.layout()
    ao, zo, oo = o.layout()
    assert np.array_equal(ag, ao) and np.array_equal(zg, zo) and np.array_equal(og, oo.astype(np.int64))


@pytest.mark.parametrize("flags", [0, 1, 2, 3, 7, 8, 16, 19])
def test_random_sessions_parity(flags):
    coop = _coop()
    for seed in range(8):
        budget = 150 + (seed * 53) % 500
        calls = PM.random_session(7000 + 100 * flags + seed, 150, budget=budget, flags=flags)
        g = coop.Pool(budget, flags)
        o = O.Pool(budget, flags)
        tg = PM.drive(g, calls)
        to = PM.drive(o, calls)
        for i, (a, b) in enumerate(zip(tg, to)):
            assert a == b, (flags, seed, i, a, b)
        assert len(tg) == len(to)
        _same_state(g, o)
        g.close()


def test_large_pool_session():
    """more blocks than threads: 1200-byte pool with tiny tensors (hundreds of blocks)"""
    coop = _coop()
    calls = PM.random_session(99, 900, budget=1200, flags=3, max_size=6)
    g = coop.Pool(1200, 3)
    o = O.Pool(1200, 3)
    assert PM.drive(g, calls) == PM.drive(o, calls)
    _same_state(g, o)
    assert g.stats()["max_blocks"] > 256


def _rec(x):
    return None if x is None else tuple(sorted((k, x[k].item()) for k in x.dtype.names))


def test_spec_examples_on_gpu():
    """SPEC.md projected-cost example through the CUDA path (numbers derived in
    test_oracle_pool.py), then a remat that must evict, compared with O3 call by call."""
    coop = _coop()
    g, o = coop.Pool(30, 0), O.Pool(30, 0)
    seq = [("alloc", 10, 100, coop.OP_UNEVICTABLE, -1, []), ("alloc", 10, 1, 0, -1, [0]),
           ("alloc", 10, 100, 0, -1, [1]), ("access", 2, 50), ("alloc", 10, 0, coop.OP_UNEVICTABLE, -1, []),
           ("alloc", 10, 0, 0, -1, []), ("access", 1, 0), ("remat", 1), ("access", 2, 7),
           ("remat", 2), ("free", 0), ("remat", 0), ("free", 1), ("free", 1)]
    outs = []
    for impl in (g, o):
        tr = []
        for c in seq:
            if c[0] == "alloc":
                st, r, ev = impl.alloc(*c[1:])
                tr.append((st, _rec(r) if st == 0 else None, ev))
            elif c[0] == "remat":
                st, r, ev = impl.remat(c[1])
                tr.append((st, _rec(r) if st == 0 else None, ev))
            elif c[0] == "access":
                tr.append(impl.access(c[1], c[2]))
            else:
                tr.append(impl.free(c[1]))
        outs.append(tr)
    assert outs[0] == outs[1]
    d, e = dict(outs[0][4][1]), dict(outs[0][5][1])
    assert d["window_cost"] == 1.0 / 50.0 and outs[0][4][2] == [1]
    assert e["window_cost"] == 101.0 and outs[0][5][2] == [2]
    assert outs[0][6] == coop.NEEDS_REMAT
    _same_state(g, o)


def test_capacity_and_double_free():
    coop = _coop()
    p = coop.Pool(100, 3, max_tensors=2, max_edges=1)
    t0 = p.alloc(10, 1)[1]["tensor_id"]
    assert p.alloc(10, 1, 0, -1, [t0, t0])[0] == coop.ERR_NOMEM
    t1 = p.alloc(10, 1, 0, -1, [t0])[1]["tensor_id"]
    assert p.alloc(10, 1)[0] == coop.ERR_NOMEM
    assert p.free(t1) == coop.OK and p.free(t1) == coop.ERR_BAD_STATE
    assert p.access(t1) == coop.ERR_BAD_STATE


@pytest.mark.parametrize("flags", [3, 7, 16])
def test_service_mode_parity(flags):
    """coop_pool_service (NEXT-4): the resident polling CTA gives call-by-call the same
    results as the oracle (and so as the launch-per-call mode)"""
    coop = _coop()
    for seed in range(4):
        budget = 200 + (seed * 71) % 400
        calls = PM.random_session(9100 + 10 * flags + seed, 150, budget=budget, flags=flags)
        g = coop.Pool(budget, flags, service_idle_us=200000)
        o = O.Pool(budget, flags)
        tg = PM.drive(g, calls)
        to = PM.drive(o, calls)
        assert tg == to, (flags, seed)
        _same_state(g, o)
        g.close()


def test_service_idle_exit_and_relaunch():
    """the resident kernel exits after its idle timeout (a device-wide synchronize then
    returns), the next call relaunches it transparently, and switching the service off and
    on mid-session keeps the results equal to the oracle's"""
    import time

    import torch
    coop = _coop()

    class Toggling:
        def __init__(self, pool):
            self.p, self.n = pool, 0

        def _tick(self):
            self.n += 1
            if self.n % 25 == 0:
                mode = (self.n // 25) % 3
                self.p.service((0, 2000, 5000)[mode])
                t0 = time.time()
                torch.cuda.synchronize()  # returns once any resident kernel went idle
                assert time.time() - t0 < 5.0
                time.sleep(0.01)

        def __getattr__(self, name):
            f = getattr(self.p, name)
            if name in ("alloc", "free", "access", "remat"):
                def g(*a, **k):
                    self._tick()
                    return f(*a, **k)
                return g
            return f

    calls = PM.random_session(4242, 150, budget=400, flags=3)
    g = coop.Pool(400, 3, service_idle_us=2000)
    o = O.Pool(400, 3)
    assert PM.drive(Toggling(g), calls) == PM.drive(o, calls)
    _same_state(g, o)
    g.close()


def test_service_invalid_timeout_and_stats_flush():
    """coop_pool_service argument check; stats / layout read the live state of a resident
    service kernel (flush) and agree with the oracle mid-session"""
    coop = _coop()
    g = coop.Pool(300, 3)
    assert coop.lib.coop_pool_service(g.handle, 10000001) == coop.ERR_INVALID_ARG
    g.service(50000)
    o = O.Pool(300, 3)
    calls = PM.random_session(31337, 60, budget=300, flags=3)
    assert PM.drive(g, calls) == PM.drive(o, calls)
    _same_state(g, o)  # while the kernel is resident
    g.close()
