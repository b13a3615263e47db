"""Pins of the oracle O3 (online single-pool calls, R38-R44) -- CPU only.

* SPEC.md's worked examples for the pool operations (alloc_left / alloc_right / free_block,
  SPEC.md:148-206) and the projected-cost examples, with expected values
  derived by hand in the comments;
* call-by-call agreement with the independent Python model tests/pool_model.py (byte-map
  memory, O(N^2) exact-Fraction windows, set closures) on seeded random sessions;
* the error statuses of every call.
"""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from oracle import oracle as O  # noqa: E402
import pool_model as PM  # noqa: E402

NOPART = 0


def test_alloc_left_examples():
    # SPEC.md alloc_left: empty pool, size 100 -> addr 0
    p = O.Pool(1000, NOPART)
    st, r, ev = p.alloc(100, 5)
    assert st == O.OK and r["addr"] == 0 and r["tensor_id"] == 0 and ev == []
    # free blocks [0,50) and [100,300), request 100 -> addr 100 (first block too small)
    p = O.Pool(300, NOPART)
    t0 = p.alloc(50, 1)[1]["tensor_id"]
    p.alloc(50, 1)
    t2 = p.alloc(200, 1)[1]["tensor_id"]
    assert p.free(t0) == O.OK and p.free(t2) == O.OK
    st, r, ev = p.alloc(100, 1)
    assert st == O.OK and r["addr"] == 100 and ev == []


def test_fit_failure_despite_free_bytes():
    # SPEC.md alloc_left: free blocks [0,50) and [60,110), request 60 -> no contiguous block
    # although bytes_free = 100; the middle tensor is unevictable, so no window exists
    p = O.Pool(110, NOPART)
    t0 = p.alloc(50, 1)[1]["tensor_id"]
    p.alloc(10, 1, O.OP_UNEVICTABLE)
    t2 = p.alloc(50, 1)[1]["tensor_id"]
    p.free(t0)
    p.free(t2)
    st, r, ev = p.alloc(60, 1)
    assert st == O.UNSATISFIABLE
    s = p.stats()
    assert s["pressure"] == 1 and s["frag_fail"] == 1 and s["evictions"] == 0
    # the failed call created no tensor: the next id is still 3
    st, r, ev = p.alloc(50, 1)
    assert st == O.OK and r["tensor_id"] == 3 and r["addr"] == 0


def test_alloc_right_examples():
    # SPEC.md alloc_right (cheap tensor partitioning, forward phase): empty pool of 1000,
    # size 100 -> addr 900 = right_addr - size
    cheap = O.OP_CHEAP | O.OP_PHASE_FWD
    p = O.Pool(1000, O.F_PARTITION)
    st, r, ev = p.alloc(100, 1, cheap)
    assert st == O.OK and r["addr"] == 900
    # free blocks [0,500) and [900,1000): request 100 -> 900 (the rightmost block)
    p = O.Pool(1000, O.F_PARTITION)
    a = p.alloc(500, 1, O.OP_EXPENSIVE)[1]["tensor_id"]  # [0,500), left
    p.alloc(400, 1, O.OP_EXPENSIVE)                      # [500,900)
    p.free(a)
    st, r, _ = p.alloc(100, 1, cheap)
    assert st == O.OK and r["addr"] == 900


def test_alloc_right_forced_by_fit():
    cheap = O.OP_CHEAP | O.OP_PHASE_FWD
    p = O.Pool(1000, O.F_PARTITION)
    a = p.alloc(500, 1, O.OP_EXPENSIVE)[1]["tensor_id"]  # [0,500)
    p.alloc(400, 1, O.OP_EXPENSIVE)                      # [500,900); free: [900,1000)
    p.free(a)                                            # free: [0,500), [900,1000)
    st, r, _ = p.alloc(200, 1, cheap)                    # [900,1000) too small -> 500-200
    assert st == O.OK and r["addr"] == 300
    # outside the forward phase, cheap outputs go left unless PARTITION_ALL_PHASES
    p = O.Pool(1000, O.F_PARTITION)
    assert p.alloc(100, 1, O.OP_CHEAP)[1]["addr"] == 0
    p = O.Pool(1000, O.F_PARTITION | O.F_PARTITION_ALL_PHASES)
    assert p.alloc(100, 1, O.OP_CHEAP)[1]["addr"] == 900
    # no class flag: the R14 threshold (cost * 2^20 >= 15 * bytes -> C1, left)
    p = O.Pool(1 << 30, O.F_PARTITION)
    assert p.alloc(1 << 20, 15, O.OP_PHASE_FWD)[1]["addr"] == 0            # 15 us/MiB: C1
    assert p.alloc(1 << 20, 14, O.OP_PHASE_FWD)[1]["addr"] == (1 << 30) - (1 << 20)  # C2


def test_free_block_examples():
    # SPEC.md free_block: a live block between two free blocks merges into one free block;
    # freeing the only live block returns the pool to [0, budget); freeing twice is an error
    p = O.Pool(300, NOPART)
    t = [p.alloc(100, 1)[1]["tensor_id"] for _ in range(3)]
    p.free(t[0])
    p.free(t[2])
    a, z, o = p.layout()
    assert list(o) == [-1, t[1], -1]
    assert p.free(t[1]) == O.OK
    a, z, o = p.layout()
    assert list(a) == [0] and list(z) == [300] and list(o) == [-1]
    assert p.free(t[1]) == O.BAD_STATE
    assert p.free(99) == O.UNKNOWN_ID


def test_projected_cost_evicted_ancestor():
    # SPEC.md projected_cost: chain a -> b -> c with b evicted and a resident: c(c) =
    # cost(c) + cost(b).  Clock (= sum of executed costs): a 100, b 101, c 201; access(c, 50)
    # -> 251.  d (unevictable) forces a window: b has s = 251 - 201 = 50, c(b) = 1 ->
    # h = 1/50; c has s = 1, h = 100 -> b is evicted, window cost RN(1/50).
    p = O.Pool(30, NOPART)
    a = p.alloc(10, 100, O.OP_UNEVICTABLE)[1]["tensor_id"]
    b = p.alloc(10, 1, 0, -1, [a])[1]["tensor_id"]
    c = p.alloc(10, 100, 0, -1, [b])[1]["tensor_id"]
    assert p.access(c, 50) == O.OK
    st, r, ev = p.alloc(10, 0, O.OP_UNEVICTABLE)
    assert st == O.OK and ev == [b] and r["window_cost"] == 1.0 / 50.0
    assert (r["window_first"], r["window_last"], r["window_span"], r["addr"]) == (1, 1, 10, 10)
    # e: only c is evictable; c(c) = cost(c) + cost(b) = 101 (b is an evicted ancestor,
    # a stops the closure), s = 1 -> h = 101
    st, r, ev = p.alloc(10, 0)
    assert st == O.OK and ev == [c] and r["window_cost"] == 101.0
    assert p.access(b) == O.NEEDS_REMAT


def test_projected_cost_evicted_descendant():
    # p -> q; r unevictable.  Clock: p 7, q 10, r 15; access(p, 100) -> 115.  x forces a
    # window: p has s = 1, c(p) = 7 (q resident) -> 7; q has s = 105, h = 3/105 -> q evicted.
    # y: only p is evictable; c(p) = 7 + cost(q) = 10 (q is an evicted descendant whose
    # recompute needs p), s = 1 -> h = 10
    P = O.Pool(30, NOPART)
    p = P.alloc(10, 7)[1]["tensor_id"]
    q = P.alloc(10, 3, 0, -1, [p])[1]["tensor_id"]
    P.alloc(10, 5, O.OP_UNEVICTABLE)
    assert P.access(p, 100) == O.OK
    st, r, ev = P.alloc(10, 0, O.OP_UNEVICTABLE)
    assert ev == [q] and r["window_cost"] == 3.0 / 105.0
    st, r, ev = P.alloc(10, 0)
    assert ev == [p] and r["window_cost"] == 10.0
    s = P.stats()
    assert s["evictions"] == 2 and s["pressure"] == 2 and s["base_us"] == 15 and s["total_us"] == 15


def test_remat_and_inplace():
    # recomputable in-place (Alg. 1 "addr <- input.addr"): the output takes the input's
    # block; the input becomes non-resident but recomputable (Sec. 3.5)
    P = O.Pool(100, O.F_INPLACE)
    x = P.alloc(40, 5)[1]["tensor_id"]
    st, r, _ = P.alloc(40, 2, O.OP_INPLACE, x, [x])
    y = r["tensor_id"]
    assert st == O.OK and r["addr"] == 0 and P.access(x) == O.NEEDS_REMAT
    s = P.stats()
    assert s["inplace_reuse"] == 1 and s["total_us"] == 7
    st, r, ev = P.remat(x)  # recomputed out of place (R21): the producer runs again
    assert st == O.OK and r["addr"] == 40 and ev == []
    s = P.stats()
    assert s["remat"] == 1 and s["total_us"] == 12 and s["base_us"] == 7
    assert P.remat(x)[0] == O.OK  # already resident: no-op
    assert P.stats()["remat"] == 1
    # copy-on-write (INPLACE flag off): a fresh block, the input stays resident
    P = O.Pool(100, 0)
    x = P.alloc(40, 5)[1]["tensor_id"]
    st, r, _ = P.alloc(40, 2, O.OP_INPLACE, x, [x])
    assert r["addr"] == 40 and P.access(x) == O.OK
    del y


def test_remat_needs_parent():
    P = O.Pool(30, NOPART)
    a = P.alloc(10, 1)[1]["tensor_id"]
    b = P.alloc(10, 1, 0, -1, [a])[1]["tensor_id"]
    P.free(a)                                       # free: [0,10), [20,30)
    assert P.access(a) == O.BAD_STATE
    assert P.alloc(10, 0, O.OP_UNEVICTABLE)[1]["addr"] == 0
    assert P.alloc(10, 0, O.OP_UNEVICTABLE)[1]["addr"] == 20
    st, r, ev = P.alloc(10, 0, O.OP_UNEVICTABLE)  # pressure: b is the only candidate
    assert st == O.OK and ev == [b] and r["addr"] == 10
    st, r, _ = P.remat(b)
    assert st == O.NEEDS_REMAT and r["tensor_id"] == a  # a was freed: recompute it first
    st, r, _ = P.remat(a)  # allowed (R44), but the pool holds only unevictable tensors
    assert st == O.UNSATISFIABLE


def test_error_statuses():
    P = O.Pool(100, 3, max_tensors=3, max_edges=2)
    assert P.alloc(0, 1)[0] == O.INVALID_ARG
    assert P.alloc(1 << 48, 1)[0] == O.INVALID_ARG
    assert P.alloc(1, 1 << 40)[0] == O.INVALID_ARG
    assert P.alloc(1, 1, 32)[0] == O.INVALID_ARG
    assert P.alloc(1, 1, O.OP_CHEAP | O.OP_EXPENSIVE)[0] == O.INVALID_ARG
    assert P.alloc(1, 1, 0, -1, [0])[0] == O.UNKNOWN_ID
    a = P.alloc(10, 1)[1]["tensor_id"]
    assert P.alloc(10, 1, 0, a, [a])[0] == O.INVALID_ARG           # src without INPLACE
    assert P.alloc(11, 1, O.OP_INPLACE, a, [a])[0] == O.INVALID_ARG  # size mismatch
    assert P.alloc(10, 1, O.OP_INPLACE, a, [])[0] == O.INVALID_ARG   # src not a parent
    assert P.alloc(10, 1, 0, -1, [a, a, a])[0] == O.NOMEM          # edge capacity
    P.alloc(10, 1)
    P.alloc(10, 1)
    assert P.alloc(10, 1)[0] == O.NOMEM                             # tensor capacity
    assert P.access(5) == O.UNKNOWN_ID and P.remat(-1)[0] == O.UNKNOWN_ID
    assert P.access(a, 1 << 40) == O.INVALID_ARG


@pytest.mark.parametrize("flags", [0, 1, 2, 3, 7])
def test_random_sessions_vs_model(flags):
    for seed in range(12):
        budget = 150 + (seed * 37) % 400
        calls = PM.random_session(1000 * flags + seed, 120, budget=budget, flags=flags)
        m = PM.OnlineModel(budget, flags)
        o = O.Pool(budget, flags)
        assert PM.drive(o, calls) == PM.drive(m, calls), (flags, seed)
        s = o.stats()
        for k, v in m.c.items():
            assert s[k].item() == v, (flags, seed, k)
        a, z, ow = o.layout()
        assert [(int(x), int(y), int(w)) for x, y, w in zip(a, z, ow)] == m.layout()


def test_dtr_dte_worked_example():
    """SPEC.md:390-402 (hand-derived): layout a[0,10) x[10,20) free[20,30) b[30,40) c[40,50),
    x and c unevictable, a and b with equal c, m, s.  A 20-byte request: DTR ties a and b
    (lowest address first) and needs both (evicting a alone frees no 20-byte block); DTE's
    denominator counts b's free neighbour (m + 10), so it evicts b alone."""
    for pol, want in ((O.F_DTR, [0, 3]), (O.F_DTE, [3])):
        P = O.Pool(50, pol)
        a = P.alloc(10, 100)[1]["tensor_id"]
        P.alloc(10, 100, O.OP_UNEVICTABLE)
        f = P.alloc(10, 100)[1]["tensor_id"]
        b = P.alloc(10, 100)[1]["tensor_id"]
        P.alloc(10, 100, O.OP_UNEVICTABLE)
        assert P.free(f) == O.OK
        assert P.access(a, 7) == O.OK and P.access(b, 0) == O.OK  # equal staleness
        st, r, ev = P.alloc(20, 1)
        assert st == O.OK and ev == want and r["window_first"] == -1
        assert r["addr"] == 20 and (a, b) == (0, 3)  # first fit: [0,10) is too small


@pytest.mark.parametrize("flags", [8, 16, 11, 19])
def test_random_sessions_vs_model_baselines(flags):
    for seed in range(6):
        budget = 150 + (seed * 41) % 400
        calls = PM.random_session(5000 + 100 * flags + seed, 100, budget=budget, flags=flags)
        m = PM.OnlineModel(budget, flags)
        o = O.Pool(budget, flags)
        assert PM.drive(o, calls) == PM.drive(m, calls), (flags, seed)
        s = o.stats()
        for k, v in m.c.items():
            assert s[k].item() == v, (flags, seed, k)
