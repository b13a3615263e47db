"""Pins for the O1 oracle (oracle/oracle_search.c): it is checked against things other
than itself -- the literal Eq. 1 over all 2^N eviction sets, an O(N^2)
enumeration of all windows with exact rational sums (fractions.Fraction) and with
math.fsum, worked examples (SPEC.md:416-417 and hand-derived cases in tests/golden/),
closed forms (first-fit, fixed-length minimum subarray), and invariants.
"""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from gen import pools as G
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "window_golden.json")
ST = {"F": G.FREE, "E": G.EVICTABLE, "P": G.PINNED}


def items_to_arrays(items):
    states = [ST[s] for s, _, _, _ in items]
    sizes = [z for _, _, _, z in items]
    return (G.pack(sizes, states), np.array([c for _, c, _, _ in items], np.float64),
            np.array([s for _, _, s, _ in items], np.float64))


def decode(ss, c, s):
    st = (ss >> np.uint64(62)).astype(int)
    sz = (ss & np.uint64((1 << 62) - 1)).astype(np.int64)
    h = [0.0 if st[k] != G.EVICTABLE else float(c[k]) / float(s[k]) for k in range(len(ss))]
    return st, sz, h


def brute_windows(ss, c, s, R, exact=True):
    """All contiguous barrier-free windows with span >= R; key (RN(cost), start, length).
    exact=True: cost = float(Fraction sum) (correctly rounded); else math.fsum."""
    st, sz, h = decode(ss, c, s)
    n = len(ss)
    best = None
    for i in range(n):
        for j in range(i, n):
            if any(st[k] == G.PINNED for k in range(i, j + 1)):
                break
            span = int(sum(sz[i:j + 1]))
            if span < R:
                continue
            cost = float(sum((Fraction(x) for x in h[i:j + 1]), Fraction(0))) if exact \
                else math.fsum(h[i:j + 1])
            key = (cost, i, j - i)
            if best is None or key < best[0]:
                nev = sum(1 for k in range(i, j + 1) if st[k] == G.EVICTABLE)
                best = (key, span, nev)
    return best


def eq1_subsets(ss, c, s, R):
    """Literal Eq. 1: min over sets S of EVICTABLE tensors of sum h(S) s.t. the largest
    contiguous free block after evicting S is >= R (M(S, L) >= M_R).  Exact rationals."""
    st, sz, h = decode(ss, c, s)
    ev = [k for k in range(len(ss)) if st[k] == G.EVICTABLE]
    best = None
    for r in range(len(ev) + 1):
        for S in itertools.combinations(ev, r):
            Sset = set(S)
            run = largest = 0
            for k in range(len(ss)):
                if st[k] == G.FREE or k in Sset:
                    run += int(sz[k])
                    largest = max(largest, run)
                else:
                    run = 0
            if largest >= R:
                cost = sum((Fraction(h[k]) for k in S), Fraction(0))
                if best is None or cost < best:
                    best = cost
    return best


def test_golden_cases():
    d = json.load(open(GOLD))
    assert len(d["cases"]) >= 8
    for case in d["cases"]:
        ss, c, s = items_to_arrays(case["items"])
        w = O.search(ss, c, s, case["request"])
        e = case["expect"]
        assert int(w["status"]) == e["status"], case["name"]
        assert int(w["first"]) == e["first"], case["name"]
        assert int(w["last"]) == e["last"], case["name"]
        assert int(w["span"]) == e["span"], case["name"]
        assert int(w["n_evict"]) == e["n_evict"], case["name"]
        assert float(w["cost"]) == float(e["cost"]), case["name"]


def test_cancellation_g5():
    """2000 x h=1e6, three tiny h, 2000 x h=1e6: the answer is the
    correctly rounded exact sum of the three tiny values -- prefix differences fail."""
    n_big = 2000
    hs = [1e6] * n_big + [1e-3, 2e-3, 1e-3] + [1e6] * n_big
    items = [["E", x, 1.0, 1] for x in hs]
    ss, c, s = items_to_arrays(items)
    w = O.search(ss, c, s, 3)
    want = float(Fraction(1e-3) + Fraction(2e-3) + Fraction(1e-3))
    assert (int(w["first"]), int(w["last"]), int(w["span"])) == (2000, 2002, 3)
    assert float(w["cost"]) == want
    pre = np.cumsum(np.array(hs))  # the naive prefix-difference answer differs
    assert pre[2002] - pre[1999] != want


def test_fig2_windows():
    """Fig. 2 scenario with the DESIGN.md readings: x0..x4 50 MiB each,
    request 100 MiB; costs from Table 1 densities x 50 MiB."""
    MiB = 1 << 20
    # with cheap tensor partitioning: layout x1 x3 x4(pinned) x2 x0
    items = [["E", 1780.0, 1975.0, 50 * MiB], ["E", 1780.0, 1.0, 50 * MiB],
             ["P", 0.0, 1.0, 50 * MiB], ["E", 195.0, 195.0, 50 * MiB],
             ["E", 195.0, 2170.0, 50 * MiB]]
    ss, c, s = items_to_arrays(items)
    w = O.search(ss, c, s, 100 * MiB)
    assert (int(w["first"]), int(w["last"])) == (3, 4)
    assert float(w["cost"]) == float(Fraction(195.0 / 195.0) + Fraction(195.0 / 2170.0))
    # without partitioning: x0 x1 x2 x3 x4(pinned)
    items = [["E", 195.0, 2170.0, 50 * MiB], ["E", 1780.0, 1975.0, 50 * MiB],
             ["E", 195.0, 195.0, 50 * MiB], ["E", 1780.0, 1.0, 50 * MiB],
             ["P", 0.0, 1.0, 50 * MiB]]
    ss, c, s = items_to_arrays(items)
    w = O.search(ss, c, s, 100 * MiB)
    assert (int(w["first"]), int(w["last"])) == (0, 1)
    assert float(w["cost"]).hex() == "0x1.fb7512c8720acp-1"


@pytest.mark.parametrize("seed", range(6))
def test_vs_eq1_subsets(seed):
    """The literal Eq. 1 over all 2^N sets has the same optimum cost (N <= 10)."""
    rng = np.random.default_rng(1000 + seed)
    for _ in range(150):
        n = int(rng.integers(1, 11))
        ss, c, s = G.random_pool(rng, n, p_free=0.2, p_pinned=0.12, max_size=64,
                                 h_choices=[0.0, 0.5, 1.0, 2.0, 3.0, 0.375])
        R = int(rng.integers(1, 121))
        w = O.search(ss, c, s, R)
        best = eq1_subsets(ss, c, s, R)
        if best is None:
            assert int(w["status"]) == O.INFEASIBLE
        else:
            assert int(w["status"]) == O.OK
            assert float(w["cost"]) == float(best)


@pytest.mark.parametrize("seed", range(8))
def test_vs_bruteforce_windows(seed):
    """O(N^2) window enumeration with exact Fractions: every field equal, incl. ties."""
    rng = np.random.default_rng(seed)
    for _ in range(250):
        n = int(rng.integers(1, 13))
        hc = None if rng.random() < 0.4 else [0.0, 0.5, 1.0, 2.0, 0.25, 1e-3, 3e-3]
        ss, c, s = G.random_pool(rng, n, p_free=0.15, p_pinned=0.1, max_size=64, h_choices=hc,
                                 coalesced=bool(rng.random() < 0.7))
        R = int(rng.integers(1, 200))
        w = O.search(ss, c, s, R)
        b = brute_windows(ss, c, s, R, exact=bool(rng.random() < 0.5))
        if b is None:
            assert int(w["status"]) == O.INFEASIBLE and int(w["first"]) == -1
            continue
        (cost, i, ln), span, nev = b
        assert (int(w["status"]), int(w["first"]), int(w["last"])) == (O.OK, i, i + ln)
        assert float(w["cost"]) == cost and int(w["span"]) == span and int(w["n_evict"]) == nev


def test_first_fit_closed_form():
    """Coalesced pool, every tensor h > 0, some FREE item >= R: the window is the first
    FREE item >= R at cost 0 (the conventional first-fit)."""
    rng = np.random.default_rng(7)
    hits = 0
    for _ in range(400):
        n = int(rng.integers(2, 40))
        ss, c, s = G.random_pool(rng, n, p_free=0.3, p_pinned=0.05, max_size=100,
                                 h_choices=[0.5, 1.0, 7.0])
        R = int(rng.integers(1, 100))
        st, sz, _ = decode(ss, c, s)
        fits = [k for k in range(n) if st[k] == G.FREE and sz[k] >= R]
        if not fits:
            continue
        hits += 1
        w = O.search(ss, c, s, R)
        assert (int(w["first"]), int(w["last"]), float(w["cost"]), int(w["n_evict"])) == \
            (fits[0], fits[0], 0.0, 0)
    assert hits > 100


def test_fixed_length_convolution_closed_form():
    """No FREE/PINNED items, equal sizes m: every window has k = ceil(R/m) items, so the
    answer is the first minimum of the length-k moving sum (np.convolve, exact ints)."""
    rng = np.random.default_rng(11)
    for _ in range(300):
        n = int(rng.integers(1, 60))
        m = int(rng.integers(1, 50))
        h = rng.integers(0, 20, n).astype(np.float64)
        ss = G.pack([m] * n, [G.EVICTABLE] * n)
        R = int(rng.integers(1, m * n + 1))
        k = -(-R // m)
        w = O.search(ss, h, np.ones(n), R)
        sums = np.convolve(h, np.ones(k), "valid")
        i = int(np.argmin(sums))
        assert (int(w["first"]), int(w["last"]), float(w["cost"])) == (i, i + k - 1, sums[i])


def test_scaling_by_power_of_two():
    """Multiplying every h by 2^e keeps the window and scales the cost exactly."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        n = int(rng.integers(1, 50))
        ss, c, s = G.random_pool(rng, n, max_size=30)
        R = int(rng.integers(1, 300))
        w0 = O.search(ss, c, s, R)
        e = int(rng.integers(-20, 20))
        w1 = O.search(ss, c * 2.0 ** e, s, R)
        assert (int(w0["first"]), int(w0["last"]), int(w0["status"])) == \
            (int(w1["first"]), int(w1["last"]), int(w1["status"]))
        if int(w0["status"]) == O.OK:
            assert float(w1["cost"]) == float(w0["cost"]) * 2.0 ** e


def test_degenerate_cases():
    # N = 1
    w = O.search(G.pack([5], [G.EVICTABLE]), [2.0], [4.0], 5)
    assert (int(w["status"]), int(w["first"]), float(w["cost"])) == (O.OK, 0, 0.5)
    w = O.search(G.pack([5], [G.EVICTABLE]), [2.0], [4.0], 6)
    assert int(w["status"]) == O.INFEASIBLE
    # all pinned
    w = O.search(G.pack([5, 5, 5], [G.PINNED] * 3), [1.0] * 3, [1.0] * 3, 1)
    assert int(w["status"]) == O.INFEASIBLE
    # invalid inputs
    bad = [
        (G.pack([0], [G.EVICTABLE]), [1.0], [1.0], 1),       # size 0
        (G.pack([1 << 48], [G.EVICTABLE]), [1.0], [1.0], 1),  # size >= 2^48
        (G.pack([1], [3]), [1.0], [1.0], 1),                  # bad state
        (G.pack([1], [G.EVICTABLE]), [-1.0], [1.0], 1),       # c < 0
        (G.pack([1], [G.EVICTABLE]), [1.0], [0.5], 1),        # s < 1
        (G.pack([1], [G.EVICTABLE]), [float("nan")], [1.0], 1),
        (G.pack([1], [G.EVICTABLE]), [1e-30], [1.0], 1),      # h below 2^-64
        (G.pack([1], [G.EVICTABLE]), [2.0 ** 61], [1.0], 1),  # h >= 2^60
        (G.pack([1], [G.EVICTABLE]), [1.0], [1.0], 0),        # R = 0
    ]
    for ss, c, s, R in bad:
        assert int(O.search(ss, c, s, R)["status"]) == O.INVALID_ARG
    # c = -0.0 is a valid (zero) cost; the window cost is +0.0 and the item an eviction
    w = O.search(G.pack([4], [G.EVICTABLE]), [-0.0], [3.0], 4)
    assert (int(w["status"]), int(w["n_evict"])) == (O.OK, 1)
    assert math.copysign(1.0, float(w["cost"])) == 1.0 and float(w["cost"]) == 0.0
    # FREE / PINNED items ignore c and s
    w = O.search(G.pack([3, 3], [G.FREE, G.PINNED]), [float("nan"), -5.0], [0.0, 0.0], 3)
    assert (int(w["status"]), int(w["first"])) == (O.OK, 0)


def test_invariants_random_pools():
    """Contiguity, no barrier, span >= R, minimal end, left FREE neighbour absorbed."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        n = int(rng.integers(1, 300))
        ss, c, s = G.random_pool(rng, n, p_free=0.12, p_pinned=0.03, max_size=1 << 20,
                                 coalesced=bool(rng.random() < 0.5))
        st, sz, _ = decode(ss, c, s)
        R = int(rng.integers(1, 1 << 23))
        w = O.search(ss, c, s, R)
        if int(w["status"]) != O.OK:
            continue
        i, j = int(w["first"]), int(w["last"])
        assert all(st[k] != G.PINNED for k in range(i, j + 1))
        assert int(w["span"]) == int(sz[i:j + 1].sum()) >= R
        assert int(sz[i:j].sum()) < R
        assert i == 0 or st[i - 1] != G.FREE


def test_fsum_matches_math_fsum():
    rng = np.random.default_rng(9)
    for _ in range(2000):
        k = int(rng.integers(0, 40))
        x = rng.random(k) * 10.0 ** rng.integers(-20, 18, k)
        if rng.random() < 0.3:  # exact midpoints and heavy cancellation between magnitudes
            x = np.concatenate([x, [2.0 ** 60, 1.0, 2.0 ** -53 * 2.0 ** 60]])
        assert O.fsum(x) == math.fsum(x)
    for x in ([-0.0], [-0.0, -0.0], [0.0, -0.0], []):  # signed zeros: +0.0, bitwise
        assert math.copysign(1.0, O.fsum(x)) == math.copysign(1.0, math.fsum(x)) == 1.0
