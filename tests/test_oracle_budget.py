"""Pins of the oracle O4 (minimum / cutoff budget searches, R45) -- CPU only:
the grid procedure re-run with the independent Python replay model (tests/replay_model.py)
on tiny traces, and the defining properties of the results (the metric holds at the result;
the grid point below it fails)."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from gen import traces as TR  # noqa: E402
from oracle import oracle as O  # noqa: E402
import replay_model as RM  # noqa: E402


def grid(lo, hi, j, steps):
    return max(1, lo + (hi - lo) * j // steps)


def model_meets(tr, budget, flags, metric):
    m = RM.Model(tr, budget, flags)
    st, _ = m.run()
    return st == 0 and (metric == 0 or m.c["evictions"] == 0)


def model_search(tr, flags, kc, kf):
    """R45 with brackets (0, P], (P, 2P], ... up to Z = the bytes of all tensors"""
    peak = O.peak_live(tr, flags)
    z = max(peak, int(sum(int(x) for x in tr.size)))
    out = []
    for metric in (0, 1):
        blo, bhi = 0, max(peak, 1)
        while True:
            ks = [k for k in range(1, kc + 1) if model_meets(tr, grid(blo, bhi, k, kc), flags, metric)]
            if ks or bhi >= z:
                break
            blo, bhi = bhi, 2 * bhi
        if not ks:
            out.append((1, 0))
            continue
        k = ks[0]
        lo, hi = (grid(blo, bhi, k - 1, kc) if k > 1 else blo), grid(blo, bhi, k, kc)
        b = hi
        for j in range(1, kf + 1):
            if model_meets(tr, grid(lo, hi, j, kf), flags, metric):
                b = grid(lo, hi, j, kf)
                break
        out.append((0, b))
    return peak, out


@pytest.mark.parametrize("seed", range(6))
def test_budget_search_vs_model(seed):
    rng = np.random.default_rng(seed)
    tr = TR.random_trace(rng, n_fwd=6 + seed % 3, iters=1 + seed % 2)
    for flags in (0, 3):
        o = O.budget_search(tr, flags, coarse=8, fine=6)
        peak, ((mst, mb), (cst, cb)) = model_search(tr, flags, 8, 6)
        assert int(o["peak"]) == peak
        assert (int(o["min_status"]), int(o["min_budget"])) == (mst, mb), (seed, flags)
        assert (int(o["cutoff_status"]), int(o["cutoff_budget"])) == (cst, cb), (seed, flags)


def test_budget_properties_fig2():
    tr = TR.fig2_trace()
    flags = O.F_PARTITION | O.F_INPLACE
    o = O.budget_search(tr, flags, coarse=32, fine=32)
    peak = int(o["peak"])
    assert o["min_status"] == 0 and o["cutoff_status"] == 0
    mb, cb = int(o["min_budget"]), int(o["cutoff_budget"])
    assert 0 < mb <= cb <= peak
    r, _ = O.replay(tr, mb, flags)
    assert r["status"] == 0
    r, _ = O.replay(tr, cb, flags)
    assert r["status"] == 0 and r["evictions"] == 0
    # the grid point just below each result fails its metric
    for b, metric in ((mb, 0), (cb, 1)):
        k = next(k for k in range(1, 33) if grid(0, peak, k, 32) >= b)
        lo, hi = (grid(0, peak, k - 1, 32) if k > 1 else 0), grid(0, peak, k, 32)
        js = [j for j in range(1, 33) if grid(lo, hi, j, 32) == b]
        below = grid(lo, hi, js[0] - 1, 32) if js[0] > 1 else lo
        if below >= 1:
            r, _ = O.replay(tr, below, flags)
            assert not (r["status"] == 0 and (metric == 0 or r["evictions"] == 0))
    # the largest tensor plus the unevictable bytes bound the minimum budget from below
    assert mb >= int(max(tr.size))


def test_cutoff_above_peak_bracket():
    """Fragmentation can force evictions at the peak itself (R25 is a resident-bytes peak,
    not an address high-water mark); the cutoff is then found in the bracket (P, 2P]
    (R45): zero evictions at the result, evictions at P."""
    rng = np.random.default_rng(0)
    tr = TR.random_trace(rng, n_fwd=6, iters=1)
    o = O.budget_search(tr, 0, coarse=8, fine=6)
    peak, cb = int(o["peak"]), int(o["cutoff_budget"])
    assert o["cutoff_status"] == 0 and peak < cb <= 2 * peak
    r, _ = O.replay(tr, peak, 0)
    assert r["status"] == 0 and r["evictions"] > 0
    r, _ = O.replay(tr, cb, 0)
    assert r["status"] == 0 and r["evictions"] == 0
    # a pool of all tensors' bytes never evicts (the bracket bound Z)
    z = int(sum(int(x) for x in tr.size))
    r, _ = O.replay(tr, z, 0)
    assert r["status"] == 0 and r["evictions"] == 0
