"""GPU parity: coop_window_search_batched (CUDA, through the C ABI) vs the O1 oracle,
element by element, bit-exact on every field (first, last, span, cost bits, n_evict,
status).  The north-star tolerance for costs (1e-9 relative) is met with margin: the
CUDA path returns the same correctly rounded value as the oracle (R3)."""
import json
import os

import numpy as np
import pytest

from gen import pools as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_2311_00591_b200 import coop  # noqa: E402

DEV = torch.device("cuda:0")
GOLD = os.path.join(os.path.dirname(__file__), "golden", "window_golden.json")


def gpu_search(ss, c, s, req, n_pools, n, stride):
    d_ss = torch.from_numpy(np.ascontiguousarray(ss).view(np.int64)).to(DEV)
    d_c = torch.from_numpy(np.ascontiguousarray(c)).to(DEV)
    d_s = torch.from_numpy(np.ascontiguousarray(s)).to(DEV)
    d_r = torch.from_numpy(np.ascontiguousarray(req, np.uint64).view(np.int64)).to(DEV)
    out = torch.full((n_pools * 4,), -7, dtype=torch.int64, device=DEV)
    coop.window_search_batched(d_ss, d_c, d_s, d_r, out, n_pools, n, stride)
    torch.cuda.synchronize()
    return coop.windows_from_device(out)


def assert_same(g, o, ctx=""):
    assert len(g) == len(o)
    for f in ("status", "first", "last", "span", "n_evict"):
        bad = np.nonzero(g[f] != o[f])[0]
        assert bad.size == 0, f"{ctx} field {f} differs at pools {bad[:10]}: gpu {g[bad[:3]]} oracle {o[bad[:3]]}"
    gb = g["cost"].view(np.uint64)
    ob = o["cost"].view(np.uint64)
    bad = np.nonzero(gb != ob)[0]
    assert bad.size == 0, f"{ctx} cost bits differ at {bad[:10]}: {g['cost'][bad[:3]]} vs {o['cost'][bad[:3]]}"


def test_golden_cases_gpu():
    d = json.load(open(GOLD))
    for case in d["cases"]:
        st = [{"F": 0, "E": 1, "P": 2}[x[0]] for x in case["items"]]
        ss = G.pack([x[3] for x in case["items"]], st)
        c = np.array([x[1] for x in case["items"]], np.float64)
        s = np.array([x[2] for x in case["items"]], np.float64)
        n = len(ss)
        g = gpu_search(ss, c, s, [case["request"]], 1, n, n)
        o = O.search_many(ss, c, s, [case["request"]], 1, n, n)
        assert_same(g, o, case["name"])
        assert int(g["first"][0]) == case["expect"]["first"]


def test_config1_small_pools_100k():
    """BASELINE config 1: 32-block pools, random int sizes, fp64 costs; 10^5 seeds."""
    P, n = 100_000, 32
    ss, c, s, r = G.bench_pools_host(G.MODE_SMALL, 1234, 0, P, n)
    g = gpu_search(ss, c, s, r, P, n, n)
    o = O.search_many(ss, c, s, r, P, n, n)
    assert_same(g, o, "config1")
    assert (o["status"] == O.OK).sum() > P // 2 and (o["status"] == O.INFEASIBLE).sum() > 0


def test_device_generator_matches_host():
    for mode, n, P in ((G.MODE_SMALL, 32, 5000), (G.MODE_BENCH, 4096, 64), (G.MODE_BENCH, 100, 300)):
        stride = (n + 15) // 16 * 16
        ss, c, s, r = G.bench_pools_host(mode, 77, 1000, P, n, stride)
        d = [torch.zeros(P * stride, dtype=torch.int64, device=DEV),
             torch.zeros(P * stride, dtype=torch.float64, device=DEV),
             torch.ones(P * stride, dtype=torch.float64, device=DEV),
             torch.zeros(P, dtype=torch.int64, device=DEV)]
        G.bench_pools_device(mode, 77, 1000, P, n, stride, *d)
        torch.cuda.synchronize()
        assert np.array_equal(d[0].cpu().numpy().view(np.uint64), ss)
        assert np.array_equal(d[1].cpu().numpy().view(np.uint64), c.view(np.uint64))
        assert np.array_equal(d[2].cpu().numpy().view(np.uint64), s.view(np.uint64))
        assert np.array_equal(d[3].cpu().numpy().view(np.uint64), r)


NS = [1, 2, 7, 16, 31, 32, 33, 100, 511, 512, 513, 1000, 2047, 4095, 4096, 4097, 6000, 8192]


@pytest.mark.parametrize("n", NS)
@pytest.mark.parametrize("layout", ["tma", "plain"])
def test_random_pools_parity(n, layout):
    rng = np.random.default_rng(n * 7 + (layout == "plain"))
    P = max(8, min(400, 40000 // n))
    pools, reqs = [], []
    for p in range(P):
        kind = p % 4
        if kind == 0:    # ties: h from a small set of dyadic values
            pool = G.random_pool(rng, n, p_free=0.15, p_pinned=0.03, max_size=64,
                                 h_choices=[0.0, 0.5, 1.0, 2.0, 0.25])
        elif kind == 1:  # generic real-valued costs, large sizes
            pool = G.random_pool(rng, n, p_free=0.12, p_pinned=0.01, max_size=1 << 30)
        elif kind == 2:  # uncoalesced free runs, pinned-heavy
            pool = G.random_pool(rng, n, p_free=0.3, p_pinned=0.1, max_size=1000,
                                 coalesced=False)
        else:            # wide dynamic range of h (cancellation-prone)
            pool = G.random_pool(rng, n, p_free=0.05, p_pinned=0.0, max_size=100,
                                 h_choices=[1e6, 1e-3, 3e-3, 2.0 ** -60, 7.0, 1e12])
        pools.append(pool)
        tot = int((pool[0] & np.uint64((1 << 62) - 1)).sum())
        reqs.append(int(rng.integers(1, max(2, tot // int(rng.choice([1, 3, 10, 100])) + 2))))
    stride = (n + 15) // 16 * 16 if layout == "tma" else n + 3
    ss, c, s = G.stack_pools(pools, stride)
    req = np.array(reqs, np.uint64)
    g = gpu_search(ss, c, s, req, P, n, stride)
    o = O.search_many(ss, c, s, req, P, n, stride)
    assert_same(g, o, f"n={n} {layout}")


def test_forced_plain_staging_same_bits(monkeypatch):
    ss, c, s, r = G.bench_pools_host(G.MODE_BENCH, 5, 0, 256, 4096)
    g1 = gpu_search(ss, c, s, r, 256, 4096, 4096)
    monkeypatch.setenv("COOP_FORCE_PLAIN_STAGING", "1")
    g2 = gpu_search(ss, c, s, r, 256, 4096, 4096)
    assert g1.tobytes() == g2.tobytes()


def test_candidate_overflow_all_equal():
    """Every start ties (equal sizes, equal h): > 1024 exact candidates -> several rounds."""
    n = 4096
    ss = G.pack([8] * n, [G.EVICTABLE] * n)
    c = np.full(n, 0.1)
    s = np.ones(n)
    req = np.array([80, 8, 8 * 4000, 8 * 4096, 8 * 4096 + 1], np.uint64)
    P = len(req)
    SS, C, S = G.stack_pools([(ss, c, s)] * P)
    g = gpu_search(SS, C, S, req, P, n, n)
    o = O.search_many(SS, C, S, req, P, n, n)
    assert_same(g, o, "overflow")
    assert list(g["first"][:4]) == [0, 0, 0, 0] and int(g["status"][4]) == O.INFEASIBLE


def test_cancellation_pool_gpu():
    hs = [1e6] * 2000 + [1e-3, 2e-3, 1e-3] + [1e6] * 2000
    n = len(hs)
    ss = G.pack([1] * n, [G.EVICTABLE] * n)
    g = gpu_search(ss, np.array(hs), np.ones(n), [3], 1, n, n)
    o = O.search_many(ss, np.array(hs), np.ones(n), [3], 1, n, n)
    assert_same(g, o, "G5")
    assert int(g["first"][0]) == 2000


def test_invalid_pools_per_element():
    n = 64
    rng = np.random.default_rng(1)
    pools = [G.random_pool(rng, n) for _ in range(6)]
    pools[1][0][5] = G.pack([0], [1])[0]                  # size 0
    pools[2][1][7] = -1.0; pools[2][0][7] = G.pack([3], [1])[0]  # negative cost (evictable)
    pools[3][2][9] = 0.5; pools[3][0][9] = G.pack([3], [1])[0]   # staleness < 1
    pools[4][0][3] = G.pack([4], [3])[0]                  # bad state
    ss, c, s = G.stack_pools(pools, 64)
    req = np.array([10, 10, 10, 10, 10, 0], np.uint64)  # pool 5: R = 0
    g = gpu_search(ss, c, s, req, 6, n, 64)
    o = O.search_many(ss, c, s, req, 6, n, 64)
    assert_same(g, o, "invalid")
    assert list(g["status"][1:]) == [-1] * 5


def test_bench_pools_4096_full_parity():
    """config-4 generator at N = 4096 (2048 pools): every pool vs the oracle."""
    P, n = 2048, 4096
    ss, c, s, r = G.bench_pools_host(G.MODE_BENCH, 0, 0, P, n)
    g = gpu_search(ss, c, s, r, P, n, n)
    o = O.search_many(ss, c, s, r, P, n, n)
    assert_same(g, o, "bench4096")
    assert (o["status"] == O.INFEASIBLE).sum() >= P // 64


def test_host_entry_point_matches_device():
    P, n = 3000, 4096
    ss, c, s, r = G.bench_pools_host(G.MODE_BENCH, 3, 0, P, n)
    g = gpu_search(ss, c, s, r, P, n, n)
    h = coop.window_search_batched_host(ss, c, s, r, P, n, n, chunk_pools=700)
    assert g.tobytes() == h.tobytes()
    # ragged host stride (re-pitched by the library)
    st = n + 5
    ss2 = np.zeros(P * st, np.uint64); c2 = np.zeros(P * st); s2 = np.ones(P * st)
    for a, b in ((ss2, ss), (c2, c), (s2, s)):
        a.reshape(P, st)[:, :n] = b.reshape(P, n)
    h2 = coop.window_search_batched_host(ss2, c2, s2, r, P, n, st, chunk_pools=1024)
    assert g.tobytes() == h2.tobytes()


def test_config4_full_size_sampled():
    """BASELINE config 4 at full size (2^20 pools x 4096 blocks, generated on device, the
    launch configuration bench.py times); 512 sampled pools checked against the oracle."""
    P, n = 1 << 20, 4096
    free, _ = torch.cuda.mem_get_info()
    need = P * n * 24 + P * 40
    if free < need + (2 << 30):
        pytest.skip(f"needs {need / 2**30:.0f} GiB free device memory")
    ss = torch.empty(P * n, dtype=torch.int64, device=DEV)
    c = torch.empty(P * n, dtype=torch.float64, device=DEV)
    s = torch.empty(P * n, dtype=torch.float64, device=DEV)
    r = torch.empty(P, dtype=torch.int64, device=DEV)
    out = torch.empty(P * 4, dtype=torch.int64, device=DEV)
    G.bench_pools_device(G.MODE_BENCH, 0, 0, P, n, n, ss, c, s, r)
    coop.window_search_batched(ss, c, s, r, out, P, n, n)
    torch.cuda.synchronize()
    g = coop.windows_from_device(out)
    del ss, c, s, r, out
    rng = np.random.default_rng(0)
    sample = np.unique(np.concatenate([rng.integers(0, P, 500), [63, 127, P - 1, 0]]))
    for p in sample:
        hs, hc, hst, hr = G.bench_pools_host(G.MODE_BENCH, 0, int(p), 1, n)
        o = O.search_many(hs, hc, hst, hr, 1, n, n)
        assert_same(g[p:p + 1], o, f"pool {p}")


def test_signed_zero_and_zero_runs():
    """c = -0.0 EVICTABLE items (valid, h = 0, counted as evictions), multi-item zero runs
    crossing thread chunks, and +0.0 window costs."""
    rng = np.random.default_rng(4)
    pools, reqs = [], []
    n = 600
    for p in range(64):
        ss, c, s = G.random_pool(rng, n, p_free=0.2, p_pinned=0.02, max_size=50,
                                 h_choices=[0.0, 0.0, 1.0, 2.0], coalesced=False)
        c = np.where((rng.random(n) < 0.3) & (c == 0.0), -0.0, c)
        pools.append((ss, c, s))
        reqs.append(int(rng.integers(1, 400)))
    SS, C, S = G.stack_pools(pools, 608)
    req = np.array(reqs, np.uint64)
    g = gpu_search(SS, C, S, req, 64, n, 608)
    o = O.search_many(SS, C, S, req, 64, n, 608)
    assert_same(g, o, "signed zero")
    assert (g["cost"][g["status"] == 0] == 0.0).sum() > 10


@pytest.mark.parametrize("n", [1, 31, 32, 129, 1000, 4096, 8192])
def test_stream_kernel_parity(n, monkeypatch):
    """The alternative warp-per-pool streaming kernel (COOP_SEARCH_IMPL=stream, DESIGN.md
    section 6) plus the CTA kernel on the pools it leaves pending: bit-identical to O1 on the
    same random pools (ties, cancellation, uncoalesced free runs, windows longer than its
    history ring), and on the benchmark law."""
    monkeypatch.setenv("COOP_SEARCH_IMPL", "stream")
    test_random_pools_parity(n, "tma")
    if n == 4096:
        P = 256
        ss, c, s, r = G.bench_pools_host(G.MODE_BENCH, 3, 5000, P, n)
        assert_same(gpu_search(ss, c, s, r, P, n, n), O.search_many(ss, c, s, r, P, n, n), "stream bench law")


def _edge_values():
    """(c, s) pairs on and around every R7 boundary: c = +-0, subnormal c, h underflowing
    to 0 (valid zero item), h = 2^-64 exactly and one ulp below, h just below / at 2^60,
    huge s, non-finite or negative c, s < 1, plus random pairs straddling both h bounds."""
    nb = np.nextafter
    v = [(0.0, 1.0), (-0.0, 1.0), (-0.0, 0.5), (0.0, np.nan), (0.0, np.inf),
         (5e-324, 1.0), (5e-324, 3.0), (1e-300, 1e300), (2.0 ** -64, 1.0),
         (nb(2.0 ** -64, 0.0), 1.0), (2.0 ** -63, 2.0), (nb(2.0 ** -63, 0.0), 2.0),
         (1.5 * 2.0 ** -64, 1.5), (2.0 ** 60, 1.0), (nb(2.0 ** 60, 0.0), 1.0), (2.0 ** 61, 2.0),
         (1.0, 2.0 ** 1000), (2.0 ** 1000, 2.0 ** 1022), (2.0 ** 1023, 1.5), (np.inf, 1.0),
         (np.nan, 1.0), (-1.0, 1.0), (1.0, 0.999), (1.0, -1.0), (1.0, 5e-324),
         (2.0 ** -1022, 1.0), (3.0, 3.0)]
    rng = np.random.default_rng(17)
    for _ in range(24):
        v.append((float(2.0 ** rng.uniform(-70, -58)), float(rng.uniform(1, 4))))
        v.append((float(2.0 ** rng.uniform(55, 63)), float(rng.uniform(1, 8))))
    return v


@pytest.mark.parametrize("n", [64, 4096])
def test_r7_domain_edges(n):
    """Validation (R7) and zero-ness of h decided without a division where the exponents
    allow and exactly elsewhere: bit-identical to O1 on every edge value, at several item
    positions (chunk starts / ends), as a lone large item (zero window iff h == 0), and with
    garbage c / s on FREE and PINNED items (ignored)."""
    rng = np.random.default_rng(n)
    pools, reqs = [], []
    for ci, (cv, sv) in enumerate(_edge_values()):
        for pos in (0, 7, 8, 15, n // 2 + 3, n - 1):
            ss, c, s = G.random_pool(rng, n, p_free=0.0, p_pinned=0.02, max_size=64)
            sizes = ss & np.uint64((1 << 62) - 1)
            sizes[pos] = 1 << 20
            states = np.where((ss >> np.uint64(62)) == 2, 2, 1)
            states[pos] = 1
            ss = G.pack(sizes, states)
            c[pos], s[pos] = cv, sv
            # garbage on non-evictable items must be ignored
            j = (pos + 5) % n
            ss[j] = G.pack([3], [ci % 2 * 2])[0]
            c[j], s[j] = (np.nan, -1.0) if ci % 3 else (-5.0, 0.25)
            pools.append((ss, c, s))
            reqs.append((1 << 20) if ci % 2 else int(rng.integers(1, 200)))
    SS, C, S = G.stack_pools(pools, n)
    req = np.array(reqs, np.uint64)
    g = gpu_search(SS, C, S, req, len(pools), n, n)
    o = O.search_many(SS, C, S, req, len(pools), n, n)
    assert_same(g, o, f"R7 edges n={n}")
    st = o["status"]
    assert (st == O.INVALID_ARG).sum() > 20 and (st == O.OK).sum() > 20
    assert ((st == O.OK) & (o["cost"] == 0.0) & (o["span"] >= (1 << 20))).sum() > 5  # underflow zeros
