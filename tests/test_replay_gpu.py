"""GPU parity: coop_replay_trace (one CTA per budget, through the C ABI) vs the O2 oracle.
Bit-exact on every integer counter, the eviction digest, and the full event log."""
import numpy as np
import pytest

from gen import dnn
from gen import traces as TR
from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_2311_00591_b200 import coop  # noqa: E402

FIELDS = ["status", "fail_op", "base_us", "total_us", "evictions", "remat", "pressure",
          "frag_fail", "inplace_reuse", "heuristic_evals", "sum_free_bytes_after",
          "sum_free_blocks_after", "digest", "max_depth", "max_blocks", "budget", "n_events"]
ALL_FLAGS = [0, 1, 2, 3, 7]


def check(tr, budgets, flags, log_cap=0, ctx=""):
    t = coop.Trace(tr)
    res, ev = t.replay(budgets, flags, log_cap=log_cap)
    for j, b in enumerate(budgets):
        r, log = O.replay(tr, int(b), flags, log_cap=log_cap)
        got = {f: int(res[j][f]) for f in FIELDS}
        want = {f: int(r[f]) for f in FIELDS}
        assert got == want, f"{ctx} budget {b} flags {flags}: gpu {got} oracle {want}"
        if log_cap:
            m = min(int(r["n_events"]), log_cap)
            g = ev[j][:m]
            for k in ("kind", "op", "tensor", "addr"):
                assert np.array_equal(g[k], log[:m][k]), f"{ctx} budget {b}: event field {k}"
    return res


def test_fig2_gpu():
    tr = TR.fig2_trace()
    for flags in ALL_FLAGS:
        check(tr, [250 << 20, 200 << 20, 300 << 20], flags, log_cap=200, ctx="fig2")


@pytest.mark.parametrize("seed", range(6))
def test_random_traces_gpu(seed):
    rng = np.random.default_rng(500 + seed)
    for _ in range(15):
        tr = TR.random_trace(rng, n_params=int(rng.integers(0, 4)), n_fwd=int(rng.integers(2, 12)),
                             iters=int(rng.integers(1, 3)), inplace_p=0.25)
        flags = int(rng.choice(ALL_FLAGS))
        peak = O.peak_live(tr, flags)
        budgets = [max(1, int(peak * f)) for f in (0.35, 0.5, 0.65, 0.8, 1.0, 1.4)]
        check(tr, budgets, flags, log_cap=4000, ctx=f"seed {seed}")


@pytest.mark.parametrize("name", list(dnn.DNNS))
def test_dnn_traces_gpu(name):
    tr = dnn.dnn(name)
    flags = coop.F_PARTITION | coop.F_INPLACE
    peak = O.peak_live(tr, flags)
    budgets = [int(peak * f) for f in (0.3, 0.45, 0.6, 0.75, 0.9, 1.0)]
    check(tr, budgets, flags, log_cap=20000, ctx=name)


def test_config2_resnet50_half_budget():
    """BASELINE config 2: ResNet-50 replay at 50 % of peak, partitioning + in-place."""
    tr = dnn.resnet50()
    flags = coop.F_PARTITION | coop.F_INPLACE
    res = check(tr, [O.peak_live(tr, flags) // 2], flags, log_cap=50000, ctx="config2")
    assert int(res[0]["status"]) == 0 and int(res[0]["evictions"]) > 0


def test_config3_gpt3_64_budgets():
    """BASELINE config 3: GPT-3-style 2.7B, 64 budgets from 25 % to 100 % of peak."""
    tr = dnn.gpt3_2p7b()
    flags = coop.F_PARTITION | coop.F_INPLACE
    peak = O.peak_live(tr, flags)
    budgets = [peak * (1575 + 75 * k) // 6300 for k in range(64)]
    res = check(tr, budgets, flags, ctx="config3")
    st = res["status"]
    assert (st == 0).sum() > 10 and (st == coop.ERR_UNSATISFIABLE).sum() > 0


def test_ablation_flags_dnn():
    """The same traces without partitioning / with copy-on-write (App. B ablations)."""
    for name in ("unet", "bert_large"):
        tr = dnn.dnn(name)
        for flags in (0, coop.F_INPLACE, coop.F_PARTITION, 7):
            peak = O.peak_live(tr, flags)
            check(tr, [int(peak * 0.6), int(peak * 0.85)], flags, ctx=f"{name} flags {flags}")


@pytest.mark.parametrize("name", ["resnet50", "unet"])
def test_ablation_no_sliding_window_dnn(name):
    """App. B "w/o sliding window": DTE's heuristic loop in place of the
    window search, with partitioning and recomputable in-place kept (NEXT-2)."""
    flags = coop.F_POLICY_DTE | coop.F_PARTITION | coop.F_INPLACE
    tr = dnn.dnn(name)
    peak = O.peak_live(tr, flags & 7)
    check(tr, [int(peak * 0.4), int(peak * 0.6), int(peak * 0.85)], flags, ctx=f"{name} no-window")


@pytest.mark.parametrize("name,ks", [("bilstm", (48, 100, 180, 255)), ("inception_v3", (0, 40, 120)),
                                     ("spos", (0, 64, 200))])
def test_config5_budget_samples(name, ks):
    """BASELINE config 5 budgets (k = 0..255 -> 20..100 % of peak): samples including
    heavily thrashing cells (bilstm k = 48: ~9 K pressure events, projected-cost closures of
    up to ~2.6 K tensors)."""
    tr = dnn.dnn(name)
    flags = O.F_PARTITION | O.F_INPLACE
    peak = O.peak_live(tr, flags)
    budgets = [peak * (20 * 255 + 80 * k) // (100 * 255) for k in ks]
    check(tr, budgets, flags, ctx=f"config5 {name}")


@pytest.mark.parametrize("seed", range(4))
def test_dtr_dte_random_traces_gpu(seed):
    """NEXT-1 baselines (R46) through coop_replay_trace: bit-exact with O2 incl. event logs."""
    rng = np.random.default_rng(900 + seed)
    for _ in range(6):
        tr = TR.random_trace(rng, n_params=int(rng.integers(0, 4)), n_fwd=int(rng.integers(3, 12)),
                             iters=int(rng.integers(1, 3)), inplace_p=0.25)
        for pol in (coop.F_POLICY_DTR, coop.F_POLICY_DTE):
            flags = pol | int(rng.choice([0, 1, 2, 3]))
            peak = O.peak_live(tr, flags & 7)
            budgets = [max(1, int(peak * f)) for f in (0.4, 0.6, 0.8, 1.0)]
            check(tr, budgets, flags, log_cap=4000, ctx=f"seed {seed} pol {pol}")


@pytest.mark.parametrize("name", ["resnet50", "unet", "swin_t"])
def test_dtr_dte_dnn_gpu(name):
    tr = dnn.dnn(name)
    for pol in (coop.F_POLICY_DTR, coop.F_POLICY_DTE):
        peak = O.peak_live(tr, 0)
        budgets = [int(peak * f) for f in (0.5, 0.75, 1.0)]
        check(tr, budgets, pol, ctx=f"{name} pol {pol}")


def test_fig2_dtr_half_gpu():
    """The DTR half of Fig. 2 through coop_replay_trace: x0, x2, then x1."""
    tr = TR.fig2_dtr_trace()
    for flags in (coop.F_POLICY_DTR, coop.F_POLICY_DTE, 0, 3):
        check(tr, [250 << 20, 200 << 20, 300 << 20], flags, log_cap=200, ctx="fig2_dtr")
    t = coop.Trace(tr)
    _, ev = t.replay([250 << 20], coop.F_POLICY_DTR, log_cap=200)
    e = ev[0]
    op5 = [(int(k), int(x), int(a) >> 20) for k, o, x, a in zip(e["kind"], e["op"], e["tensor"], e["addr"])
           if o == 5 and k in (O.EV_EVICT, O.EV_ALLOC)]
    assert op5 == [(O.EV_EVICT, 0, 0), (O.EV_EVICT, 2, 100), (O.EV_EVICT, 1, 50), (O.EV_ALLOC, 5, 0)]


@pytest.mark.parametrize("n", [4, 8])
def test_dead_diamond_gpu(n):
    """R22 on the GPU: the dead chain is recomputed once (3n + 2 recomputes)."""
    tr = TR.dead_diamond_trace(n)
    res = check(tr, [3 * n + 5, 3 * n + 8], 0, log_cap=1000, ctx="dead_diamond")
    assert int(res[0]["remat"]) == 3 * n + 2


@pytest.mark.parametrize("walk", ["Group", "warp", "lane", "generic"])
def test_closure_walk_variants(walk, monkeypatch):
    """Every projected-cost walk of the replay engine (the warp BFS,
    the per-thread walk over the shared-memory graph, round 1's generic walk) is bit-exact
    with O2 on thrashing DNN cells and random traces."""
    monkeypatch.setenv("COOP_REPLAY_WALK", walk)
    for name, fracs in (("bilstm", (0.3,)), ("gpt3_2.7b", (0.45,)), ("inception_v3", (0.3,)), ("unet", (0.45,))):
        tr = dnn.dnn(name)
        flags = coop.F_PARTITION | coop.F_INPLACE
        peak = O.peak_live(tr, flags)
        check(tr, [int(peak * f) for f in fracs], flags, ctx=f"{walk} {name}")
    rng = np.random.default_rng(42)
    for _ in range(6):
        tr = TR.random_trace(rng, n_params=2, n_fwd=10, iters=2, inplace_p=0.25)
        peak = O.peak_live(tr, 3)
        check(tr, [max(1, int(peak * 0.5)), max(1, int(peak * 0.7))], 3, log_cap=2000, ctx=f"{walk} random")


def test_r37_block_capacity_nomem():
    """DESIGN.md R37: the replay kernel holds at most 4096 blocks per pool in shared memory;
    a pool that needs more ends with COOP_ERR_NOMEM at the op that would exceed it (the
    oracle's own limit is the search's 8192, so it completes).  4200 one-byte tensors stay
    live until a final op reads them all."""
    b = TR.Builder("many_blocks")
    xs = [b.op([], 1, 1) for _ in range(4200)]
    b.op(xs, 1, 1)
    tr = b.build()
    budget = 100000
    res, _ = coop.Trace(tr).replay([budget], 0)
    assert int(res[0]["status"]) == coop.ERR_NOMEM
    assert int(res[0]["max_blocks"]) <= 4096
    want, _ = O.replay(tr, budget, 0)
    assert int(want["status"]) == O.OK


@pytest.mark.parametrize("helpers", [0, 1, 3])
def test_cluster_helpers(helpers, monkeypatch):
    """Thread-block clusters of 1 + helpers CTAs per cell: the helper
    CTAs walk projected-cost closures from the leader's work counter at every pressure
    event; every counter, the digest and the event log stay bit-exact with O2."""
    monkeypatch.setenv("COOP_REPLAY_HELPER", str(helpers))
    for name, frac in (("bilstm", 0.3), ("gpt3_2.7b", 0.5), ("resnet50", 0.4)):
        tr = dnn.dnn(name)
        flags = coop.F_PARTITION | coop.F_INPLACE
        peak = O.peak_live(tr, flags)
        check(tr, [int(peak * frac), int(peak * (frac + 0.1))], flags, log_cap=30000, ctx=f"helpers {helpers} {name}")
    for pol in (coop.F_POLICY_DTR, coop.F_POLICY_DTE):
        tr = dnn.unet()
        peak = O.peak_live(tr, 0)
        check(tr, [int(peak * 0.6)], pol, ctx=f"helpers {helpers} pol {pol}")
