"""Pins for the O2 replay oracle (oracle/oracle_replay.c): a worked example derived by hand
from Fig. 2, an independent Python model with different data
structures (tests/replay_model.py: byte-map memory, O(N^2) Fraction window search, set
closures), and invariants: no-pressure identity, memory-content consistency of every
executed op, unevictable address stability with recomputable in-place,
counter consistency, and the peak-memory definition."""
import numpy as np
import pytest

from gen import traces as TR
from oracle import oracle as O
from replay_model import Model

MiB = 1 << 20
ALL_FLAGS = [0, O.F_PARTITION, O.F_INPLACE, O.F_PARTITION | O.F_INPLACE,
             O.F_PARTITION | O.F_INPLACE | O.F_PARTITION_ALL_PHASES]
RESULT_FIELDS = ["status", "fail_op", "base_us", "total_us", "evictions", "remat", "pressure",
                 "frag_fail", "inplace_reuse", "heuristic_evals", "sum_free_bytes_after",
                 "sum_free_blocks_after", "digest", "max_depth"]


def ev_tuples(log):
    return [(int(e["kind"]), int(e["op"]), int(e["tensor"]), int(e["addr"])) for e in log]


def test_fig2_partition_worked_example():
    """Hand-derived: partitioned layout
    x1[0,50) x3[50,100) x4[100,150) x2[150,200) x0[200,250) MiB; at op5 (x4 pinned as the
    input) h = (195/2170, 1780/1975, 195/195, 1780/1) for x0..x3; the window {x2, x0}
    costs 1.0898...; x2 and x0 are evicted and x5 (C1) lands at the left end, 150 MiB."""
    tr = TR.fig2_trace()
    r, log = O.replay(tr, 250 * MiB, O.F_PARTITION | O.F_INPLACE, log_cap=200)
    ev = ev_tuples(log)
    allocs = {t: a for k, _, t, a in ev if k == O.EV_ALLOC and t <= 4}
    assert allocs == {0: 200 * MiB, 1: 0, 2: 150 * MiB, 3: 50 * MiB, 4: 100 * MiB}
    op5 = [(k, t, a) for k, op, t, a in ev if op == 5 and k in (O.EV_EVICT, O.EV_ALLOC)]
    assert op5 == [(O.EV_EVICT, 2, 150 * MiB), (O.EV_EVICT, 0, 200 * MiB),
                   (O.EV_ALLOC, 5, 150 * MiB)]
    assert int(r["status"]) == O.OK


def test_fig2_no_partition_worked_example():
    """Without partitioning: x0..x4 left to right; window {x0, x1} (cost 0.9911...)."""
    tr = TR.fig2_trace()
    r, log = O.replay(tr, 250 * MiB, O.F_INPLACE, log_cap=200)
    op5 = [(k, t, a) for k, op, t, a in ev_tuples(log) if op == 5 and k in (O.EV_EVICT, O.EV_ALLOC)]
    assert op5 == [(O.EV_EVICT, 0, 0), (O.EV_EVICT, 1, 50 * MiB), (O.EV_ALLOC, 5, 0)]


def _random_cases(n_cases, seed):
    rng = np.random.default_rng(seed)
    for _ in range(n_cases):
        tr = TR.random_trace(rng, n_params=int(rng.integers(0, 4)), n_fwd=int(rng.integers(2, 10)),
                             iters=int(rng.integers(1, 3)), inplace_p=0.25)
        flags = int(rng.choice(ALL_FLAGS))
        peak = O.peak_live(tr, flags)
        frac = float(rng.choice([0.4, 0.55, 0.7, 0.85, 1.0, 1.3]))
        budget = max(1, int(peak * frac))
        yield tr, flags, budget


@pytest.mark.parametrize("seed", range(12))
def test_vs_independent_python_model(seed):
    for tr, flags, budget in _random_cases(25, seed):
        r, log = O.replay(tr, budget, flags, log_cap=100000)
        m = Model(tr, budget, flags)
        status, fail_op = m.run()
        got = {f: int(r[f]) for f in RESULT_FIELDS}
        want = dict(m.c, status=status, fail_op=fail_op)
        assert got == {f: int(want[f]) for f in RESULT_FIELDS}, (flags, budget)
        assert ev_tuples(log) == m.events


def test_no_pressure_identity():
    """Budget far above need: no eviction, no recompute; and a plain
    first-fit run (no partitioning, COW) at exactly its own address high-water mark
    replays identically."""
    rng = np.random.default_rng(21)
    for _ in range(100):
        tr = TR.random_trace(rng, n_params=int(rng.integers(0, 4)), n_fwd=int(rng.integers(2, 12)),
                             iters=2)
        for flags in ALL_FLAGS:
            r, _ = O.replay(tr, 1 << 40, flags)
            assert int(r["status"]) == O.OK
            assert int(r["evictions"]) == 0 and int(r["total_us"]) == int(r["base_us"])
        r, log = O.replay(tr, 1 << 40, 0, log_cap=10000)
        hw = max(int(e["addr"]) + int(tr.size[int(e["tensor"])]) for e in log
                 if int(e["kind"]) in (O.EV_PARAM, O.EV_ALLOC))
        r2, log2 = O.replay(tr, hw, 0, log_cap=10000)
        assert int(r2["evictions"]) == 0 and ev_tuples(log2) == ev_tuples(log)


def test_memory_contents_and_counters():
    """Rebuild memory from the event log: every executed op (original or recompute) finds
    all its inputs resident at their recorded addresses and untouched (the simulator's
    stand-in for value correctness); counters match the log."""
    for tr, flags, budget in _random_cases(300, 99):
        r, log = O.replay(tr, budget, flags, log_cap=100000)
        owner = {}   # byte range start -> tensor
        where = {}   # tensor -> addr while resident
        recompute = 0
        consumed_inplace = set()  # (op, src) whose block the output took just before EXEC
        for k, op, t, a in ev_tuples(log):
            size = int(tr.size[t])
            if k in (O.EV_PARAM, O.EV_ALLOC, O.EV_REMAT):
                for (b, u) in list(owner.items()):
                    assert b + int(tr.size[u]) <= a or a + size <= b, "overlap"
                owner[a] = t
                where[t] = a
            elif k == O.EV_INPLACE:
                src = int(tr.inplace_src[op])
                assert where.get(src) == a
                consumed_inplace.add((op, src))
                del owner[a]
                del where[src]
                owner[a] = t
                where[t] = a
            elif k in (O.EV_EVICT, O.EV_FREE):
                assert where.get(t) == a and owner.get(a) == t
                del owner[a]
                del where[t]
            elif k in (O.EV_EXEC, O.EV_REXEC):
                for u in tr.inputs(op):
                    if k == O.EV_EXEC and (op, int(u)) in consumed_inplace:
                        continue  # the in-place op reads the value it overwrites (Sec. 3.5)
                    assert int(u) in where, f"op {op} reads non-resident tensor {u}"
                if k == O.EV_REXEC:
                    recompute += int(tr.cost_us[op])
        if int(r["status"]) == O.OK:
            assert int(r["total_us"]) - int(r["base_us"]) == recompute
        kinds = [int(e["kind"]) for e in log]
        assert kinds.count(O.EV_EVICT) == int(r["evictions"])
        assert kinds.count(O.EV_REXEC) == int(r["remat"])
        assert int(r["frag_fail"]) <= int(r["pressure"])


def test_unevictable_addresses_stable_with_recomputable_inplace():
    """PAPER.md:222 / SPEC.md:617: with recomputable in-place, every parameter version
    lives at its parameter's original address; with copy-on-write (flag off) some
    parameter moves."""
    rng = np.random.default_rng(5)
    moved_cow = 0
    for _ in range(60):
        tr = TR.random_trace(rng, n_params=3, n_fwd=int(rng.integers(3, 10)), iters=2)
        peak = O.peak_live(tr, O.F_INPLACE)
        for flags, budget in ((O.F_PARTITION | O.F_INPLACE, int(peak * 0.8)), (O.F_INPLACE, peak)):
            r, log = O.replay(tr, budget, flags, log_cap=100000)
            home = {int(e["tensor"]): int(e["addr"]) for e in log if int(e["kind"]) == O.EV_PARAM}
            addr_of = dict(home)
            for e in log:
                if int(e["kind"]) == O.EV_INPLACE:
                    src = int(tr.inplace_src[int(e["op"])])
                    if src in addr_of:
                        assert int(e["addr"]) == addr_of[src]
                        addr_of[int(e["tensor"])] = int(e["addr"])
        r, log = O.replay(tr, 1 << 30, O.F_PARTITION, log_cap=100000)
        home = {int(e["tensor"]): int(e["addr"]) for e in log if int(e["kind"]) == O.EV_PARAM}
        for e in log:
            if int(e["kind"]) == O.EV_ALLOC and int(tr.inplace_src[int(e["op"])]) in home:
                moved_cow += int(e["addr"]) != home[int(tr.inplace_src[int(e["op"])])]
    assert moved_cow > 0


def test_peak_live_definition():
    """one 100-byte output and a 50-byte parameter -> 150; and the peak is
    the maximum of live bytes along the eviction-free replay."""
    b = TR.Builder("one")
    p = b.param(50)
    b.op([p], 100, 10)
    assert O.peak_live(b.build(), 0) == 150
    rng = np.random.default_rng(8)
    for _ in range(50):
        tr = TR.random_trace(rng, n_params=2, n_fwd=8, iters=2)
        for flags in (0, O.F_INPLACE):
            r, log = O.replay(tr, 1 << 40, flags, log_cap=100000)
            live = peak = 0
            for k, op, t, a in ev_tuples(log):
                if k in (O.EV_PARAM, O.EV_ALLOC, O.EV_REMAT):
                    live += int(tr.size[t])
                elif k in (O.EV_FREE, O.EV_EVICT):
                    live -= int(tr.size[t])
                peak = max(peak, live)
            assert O.peak_live(tr, flags) == peak


def test_invalid_traces_rejected():
    b = TR.Builder("bad")
    x = b.op([], 10, 1)
    y = b.op([x], 10, 1, inplace=x)
    b.op([x], 10, 1)  # reads the mutated input after the in-place op
    r, _ = O.replay(b.build(), 1000)
    assert int(r["status"]) == O.INVALID_ARG
    b = TR.Builder("bad2")
    x = b.op([], 10, 1)
    b.op([x], 20, 1, inplace=x)  # size mismatch
    r, _ = O.replay(b.build(), 1000)
    assert int(r["status"]) == O.INVALID_ARG


@pytest.mark.parametrize("seed", range(6))
def test_dtr_dte_baselines_vs_model(seed):
    """NEXT-1 baselines (R46): DTR / DTE argmin loops, same comparison with the independent
    Python model (counters incl. heuristic evaluations, digest, full event log)."""
    for tr, flags, budget in _random_cases(15, 700 + seed):
        for pol in (O.F_DTR, O.F_DTE):
            f = (flags & 7) | pol
            r, log = O.replay(tr, budget, f, log_cap=100000)
            m = Model(tr, budget, f)
            status, fail_op = m.run()
            got = {k: int(r[k]) for k in RESULT_FIELDS}
            want = dict(m.c, status=status, fail_op=fail_op)
            assert got == {k: int(want[k]) for k in RESULT_FIELDS}, (f, budget)
            assert ev_tuples(log) == m.events


def test_fig2_dtr_half():
    """The DTR half of Fig. 2 (NEXT-1, R46) on fig2_dtr_trace: at op 5 DTR
    evicts x0 (stalest and cheapest: h = 195 / (m 2170)), then x2 (x0's eviction raised
    h(x1) to (3560 + 195) / (m 1975) > h(x2) = 195 / (m 195)), finds the freed 50 MB
    chunks [0, 50) and [100, 150) non-contiguous and evicts x1 too: three evictions before
    x5 fits at 0.  Coop's window search on the same state evicts the contiguous pair
    {x0, x1} (h sum 195/2170 + 3560/1975, the cheapest two-tensor window)."""
    tr = TR.fig2_dtr_trace()
    _, log = O.replay(tr, 250 * MiB, O.F_DTR, log_cap=200)
    op5 = [(k, t, a) for k, op, t, a in ev_tuples(log) if op == 5 and k in (O.EV_EVICT, O.EV_ALLOC)]
    assert op5 == [(O.EV_EVICT, 0, 0), (O.EV_EVICT, 2, 100 * MiB), (O.EV_EVICT, 1, 50 * MiB),
                   (O.EV_ALLOC, 5, 0)]
    _, log = O.replay(tr, 250 * MiB, 0, log_cap=200)
    op5 = [(k, t, a) for k, op, t, a in ev_tuples(log) if op == 5 and k in (O.EV_EVICT, O.EV_ALLOC)]
    assert op5 == [(O.EV_EVICT, 0, 0), (O.EV_EVICT, 1, 50 * MiB), (O.EV_ALLOC, 5, 0)]
    # the independent byte-map model agrees on the whole run (byte units: sizes 50 B)
    small = TR.fig2_dtr_trace(mib=1)
    for f in (O.F_DTR, 0, O.F_DTE, O.F_PARTITION | O.F_INPLACE):
        r, log = O.replay(small, 250, f, log_cap=1000)
        m = Model(small, 250, f)
        status, fail_op = m.run()
        got = {k: int(r[k]) for k in RESULT_FIELDS}
        want = dict(m.c, status=status, fail_op=fail_op)
        assert got == {k: int(want[k]) for k in RESULT_FIELDS}, f
        assert ev_tuples(log) == m.events, f


@pytest.mark.parametrize("n", [4, 6, 8])
def test_r22_dead_recomputes_kept_until_end_of_op(n):
    """DESIGN.md R22 vs SURVEY N22 on a chain of dead diamonds (gen/traces.py
    dead_diamond_trace): under R22 (the oracle) the dead chain recomputed for y stays
    resident until the end of the op, so every tensor of it is recomputed once (3n + 2
    recomputes: x0, n x (a, b, x), y); freeing each dead input right after the recompute
    that consumed it (N22, modelled by the independent Python model with n22=True) makes the
    sibling b_k recompute x_{k-1} again, T(x_k) = 3 + 2 T(x_{k-1}): exponential.  The model
    without n22 agrees with the oracle on every counter and event."""
    tr = TR.dead_diamond_trace(n)
    budget = (3 * n + 4) + 1
    r, log = O.replay(tr, budget, 0, log_cap=100000)
    assert int(r["status"]) == O.OK and int(r["evictions"]) == 1
    assert int(r["remat"]) == 3 * n + 2
    m = Model(tr, budget, 0)
    status, fail_op = m.run()
    assert (status, m.c["remat"]) == (0, 3 * n + 2)
    assert ev_tuples(log) == m.events
    m22 = Model(tr, budget, 0, n22=True)
    status22, _ = m22.run()
    t = 1  # T(x0)
    for _ in range(n):
        t = 3 + 2 * t
    assert status22 == 0 and m22.c["remat"] == t + 1  # + y
    assert m22.c["remat"] >= 2 ** n


def test_r34_input_batch_is_recomputable():
    """DESIGN.md R34 (vs SURVEY N34): an input batch is the output of a source op (no
    inputs; re-running it reloads the batch), so it is evictable and rematerializable like
    any activation.  In Fig. 2's chain x0 is such a source output: at 250 MiB Coop evicts
    it at op 5 and the backward pass recomputes it by re-running op 0 (a remat event of op
    0).  Under N34 x0 would be a barrier while live and the op-5 window could not use it."""
    tr = TR.fig2_trace()
    r, log = O.replay(tr, 250 * MiB, O.F_INPLACE, log_cap=200)
    ev = ev_tuples(log)
    assert (O.EV_EVICT, 5, 0, 0) in ev
    assert any(k == O.EV_REXEC and op == 0 and t == 0 for k, op, t, _ in ev)
    assert int(r["status"]) == O.OK
