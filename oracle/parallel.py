"""Multi-process drivers of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

One worker process per host core (fork), each running the single-threaded C oracle on a
share of independent units: replay cells (O2, one (trace, budget) per unit, longest-first
dynamic scheduling) or window-search pools (O1, contiguous slices, inputs generated in the
worker by the seeded counter-based generator of gen/).  May be imported only by tests/,
__graft_entry__.smoke() and bench.py's oracle baseline legs; the oracle arithmetic stays in
liboracle.so.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from oracle import oracle as O

_TRACES: dict = {}


def _trace(name: str):
    tr = _TRACES.get(name)
    if tr is None:
        from gen import dnn
        tr = _TRACES[name] = dnn.dnn(name)
    return tr


def _warm(names):
    for n in names:
        _trace(n)


def _noop(_):
    time.sleep(0.05)


def _replay_unit(args):
    idx, name, budget, flags = args
    tr = _trace(name)  # generated once per worker, outside the timed call
    t = time.perf_counter()
    r, _ = O.replay(tr, int(budget), int(flags))
    return idx, r, time.perf_counter() - t


def replay_cells(cells, flags: int, procs: int | None = None):
    """O2 on every (trace_name, budget) cell -> (ORC_RESULT array in cell order, wall s,
    per-cell seconds, processes).  Cells are handed out dynamically, slowest first (low
    budget fractions first; BiLSTM and GPT-3 first among equals), one per task."""
    procs = procs or os.cpu_count() or 1
    heavy = {"bilstm": 0, "gpt3_2.7b": 1}
    order = sorted(range(len(cells)), key=lambda i: (heavy.get(cells[i][0], 2), cells[i][2]
                                                     if len(cells[i]) > 2 else 0, i))
    units = [(i, cells[i][0], cells[i][1], flags) for i in order]
    out = np.zeros(len(cells), O.ORC_RESULT)
    secs = np.zeros(len(cells))
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_warm, initargs=(sorted({c[0] for c in cells}),)) as pool:
        pool.map(_noop, range(procs), chunksize=1)  # workers up, traces generated
        t0 = time.perf_counter()
        for idx, r, dt in pool.imap_unordered(_replay_unit, units, chunksize=1):
            out[idx] = r
            secs[idx] = dt
        wall = time.perf_counter() - t0
    return out, wall, secs, procs


def _search_unit(args):
    mode, seed, p0, n_pools, n, stride = args
    from gen import pools as G
    ss, c, s, r = G.bench_pools_host(mode, seed, p0, n_pools, n, stride)
    t = time.perf_counter()
    w = O.search_many(ss, c, s, r, n_pools, n, stride)
    return p0, w, time.perf_counter() - t


def search_pools(mode: int, seed: int, p0: int, n_pools: int, n: int, stride: int | None = None,
                 procs: int | None = None, chunk: int = 256):
    """O1 on the generator's pools [p0, p0 + n_pools) -> (ORC_WINDOW array, wall s of the
    oracle calls (max over workers' summed search time is not used: wall of the whole map),
    processes)."""
    procs = procs or os.cpu_count() or 1
    stride = stride or n
    units = [(mode, seed, q, min(chunk, p0 + n_pools - q), n, stride)
             for q in range(p0, p0 + n_pools, chunk)]
    out = np.zeros(n_pools, O.ORC_WINDOW)
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        for q, w, _ in pool.imap_unordered(_search_unit, units, chunksize=1):
            out[q - p0:q - p0 + len(w)] = w
    return out, time.perf_counter() - t0, procs
