"""Seeded synthetic allocation traces (input generation only; no replay arithmetic here).

A trace is the execution-ordered op list of one or more training iterations, in the SoA
form both the oracle (oracle/oracle_replay.c) and libcoop (coop_trace_create) consume:

  tensors: size[T] (bytes), is_param[T] (parameter / optimizer state: unevictable,
           pre-placed), producer[T] (op id, -1 for parameters)
  ops:     cost_us[M], out[M] (single output, R30), inplace_src[M] (mutated
           input or -1), phase[M] (0 forward, 1 backward, 2 update), inputs in CSR
           (in_ptr[M+1], in_idx[...]).

`dnn(name, ...)` builds the eight DNN shapes of the paper's evaluation (
DESIGN.md "Input recipe"): forward + backward (+ gradient accumulation) + optimizer
updates as in-place ops, I iterations.  Costs are Table 1 densities
times output MiB.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

FWD, BWD, UPD = 0, 1, 2
MiB = 1 << 20


@dataclass
class Trace:
    name: str
    size: np.ndarray
    is_param: np.ndarray
    producer: np.ndarray
    cost_us: np.ndarray
    out: np.ndarray
    inplace_src: np.ndarray
    phase: np.ndarray
    in_ptr: np.ndarray
    in_idx: np.ndarray

    @property
    def n_tensors(self) -> int:
        return len(self.size)

    @property
    def n_ops(self) -> int:
        return len(self.out)

    def inputs(self, k: int):
        return self.in_idx[self.in_ptr[k]:self.in_ptr[k + 1]]

    def summary(self) -> dict:
        return {"name": self.name, "tensors": self.n_tensors, "ops": self.n_ops,
                "params": int(self.is_param.sum()),
                "param_bytes": int(self.size[self.is_param.astype(bool)].sum()),
                "inplace_ops": int((self.inplace_src >= 0).sum()),
                "base_us": int(self.cost_us.sum())}


class Builder:
    def __init__(self, name: str):
        self.name = name
        self.size, self.is_param, self.producer = [], [], []
        self.cost, self.out, self.src, self.phase, self.ins = [], [], [], [], []

    def param(self, nbytes: int) -> int:
        self.size.append(int(nbytes))
        self.is_param.append(1)
        self.producer.append(-1)
        return len(self.size) - 1

    def op(self, inputs, out_bytes: int, cost_us: int, phase: int = FWD, inplace: int = -1) -> int:
        t = len(self.size)
        self.size.append(int(out_bytes))
        self.is_param.append(0)
        self.producer.append(len(self.out))
        self.cost.append(int(max(0, cost_us)))
        self.out.append(t)
        self.src.append(int(inplace))
        self.phase.append(int(phase))
        self.ins.append([int(x) for x in inputs])
        return t

    def build(self) -> Trace:
        ptr = np.zeros(len(self.ins) + 1, np.int32)
        ptr[1:] = np.cumsum([len(x) for x in self.ins])
        idx = np.array([u for x in self.ins for u in x], np.int32)
        return Trace(self.name, np.array(self.size, np.uint64), np.array(self.is_param, np.uint8),
                     np.array(self.producer, np.int32), np.array(self.cost, np.int64),
                     np.array(self.out, np.int32), np.array(self.src, np.int32),
                     np.array(self.phase, np.uint8), ptr, idx)


# ------------------------------------------------------------------ small scenarios
def fig2_trace(mib: int = MiB) -> Trace:
    """Fig. 2: conv/activation chain x0..x4 (50 MB each), then a
    100 MB request for x5; densities from Table 1's ResNet-50 column (conv 35.6, ReLU 3.9
    us/MB).  A mirrored backward then reads x5, x4, ..., x0 once each."""
    b = Builder("fig2")
    x0 = b.op([], 50 * mib, 195)           # activation output (3.9 us/MB x 50)
    x1 = b.op([x0], 50 * mib, 1780)        # conv (35.6 x 50)
    x2 = b.op([x1], 50 * mib, 195)
    x3 = b.op([x2], 50 * mib, 1780)
    x4 = b.op([x3], 50 * mib, 195)
    x5 = b.op([x4], 100 * mib, 3560)       # conv producing 100 MB
    g = b.op([x5], 1 * mib, 10, BWD)
    for x in (x4, x3, x2, x1, x0):
        g = b.op([g, x], 1 * mib, 10, BWD)
    return b.build()


def fig2_dtr_trace(mib: int = MiB) -> Trace:
    """Fig. 2 as the DTR half of PAPER.md:202 tells it: the same chain, but the first conv
    is the more expensive one (twice the FLOPs of the second: 3560 us vs 1780 us at Table 1's
    35.6 us/MB).  With equal conv costs the DTR heuristics of x1 and x2 tie exactly after
    x0's eviction ((1780 + 195) / 1975 = 195 / 195), which is not the paper's scenario.
    Here x0 is the stalest and cheapest tensor (c = 195, s = 2170), its eviction raises
    h(x1) to (3560 + 195) / 1975 > h(x2) = 195 / 195, so DTR (h = c / (m s), R46) evicts x0,
    then x2, finds the two freed 50 MB chunks non-contiguous, and evicts x1 as well; Coop's
    window search evicts one contiguous run of two tensors."""
    b = Builder("fig2_dtr")
    x0 = b.op([], 50 * mib, 195)
    x1 = b.op([x0], 50 * mib, 3560)
    x2 = b.op([x1], 50 * mib, 195)
    x3 = b.op([x2], 50 * mib, 1780)
    x4 = b.op([x3], 50 * mib, 195)
    x5 = b.op([x4], 100 * mib, 3560)
    g = b.op([x5], 1 * mib, 10, BWD)
    for x in (x4, x3, x2, x1, x0):
        g = b.op([g, x], 1 * mib, 10, BWD)
    return b.build()


def dead_diamond_trace(n: int = 8, unit: int = 1) -> Trace:
    """A chain of n diamonds whose tensors are all dead when the chain's tip must be
    recomputed (pins DESIGN.md R22 against SURVEY N22):
        x0 = src(); a_k = g(x_{k-1}); b_k = h(x_{k-1}); x_k = f(a_k, b_k)   (k = 1..n)
        y = f(x_n)                              -- every x, a, b dies in the forward pass
        z = src() (size Z)                      -- with budget Z + 1, y (2 units) is evicted
        u = f(z); w = f(y, u)                   -- y is needed again: recompute the chain
    Under R22 each dead tensor recomputed for y stays resident until the end of the op, so
    the chain is recomputed once (3n + 2 recomputes).  Freeing a dead tensor right after the
    recompute that consumed it (N22) makes b_k recompute x_{k-1} again after a_k did:
    T(x_k) = 3 + 2 T(x_{k-1}), exponential in n."""
    b = Builder("dead_diamond")
    x = b.op([], unit, 3)
    for _ in range(n):
        a = b.op([x], unit, 5)
        c = b.op([x], unit, 5)
        x = b.op([a, c], unit, 7)
    y = b.op([x], 2 * unit, 11)
    big = (3 * n + 4) * unit
    z = b.op([], big, 13)
    u = b.op([z], unit, 1)
    b.op([y, u], unit, 1)
    return b.build()


def random_trace(rng: np.random.Generator, n_params=3, n_fwd=12, max_in=3, inplace_p=0.15,
                 size_choices=(1, 2, 3, 4, 6, 8), unit=1, iters=1) -> Trace:
    """Random small training-like DAG: forward chain-ish ops reading recent tensors and
    parameters, a mirrored backward that reads forward tensors, in-place parameter
    updates, optionally iterated.  Sizes are small multiples of `unit` so byte-map models
    stay tiny."""
    b = Builder("random")
    params = [b.param(int(rng.choice(size_choices)) * unit) for _ in range(n_params)]
    for _ in range(iters):
        acts = []
        for _ in range(n_fwd):
            pool = acts[-4:]
            k = int(rng.integers(0, min(max_in, len(pool)) + 1)) if pool else 0
            ins = list(rng.choice(pool, size=k, replace=False)) if k else []
            if params and rng.random() < 0.5:
                ins.append(int(rng.choice(params)))
            sz = int(rng.choice(size_choices)) * unit
            cost = int(rng.integers(1, 100)) * (1 if rng.random() < 0.5 else 20)
            if acts and rng.random() < inplace_p:
                src = acts[-1]
                if src not in ins:
                    ins.append(src)
                t = b.op(ins, b.size[src], cost, FWD, inplace=src)
                acts[-1] = t
                continue
            acts.append(b.op(ins, sz, cost, FWD))
        grads = []
        g = b.op([acts[-1]], int(rng.choice(size_choices)) * unit, 5, BWD)
        for a in reversed(acts[:-1]):
            ins = [g, a]
            g = b.op(ins, int(rng.choice(size_choices)) * unit, int(rng.integers(1, 100)), BWD)
            grads.append(g)
        for j, p in enumerate(params):
            gp = grads[j % len(grads)] if grads else g
            new = b.op([p, gp], b.size[p], 3, UPD, inplace=p)
            params[j] = new
    return b.build()
