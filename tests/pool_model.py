"""Independent Python model of the online single-pool calls (R38-R44), for pinning
the C oracle O3 on tiny pools.  Same deliberate differences as tests/replay_model.py:

* memory is a byte map (one owner per byte), so free chunks coalesce by construction and
  the address-ordered item list is the run-length view of the map;
* the window search enumerates all O(N^2) windows with exact Fractions (Eq. 1,
  PAPER.md:104-112; the cost is RN of the exact sum via float(Fraction));
* projected costs are set closures over Python sets (R18).

Also home of the seeded random "framework" driver shared by the oracle pins and the GPU
parity tests (it decides calls from returned statuses only, never from internals).
"""
from __future__ import annotations

import random
from fractions import Fraction

FREE = -1
M64 = (1 << 64) - 1
OK, NEEDS_REMAT, INVALID_ARG, UNKNOWN_ID, UNSAT, NOMEM, BAD_STATE = 0, 1, -1, -2, -3, -6, -7
EXPENSIVE, CHEAP, INPLACE, UNEVICTABLE, PHASE_FWD = 1, 2, 4, 8, 16


def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class OnlineModel:
    def __init__(self, budget, flags, threshold=15, max_tensors=4096, max_edges=16384):
        self.flags, self.thr = flags, threshold
        self.max_tensors, self.max_edges = max_tensors, max_edges
        self.mem = [FREE] * budget
        self.size, self.cost, self.ins, self.src, self.cls, self.fwd = [], [], [], [], [], []
        self.unev, self.resident, self.born, self.dead = [], [], [], []
        self.pins, self.last_access, self.addr = [], [], []
        self.clock = 0
        self.cur = -1
        self.c = dict(base_us=0, total_us=0, evictions=0, remat=0, pressure=0, frag_fail=0,
                      inplace_reuse=0, heuristic_evals=0, sum_free_bytes_after=0,
                      sum_free_blocks_after=0, digest=0x9E3779B97F4A7C15, max_blocks=1,
                      fail_op=-1, n_events=0)
        self.win = None

    # ---------------------------------------------------------------- memory
    def runs(self):
        out, i, n = [], 0, len(self.mem)
        while i < n:
            j = i
            while j < n and self.mem[j] == self.mem[i]:
                j += 1
            out.append((i, j - i, self.mem[i]))
            i = j
        return out

    def _blocks_seen(self):
        self.c["max_blocks"] = max(self.c["max_blocks"], len(self.runs()))

    def fit(self, size, right):
        cands = [(a, s) for a, s, o in self.runs() if o == FREE and s >= size]
        if not cands:
            return None
        a, s = cands[-1] if right else cands[0]
        return a + s - size if right else a

    def put(self, t, a):
        for x in range(a, a + self.size[t]):
            assert self.mem[x] == FREE
            self.mem[x] = t
        self.addr[t] = a
        self.resident[t] = True
        self._blocks_seen()

    def clear(self, t):
        a = self.addr[t]
        for x in range(a, a + self.size[t]):
            assert self.mem[x] == t
            self.mem[x] = FREE
        self.resident[t] = False
        return a

    def right(self, t):
        if not (self.flags & 1):
            return False
        if not self.fwd[t] and not (self.flags & 4):
            return False
        if self.cls[t]:
            return self.cls[t] == 2
        return not (self.cost[t] * (1 << 20) >= self.thr * self.size[t])

    # ---------------------------------------------------------------- heuristic
    def consumers(self, x):
        return [k for k in range(len(self.ins)) if x in self.ins[k] and self.born[k]]

    def projected(self, t):
        seen = {t}
        total = self.cost[t]
        stack = list(self.ins[t])
        while stack:
            u = stack.pop()
            if u in seen:
                continue
            seen.add(u)
            if self.resident[u]:
                continue
            total += self.cost[u]
            stack += self.ins[u]
        stack = self.consumers(t)
        while stack:
            d = stack.pop()
            if d in seen:
                continue
            seen.add(d)
            if not self.born[d] or self.resident[d] or self.dead[d]:
                continue
            total += self.cost[d]
            stack += self.consumers(d)
        return total

    def search(self, R):
        items = []
        for a, s, o in self.runs():
            if o == FREE:
                items.append((a, s, o, Fraction(0), False))
            elif self.unev[o] or self.pins[o] > 0:
                items.append((a, s, o, None, True))
            else:
                st = max(1, self.clock - self.last_access[o])
                h = Fraction(float(self.projected(o)) / float(st))
                self.c["heuristic_evals"] += 1
                items.append((a, s, o, h, False))
        best = None
        for i in range(len(items)):
            span, tot = 0, Fraction(0)
            for j in range(i, len(items)):
                if items[j][4]:
                    break
                span += items[j][1]
                tot += items[j][3]
                if span >= R:
                    key = (float(tot), i)
                    if best is None or key < best[0]:
                        best = (key, i, j, span)
                    break
        if best is None:
            return None
        (cost, _), i, j, span = best
        self.win = (i, j, span, cost)
        return [items[k][2] for k in range(i, j + 1) if items[k][2] != FREE]

    def evict_loop(self, size):
        """DTR / DTE baselines (R46), as tests/replay_model.py"""
        dte = bool(self.flags & 16)
        victims = []
        while self.fit(size, False) is None:
            best = None
            runs = self.runs()
            for idx, (a, sz, o) in enumerate(runs):
                if o == FREE or self.unev[o] or self.pins[o] > 0:
                    continue
                st = max(1, self.clock - self.last_access[o])
                m = sz
                if dte:
                    if idx > 0 and runs[idx - 1][2] == FREE:
                        m += runs[idx - 1][1]
                    if idx + 1 < len(runs) and runs[idx + 1][2] == FREE:
                        m += runs[idx + 1][1]
                h = float(self.projected(o)) / (float(m) * float(st))
                self.c["heuristic_evals"] += 1
                if best is None or h < best[0]:
                    best = (h, o)
            if best is None:
                return None
            victims.append(best[1])
            self.evict(best[1])
        return victims

    def evict(self, t):
        a = self.clear(t)
        self.c["evictions"] += 1
        self.c["n_events"] += 1
        d = self.c["digest"]
        d = splitmix64(d ^ (((self.cur & 0xFFFFFFFF) << 32) | t))
        self.c["digest"] = splitmix64(d ^ a)

    # ---------------------------------------------------------------- Alg. 1
    def allocate(self, t, allow_inplace):
        src = self.src[t]
        if allow_inplace and src >= 0 and (self.flags & 2):
            a = self.addr[src]
            for x in range(a, a + self.size[t]):
                self.mem[x] = t
            self.addr[t] = a
            self.resident[src] = False
            self.resident[t] = True
            self.c["inplace_reuse"] += 1
            self.c["n_events"] += 1
            return [], True
        right = self.right(t)
        a = self.fit(self.size[t], right)
        victims = []
        if a is None:
            self.c["pressure"] += 1
            if sum(1 for x in self.mem if x == FREE) >= self.size[t]:
                self.c["frag_fail"] += 1
            if self.flags & 24:
                victims = self.evict_loop(self.size[t])
            else:
                victims = self.search(self.size[t])
                if victims is not None:
                    for v in victims:
                        self.evict(v)
            if victims is None:
                self.c["fail_op"] = self.cur
                return None, False
            a = self.fit(self.size[t], right)
            self.put(t, a)
            fr = [s for _, s, o in self.runs() if o == FREE]
            self.c["sum_free_bytes_after"] += sum(fr)
            self.c["sum_free_blocks_after"] += len(fr)
        else:
            self.put(t, a)
        self.c["n_events"] += 1
        return victims, True

    def _result(self, t, victims):
        if self.win is not None:
            i, j, span, cost = self.win
        else:
            i, j, span, cost = -1, -1, 0, 0.0
        return dict(tensor_id=t, addr=self.addr[t], size=self.size[t], n_evicted=len(victims),
                    window_first=i, window_last=j, window_span=span, window_cost=cost), victims

    # ---------------------------------------------------------------- the calls
    def alloc(self, size, cost, op_flags=0, src=-1, parents=()):
        T = len(self.size)
        if size < 1 or size >= 1 << 48 or cost >= 1 << 40:
            return INVALID_ARG, None, []
        if op_flags & ~31 or (op_flags & EXPENSIVE and op_flags & CHEAP):
            return INVALID_ARG, None, []
        if any(p < 0 or p >= T for p in parents):
            return UNKNOWN_ID, None, []
        if op_flags & INPLACE:
            if src not in parents or self.size[src] != size:
                return INVALID_ARG, None, []
        elif src != -1:
            return INVALID_ARG, None, []
        if T >= self.max_tensors or sum(len(x) for x in self.ins) + len(parents) > self.max_edges:
            return NOMEM, None, []
        for p in parents:
            if not self.resident[p]:
                return NEEDS_REMAT, dict(tensor_id=p), []
        t = T
        self.size.append(size)
        self.cost.append(cost)
        self.ins.append(list(parents))
        self.src.append(src if op_flags & INPLACE else -1)
        self.cls.append(1 if op_flags & EXPENSIVE else 2 if op_flags & CHEAP else 0)
        self.fwd.append(bool(op_flags & PHASE_FWD))
        self.unev.append(bool(op_flags & UNEVICTABLE) or (self.src[t] >= 0 and self.unev[self.src[t]]))
        self.resident.append(False)
        self.born.append(False)
        self.dead.append(False)
        self.pins.append(0)
        self.last_access.append(0)
        self.addr.append(0)
        self.cur, self.win = t, None
        for p in parents:
            self.pins[p] += 1
        victims, ok = self.allocate(t, True)
        for p in parents:
            self.pins[p] -= 1
        if not ok:
            for lst in (self.size, self.cost, self.ins, self.src, self.cls, self.fwd, self.unev,
                        self.resident, self.born, self.dead, self.pins, self.last_access, self.addr):
                lst.pop()
            return UNSAT, None, []
        self.born[t] = True
        self.clock += cost
        self.c["base_us"] += cost
        self.c["total_us"] += cost
        self.c["n_events"] += 1
        for p in parents:
            self.last_access[p] = self.clock
        self.last_access[t] = self.clock
        r, v = self._result(t, victims)
        return OK, r, v

    def free(self, t):
        if t < 0 or t >= len(self.size):
            return UNKNOWN_ID
        if self.dead[t] and not self.resident[t]:
            return BAD_STATE
        if self.resident[t]:
            self.clear(t)
            self.c["n_events"] += 1
        self.dead[t] = True
        return OK

    def access(self, t, adv=0):
        if t < 0 or t >= len(self.size):
            return UNKNOWN_ID
        if adv >= 1 << 40:
            return INVALID_ARG
        if self.dead[t] and not self.resident[t]:
            return BAD_STATE
        self.clock += adv
        if not self.resident[t]:
            return NEEDS_REMAT
        self.last_access[t] = self.clock
        return OK

    def remat(self, t):
        if t < 0 or t >= len(self.size):
            return UNKNOWN_ID, None, []
        self.win = None
        if self.resident[t]:
            r, v = self._result(t, [])
            return OK, r, v
        for p in self.ins[t]:
            if not self.resident[p]:
                return NEEDS_REMAT, dict(tensor_id=p), []
        self.cur = t
        for p in self.ins[t]:
            self.pins[p] += 1
        victims, ok = self.allocate(t, False)
        for p in self.ins[t]:
            self.pins[p] -= 1
        if not ok:
            return UNSAT, None, []
        self.clock += self.cost[t]
        self.c["total_us"] += self.cost[t]
        self.c["remat"] += 1
        self.c["n_events"] += 1
        for p in self.ins[t]:
            self.last_access[p] = self.clock
        self.last_access[t] = self.clock
        r, v = self._result(t, victims)
        return OK, r, v

    def layout(self):
        return [(a, s, o) for a, s, o in self.runs()]


# -------------------------------------------------------------------- the random driver
def random_session(seed, n_calls, budget=400, flags=3, max_size=48):
    """A seeded list of abstract calls.  Tensor choices are indices into the list of ids
    created so far (resolved at run time), so the same list drives every implementation."""
    rng = random.Random(seed)
    calls = []
    for _ in range(n_calls):
        x = rng.random()
        if x < 0.55:
            size = rng.randint(1, max_size)
            cost = rng.choice([0, 1, 2, 3, 5, 8, 40, 1000, rng.randint(0, 5000)])
            f = rng.choice([0, EXPENSIVE, CHEAP]) | (PHASE_FWD if rng.random() < 0.6 else 0)
            if rng.random() < 0.06:
                f |= UNEVICTABLE
            npar = rng.choice([0, 1, 1, 2, 2, 3])
            picks = [rng.random() for _ in range(npar)]
            inplace = rng.random() < 0.15 and npar > 0
            calls.append(("alloc", size, cost, f, picks, inplace))
        elif x < 0.75:
            calls.append(("free", rng.random()))
        elif x < 0.95:
            calls.append(("access", rng.random(), rng.choice([0, 1, 3, 10, 100])))
        else:
            calls.append(("remat", rng.random()))
    return calls


def drive(impl, calls, size_of=None):
    """Run abstract calls against `impl` (alloc/free/access/remat with the O3 signatures,
    returning (status, result-dict-or-record, evicted list) / status).  Parents are picked
    among non-dead ids; a NEEDS_REMAT answer is served depth-first by remat calls.  Returns
    the transcript of (call, status, payload) for comparison."""
    ids, dead, sizes, out = [], set(), {}, []

    def rec(x):
        if x is None:
            return None
        if isinstance(x, dict):
            return tuple(sorted(x.items()))
        return tuple(sorted((k, x[k].item()) for k in x.dtype.names if k != "reserved"))

    def remat_chain(t, depth=0):
        st, r, v = impl.remat(t)
        out.append(("remat", t, st, rec(r) if st == OK else None, tuple(v)))
        if st == NEEDS_REMAT and depth < 64:
            p = int(r["tensor_id"])  # a freed parent is recomputed too (R44)
            st2 = remat_chain(p, depth + 1)
            if st2 == OK:
                return remat_chain(t, depth + 1)
        return st

    for c in calls:
        live = [t for t in ids if t not in dead]
        if c[0] == "alloc":
            _, size, cost, f, picks, inplace = c
            parents = []
            for q in picks:
                if live:
                    p = live[int(q * len(live))]
                    if p not in parents:
                        parents.append(p)
            src = -1
            if inplace and parents:
                src = parents[0]
                size = sizes[src]
                f |= INPLACE
            for p in parents:  # the framework materializes the inputs first
                st = impl.access(p, 0)
                out.append(("access", p, st))
                if st == NEEDS_REMAT:
                    remat_chain(p)
            st, r, v = impl.alloc(size, cost, f, src, parents)
            if st == NEEDS_REMAT:
                out.append(("alloc", st))
                continue
            out.append(("alloc", st, rec(r) if st == OK else None, tuple(v)))
            if st == OK:
                t = int(r["tensor_id"])
                ids.append(t)
                sizes[t] = size
        elif c[0] == "free":
            if not live:
                continue
            t = live[int(c[1] * len(live))]
            st = impl.free(t)
            out.append(("free", t, st))
            if st == OK:
                dead.add(t)
        elif c[0] == "access":
            if not live:
                continue
            t = live[int(c[1] * len(live))]
            st = impl.access(t, c[2])
            out.append(("access", t, st))
            if st == NEEDS_REMAT:
                remat_chain(t)
        else:
            if not ids:
                continue
            t = ids[int(c[1] * len(ids))]
            st, r, v = impl.remat(t)
            out.append(("remat", t, st, rec(r) if st == OK else None, tuple(v)))
    return out
