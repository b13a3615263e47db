"""Independent Python model of the replay (readings R10-R36), for pinning the C
oracle O2 on tiny traces.  Deliberately different data structures and algorithms:

* memory is a byte map (one owner per byte; budgets of a few hundred bytes), so free
  chunks coalesce by construction and the address-ordered item list is the run-length
  view of the map;
* the window search is the O(N^2) enumeration of all windows with exact Fractions
  (Eq. 1; RN via float(Fraction));
* projected costs are recursive set closures over Python sets.
"""
from __future__ import annotations

from fractions import Fraction

FREE = -1
M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class Unsat(Exception):
    pass


class Thrash(Exception):
    pass


class Model:
    def __init__(self, tr, budget, flags, threshold=15, max_depth=512, n22=False):
        # n22: the alternative reading SURVEY N22 (a dead tensor recomputed for another
        # recompute is freed right after the recompute that consumed it, once unpinned)
        # instead of DESIGN.md R22 (kept resident until the end of the trace op); used only
        # to show that the two readings differ (tests/test_oracle_replay.py)
        self.n22 = n22
        self.tr = tr
        self.flags = flags
        self.thr = threshold
        self.max_depth = max_depth
        self.mem = [FREE] * budget
        T, M = tr.n_tensors, tr.n_ops
        self.ins = [list(map(int, tr.inputs(k))) for k in range(M)]
        self.prod = [int(x) for x in tr.producer]
        self.size = [int(x) for x in tr.size]
        self.cost = [int(x) for x in tr.cost_us]
        self.last_use = [-1] * T
        for k in range(M):
            for u in self.ins[k]:
                self.last_use[u] = k
        for t in range(T):
            if self.last_use[t] < 0 and not tr.is_param[t]:
                self.last_use[t] = self.prod[t]
        self.unev = [bool(tr.is_param[t]) for t in range(T)]
        for k in range(M):
            s = int(tr.inplace_src[k])
            if s >= 0 and self.unev[s]:
                self.unev[int(tr.out[k])] = True
        self.consumers = [[] for _ in range(T)]
        for k in range(M):
            for u in self.ins[k]:
                self.consumers[u].append(k)
        # R36 lock lists via explicit need-sets
        need = [set() for _ in range(T)]
        for k in range(M):
            o = int(tr.out[k])
            for u in self.ins[k]:
                need[o] |= {u} if self.unev[u] else need[u]
        self.locks = [[] for _ in range(M)]
        for k in range(M):
            s = int(tr.inplace_src[k])
            if s >= 0 and self.unev[s]:
                self.locks[k] = [t for t in range(T) if not self.unev[t] and not tr.is_param[t]
                                 and self.prod[t] < k and self.last_use[t] > k and s in need[t]]
        self.resident = [False] * T
        self.born = [False] * T
        self.dead = [False] * T
        self.locked = [False] * T
        self.pins = [0] * T
        self.last_access = [0] * T
        self.addr = [0] * T
        self.clock = 0
        self.cur_op = -1
        self.c = dict(base_us=0, total_us=0, evictions=0, remat=0, pressure=0, frag_fail=0,
                      inplace_reuse=0, heuristic_evals=0, sum_free_bytes_after=0,
                      sum_free_blocks_after=0, digest=0x9E3779B97F4A7C15, max_depth=0)
        self.events = []

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

    def clear(self, t):
        a = self.addr[t]
        for x in range(a, a + self.size[t]):
            assert self.mem[x] == t
            self.mem[x] = FREE
        self.resident[t] = False
        return a

    def is_c1(self, op):
        return self.cost[op] * (1 << 20) >= self.thr * self.size[int(self.tr.out[op])]

    def right(self, op):
        if not (self.flags & 1):
            return False
        if int(self.tr.phase[op]) != 0 and not (self.flags & 4):
            return False
        return not self.is_c1(op)

    # ---------------------------------------------------------------- heuristic
    def projected(self, t):
        seen = {t}
        total = self.cost[self.prod[t]]
        stack = list(self.ins[self.prod[t]])
        while stack:
            u = stack.pop()
            if u in seen:
                continue
            seen.add(u)
            if self.resident[u] or self.prod[u] < 0:
                continue
            total += self.cost[self.prod[u]]
            stack += self.ins[self.prod[u]]
        stack = [int(self.tr.out[k]) for k in self.consumers[t]]
        while stack:
            d = stack.pop()
            if d in seen:
                continue
            seen.add(d)
            if not self.born[d] or self.resident[d] or self.dead[d]:
                continue
            total += self.cost[self.prod[d]]
            stack += [int(self.tr.out[k]) for k in self.consumers[d]]
        return total

    def search(self, R):
        items = []
        for a, s, o in self.runs():
            if o == FREE:
                items.append((a, s, o, Fraction(0), False))
            elif self.unev[o] or self.pins[o] > 0 or self.locked[o]:
                items.append((a, s, o, None, True))
            else:
                st = max(1, self.clock - self.last_access[o])
                h = Fraction(float(self.projected(o)) / float(st))  # h = c/s in binary64
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
                        best = (key, i, j)
                    break
        if best is None:
            raise Unsat()
        return [items[k][2] for k in range(best[1], best[2] + 1) if items[k][2] != FREE]

    def evict_loop(self, size):
        """DTR / DTE baselines (R46): evict argmin h one tensor at a time until a free
        block can hold `size`; h = c / (m s), DTE adds the adjacent free bytes to m."""
        dte = bool(self.flags & 16)
        while self.fit(size, False) is None:
            best = None
            runs = self.runs()
            for idx, (a, sz, o) in enumerate(runs):
                if o == FREE or self.unev[o] or self.pins[o] > 0 or self.locked[o]:
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
                raise Unsat()
            self.evict(best[1])

    def evict(self, t):
        a = self.clear(t)
        self.c["evictions"] += 1
        self.events.append((3, self.cur_op, t, a))
        d = self.c["digest"]
        d = splitmix64(d ^ (((self.cur_op & 0xFFFFFFFF) << 32) | t))
        d = splitmix64(d ^ a)
        self.c["digest"] = d

    # ---------------------------------------------------------------- Alg. 1
    def allocate(self, op, t, allow_inplace, kind):
        src = int(self.tr.inplace_src[op])
        if allow_inplace and src >= 0 and (self.flags & 2):
            a = self.addr[src]
            for x in range(a, a + self.size[t]):
                self.mem[x] = t
            self.addr[t] = a
            self.resident[src] = False
            self.resident[t] = True
            self.c["inplace_reuse"] += 1
            self.events.append((2, op, t, a))
            return
        right = self.right(op)
        a = self.fit(self.size[t], right)
        if a is None:
            self.c["pressure"] += 1
            if sum(1 for x in self.mem if x == FREE) >= self.size[t]:
                self.c["frag_fail"] += 1
            if self.flags & 24:
                self.evict_loop(self.size[t])
            else:
                for v in self.search(self.size[t]):
                    self.evict(v)
            a = self.fit(self.size[t], right)
            self.put(t, a)
            fr = [s for _, s, o in self.runs() if o == FREE]
            self.c["sum_free_bytes_after"] += sum(fr)
            self.c["sum_free_blocks_after"] += len(fr)
        else:
            self.put(t, a)
        self.events.append((kind, op, t, a))

    def materialize(self, t, depth):
        if depth > self.max_depth:
            raise Thrash()
        self.c["max_depth"] = max(self.c["max_depth"], depth)
        op = self.prod[t]
        if op < 0:
            raise Unsat()
        for u in self.ins[op]:
            self.pins[u] += 1
        for u in self.ins[op]:
            if not self.resident[u]:
                self.materialize(u, depth + 1)
        self.allocate(op, t, False, 5)
        self.clock += self.cost[op]
        self.c["total_us"] += self.cost[op]
        self.c["remat"] += 1
        self.events.append((7, op, t, self.addr[t]))
        for u in self.ins[op]:
            self.last_access[u] = self.clock
        self.last_access[t] = self.clock
        for u in self.ins[op]:
            self.pins[u] -= 1
        if self.n22:
            for u in self.ins[op]:
                if self.dead[u] and self.resident[u] and self.pins[u] == 0 and not self.unev[u]:
                    a = self.clear(u)
                    self.events.append((4, self.cur_op, u, a))

    def run(self):
        tr = self.tr
        status, fail_op = 0, -1
        lb = rb = 0
        try:
            for t in range(tr.n_tensors):
                if not tr.is_param[t]:
                    continue
                right = bool(self.flags & 2) and rb < lb
                a = self.fit(self.size[t], right)
                if a is None:
                    raise Unsat()
                self.put(t, a)
                if right:
                    rb += self.size[t]
                else:
                    lb += self.size[t]
                self.born[t] = True
                self.events.append((0, -1, t, a))
            for k in range(tr.n_ops):
                self.cur_op = k
                o = int(tr.out[k])
                for u in self.ins[k]:
                    self.pins[u] += 1
                for u in self.locks[k]:
                    self.locked[u] = True
                for u in self.ins[k]:
                    if not self.resident[u]:
                        self.materialize(u, 0)
                for u in self.locks[k]:
                    if not self.resident[u]:
                        self.materialize(u, 0)
                self.allocate(k, o, True, 1)
                self.born[o] = True
                self.clock += self.cost[k]
                self.c["base_us"] += self.cost[k]
                self.c["total_us"] += self.cost[k]
                self.events.append((6, k, o, self.addr[o]))
                for u in self.ins[k]:
                    self.last_access[u] = self.clock
                self.last_access[o] = self.clock
                for u in self.ins[k]:
                    self.pins[u] -= 1
                src = int(tr.inplace_src[k])
                for t in range(tr.n_tensors):
                    keep = self.unev[t] and t != src
                    if self.last_use[t] == k and not keep:
                        self.dead[t] = True
                    if self.dead[t] and self.resident[t] and not keep:
                        a = self.clear(t)
                        self.events.append((4, k, t, a))
        except Unsat:
            status, fail_op = -3, self.cur_op
        except Thrash:
            status, fail_op = -4, self.cur_op
        return status, fail_op
