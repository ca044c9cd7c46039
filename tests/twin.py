"""A second, independent, tiny simrd V2 written in Python with exact Fractions.

Test infrastructure. It differs from the C oracle on purpose where the paper
allows two readings, so agreement is evidence rather than repetition:

* staleness uses the paper's RATIO form stale = (clock - T) / clock,
  the C oracle uses the difference form -- reading C-2 says both give
  the same argmin;
* E(t) is always a literal per-candidate BFS;
* get_internal is the recursive pseudocode of P:213-245 with sets as lists.

It also supports enumerating every eviction choice (`chooser`) for the
brute-force optimality bound.
"""
from __future__ import annotations

import copy
from fractions import Fraction

INF = "inf"
NEG_INF = None   # last_access := -infinity (banish_V2)

H_DTR, H_DTR_EQ, H_LRU, H_SIZE, H_MSPS, H_LOCAL = range(6)
H_DTR_FULL, H_ESTAR = 7, 8


class OOM(Exception):
    pass


class Thrash(Exception):
    pass


class Twin:
    def __init__(self, heuristic=H_DTR, budget=1 << 62, thrash_kill=0, dealloc="v2"):
        self.h = heuristic
        self.dealloc = dealloc
        self.banished = []
        self.B = budget
        self.kill = thrash_kill
        self.P, self.C = [], []
        self.mem, self.cost, self.la = [], [], []
        self.m, self.once, self.rho, self.l = [], [], [], []
        self.pool = set()
        self.clock = 0
        self.M = 0
        self.peak = 0
        self.base = 0
        self.decisions = 0
        self.remats = 0
        self.computations = 0
        self.trace = []
        self.chooser = None
        # union-find: node -> [parent, cost, maxla]
        self.uf = []
        self.set_of = []

    # -- union-find ------------------------------------------------------
    def uf_new(self):
        self.uf.append([len(self.uf), 0, NEG_INF])
        return len(self.uf) - 1

    def find(self, x):
        while self.uf[x][0] != x:
            x = self.uf[x][0]
        return x

    def union(self, a, b):
        a, b = self.find(a), self.find(b)
        if a != b:
            self.uf[b][0] = a
            self.uf[a][1] += self.uf[b][1]
            self.uf[a][2] = _max_la(self.uf[a][2], self.uf[b][2])

    # -- metadata ----------------------------------------------------------
    def evicted(self, x):
        return (not self.m[x]) and self.once[x] and not self.banished[x]

    def E(self, t):
        seen = {t}
        stack = [t]
        out = set()
        while stack:
            x = stack.pop()
            for y in self.P[x] + self.C[x]:
                if y not in seen and self.evicted(y):
                    seen.add(y)
                    out.add(y)
                    stack.append(y)
        return out

    def estar(self, t):
        """e*(t): evicted ancestors through evicted deps, plus evicted descendants
        through evicted dependents."""
        out = set(self.eR(t))
        seen = {t}
        stack = [t]
        while stack:
            x = stack.pop()
            for c in self.C[x]:
                if c not in seen and self.evicted(c):
                    seen.add(c)
                    out.add(c)
                    stack.append(c)
        return out

    def eR(self, t):
        seen = {t}
        stack = [t]
        out = set()
        while stack:
            x = stack.pop()
            for p in self.P[x]:
                if p not in seen and self.evicted(p):
                    seen.add(p)
                    out.add(p)
                    stack.append(p)
        return out

    def stale(self, T):
        """Ratio form. Returns None for +infinity staleness."""
        if T is NEG_INF:
            return None
        return Fraction(self.clock - T, self.clock)

    def _stale_score(self, num, mem, T):
        st = self.stale(T)
        if st is None:
            return Fraction(0)
        if st == 0:
            return INF
        return Fraction(num) / (mem * st)

    def score(self, t):
        if self.h == H_DTR:
            E = self.E(t)
            num = self.cost[t] + sum(self.cost[s] for s in E)
            T = self.la[t]
            for s in E:
                T = _max_la(T, self.la[s])
            return self._stale_score(num, self.mem[t], T)
        if self.h == H_DTR_EQ:
            roots = {self.find(self.set_of[q]) for q in self.P[t] + self.C[t] if self.evicted(q)}
            num = self.cost[t] + sum(self.uf[r][1] for r in roots)
            T = self.la[t]
            for r in roots:
                T = _max_la(T, self.uf[r][2])
            return self._stale_score(num, self.mem[t], T)
        if self.h == H_LRU:
            st = self.stale(self.la[t])
            return Fraction(0) if st is None else (INF if st == 0 else 1 / st)
        if self.h == H_SIZE:
            return Fraction(1, self.mem[t])
        if self.h == H_MSPS:
            return Fraction(self.cost[t] + sum(self.cost[s] for s in self.eR(t)), self.mem[t])
        if self.h == H_LOCAL:
            return self._stale_score(self.cost[t], self.mem[t], self.la[t])
        if self.h == H_DTR_FULL:
            num = self.cost[t] + sum(self.cost[s] for s in self.estar(t))
            return self._stale_score(num, self.mem[t], self.la[t])
        if self.h == H_ESTAR:
            return Fraction(self.cost[t] + sum(self.cost[s] for s in self.estar(t)), self.mem[t])
        if 16 <= self.h < 32:       # h'(s, m, c) = c / (m * s), ablated measures = 1
            code = self.h - 16
            kind, use_m, use_s = code >> 2, (code >> 1) & 1, code & 1
            if kind == 0:
                c = self.cost[t] + sum(self.cost[s] for s in self.estar(t))
            elif kind == 1:
                roots = {self.find(self.set_of[q]) for q in self.P[t] + self.C[t] if self.evicted(q)}
                c = self.cost[t] + sum(self.uf[r][1] for r in roots)
            elif kind == 2:
                c = self.cost[t]
            else:
                c = 1
            m = self.mem[t] if use_m else 1
            return self._stale_score(c, m, self.la[t]) if use_s else Fraction(c, m)
        raise ValueError(self.h)

    def uses_uf(self):
        return self.h == H_DTR_EQ or (16 <= self.h < 32 and (self.h - 16) >> 2 == 1)

    # -- internal API -------------------------------------------
    def evict(self, t):
        self.m[t] = False
        self.M -= self.mem[t]
        self.pool.discard(t)
        if self.uses_uf():
            r = self.find(self.set_of[t])
            self.uf[r][1] += self.cost[t]
            self.uf[r][2] = _max_la(self.uf[r][2], self.la[t])
            for q in self.P[t] + self.C[t]:
                if self.evicted(q):
                    self.union(self.set_of[t], self.set_of[q])

    def free(self, size):
        while self.M + size > self.B:
            if not self.pool:
                raise OOM()
            cands = sorted(self.pool)
            if self.chooser is not None:
                t = self.chooser(self, cands)
            else:
                t = min(cands, key=lambda x: (_key(self.score(x)), x))
            self.trace.append((self.clock, t))
            self.decisions += 1
            self.evict(t)

    def release_internal(self, t):
        self.l[t] -= 1
        if self.l[t] == 0 and not self.banished[t]:
            self.pool.add(t)
        self.maybe_banish(t)

    def maybe_banish(self, t):
        """V1: rho = 0 and every child material -> banish."""
        if self.dealloc != "v1" or self.banished[t] or self.rho[t] != 0:
            return
        if not all(self.m[c] for c in self.C[t]):
            return
        if self.m[t]:
            self.m[t] = False
            self.M -= self.mem[t]
            self.pool.discard(t)
        elif self.uses_uf() and self.evicted(t):
            r = self.find(self.set_of[t])
            self.uf[r][1] -= self.cost[t]
        self.banished[t] = True
        for c in self.C[t]:
            self.l[c] += 1
            self.pool.discard(c)
            self.P[c].remove(t)
        for p in self.P[t]:
            self.C[p].remove(t)
        self.C[t] = []
        self.P[t] = []

    def get_internal(self, t):
        if self.m[t]:
            self.l[t] += 1
            self.pool.discard(t)
            return
        Pt = [p for p in self.P[t] if self.m[p]]
        Pb = [p for p in self.P[t] if not self.m[p]]
        for p in Pt:
            self.get_internal(p)
        for p in Pb:
            self.get_internal(p)
        if self.M + self.mem[t] > self.B:
            self.free(self.mem[t])
        self.m[t] = True
        self.l[t] = 1
        self.M += self.mem[t]
        self.peak = max(self.peak, self.M)
        self.clock += self.cost[t]
        self.computations += 1
        if self.once[t]:
            self.remats += 1
            if self.uses_uf():
                r = self.find(self.set_of[t])
                self.uf[r][1] -= self.cost[t]
                self.set_of[t] = self.uf_new()
        else:
            self.once[t] = True
            if self.uses_uf():
                self.set_of[t] = self.uf_new()
        if self.kill and self.clock > self.kill * self.base:
            raise Thrash()
        for p in list(self.P[t]):      # a V1 banish removes p from t.P mid-loop (reading C-22)
            self.release_internal(p)

    # -- external API -------------------------------------------
    def make(self, mem, cost, parents):
        ps = []
        for p in parents:
            if p not in ps:
                ps.append(p)
        t = len(self.mem)
        self.P.append(ps)
        self.C.append([])
        self.mem.append(mem)
        self.cost.append(cost)
        self.la.append(self.clock)
        self.m.append(False)
        self.once.append(False)
        self.rho.append(1)
        self.l.append(0)
        self.set_of.append(None)
        self.banished.append(False)
        self.base += cost
        for p in ps:
            self.C[p].append(t)
            self.la[p] = self.clock
            if self.uses_uf() and self.evicted(p):
                r = self.find(self.set_of[p])
                self.uf[r][2] = _max_la(self.uf[r][2], self.clock)
        self.get_internal(t)
        self.release_internal(t)
        return t

    def get(self, t):
        assert self.rho[t] > 0
        self.rho[t] += 1

    def release(self, t):
        assert self.rho[t] > 0
        self.rho[t] -= 1
        if self.rho[t] != 0:
            return
        if self.dealloc == "v2":
            self.la[t] = NEG_INF
        elif self.dealloc == "v1":
            self.maybe_banish(t)
        elif self.dealloc == "eager" and t in self.pool:
            self.evict(t)

    def rematerialize(self, t):
        assert not self.m[t] and not self.banished[t]
        self.get_internal(t)
        self.release_internal(t)

    def ensure(self, t):
        assert not self.banished[t]
        self.get_internal(t)


def _max_la(a, b):
    if a is NEG_INF:
        return b
    if b is NEG_INF:
        return a
    return max(a, b)


def _key(s):
    # +infinity sorts last; Fractions compare exactly
    return (1, 0) if s == INF else (0, s)


def replay_log(view, heuristic, budget, thrash_kill=0, chooser=None, dealloc="v2"):
    """Replay a decoded log (dtr_inputs.LogView). Returns (twin, status)."""
    from dtr_inputs.logfmt import (OP_MAKE, OP_GET, OP_RELEASE, OP_REMAT, OP_ENSURE, OP_DEBUG_EVICT,
                                   OP_SHIFT, ID_MASK)
    tw = Twin(heuristic, budget, thrash_kill, dealloc)
    tw.chooser = chooser
    status = "ok"
    try:
        for w in view.ops:
            op, i = int(w) >> OP_SHIFT, int(w) & ID_MASK
            if op == OP_MAKE:
                tw.make(int(view.mem[i]), int(view.cost[i]), view.parents(i))
            elif op == OP_GET:
                tw.get(i)
            elif op == OP_RELEASE:
                tw.release(i)
            elif op == OP_REMAT:
                tw.rematerialize(i)
            elif op == OP_ENSURE:
                tw.ensure(i)
            elif op == OP_DEBUG_EVICT:
                tw.evict(i)
    except OOM:
        status = "oom"
    except Thrash:
        status = "thrash"
    return tw, status


def brute_force_min_clock(view, budget, limit_leaves=200000):
    """Enumerate every eviction choice at every free() iteration (simrd semantics,
    any choice rule) and return (min final clock over non-OOM leaves, leaves).
    A lower bound on what any heuristic can achieve within simrd."""
    import itertools

    best = [None]
    leaves = [0]

    class Choice(Exception):
        def __init__(self, cands):
            self.cands = cands

    def run(prefix):
        it = iter(prefix)

        def chooser(tw, cands):
            try:
                return next(it)
            except StopIteration:
                raise Choice(cands)

        try:
            tw, status = replay_log(view, H_SIZE, budget, chooser=chooser)
        except Choice as c:
            for x in c.cands:
                run(prefix + [x])
            return
        leaves[0] += 1
        if leaves[0] > limit_leaves:
            raise RuntimeError("too many leaves")
        if status == "ok" and (best[0] is None or tw.clock < best[0]):
            best[0] = tw.clock

    run([])
    return best[0], leaves[0]
