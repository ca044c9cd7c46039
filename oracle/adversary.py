"""The Theorem 2 adversary (App. B) driven through the
CPU oracle's per-call runtime, plus the path-sequential static baseline
(P:2093-2096).

TEST INFRASTRUCTURE ONLY: imported by tests/ and bench.py's cpu_baseline /
`--impl reference` legs; the product package never imports it.

Construction, in the paper's order (readings C-24 in DESIGN.md):
  1. t0 = f() with unit size and cost; "by the behavior of DTR, [it] must
     remain in memory" -- realised as one ENSURE (a lock that is never
     released).  t0 holds one of the B memory units, leaving "B - 1 units of
     memory to allocate among its descendants".
  2. t0's B children t1 ... tB are revealed in order (steps 1 ... B); each
     starts a path.
  3. Afterwards, after every step, the adversary inspects residency, takes a
     path from t0 whose nodes are all non-resident (one exists: B paths share
     B - 1 units) -- the lowest-indexed one -- and reveals the next node as
     the child of that path's last node, "causing DTR to rematerialize the
     entire path".  This repeats until all N nodes (t0
     included) are revealed.
Every node has unit size and cost, and the user keeps every reference (no
RELEASE).  The static algorithm computes one path at a time: N computations.
"""
from __future__ import annotations

import numpy as np

from . import oracle as O

NONE = 0xFFFFFFFF


def run_adversary(N: int, B: int, heuristic: int, seed: int = 0, trace_cap: int = 0, dealloc: int = 0):
    """Returns (result_row, parents[N] (NONE for t0), path_of[N] (NONE for t0), trace)."""
    if B < 3 or N < 1:
        raise ValueError("the construction needs N >= 1 and B >= 3 (t0, a parent and a child resident)")
    rt = O.Runtime(heuristic, budget=B, seed=seed, trace_cap=trace_cap, dealloc=dealloc)
    parents = np.full(N, NONE, dtype=np.uint32)
    path_of = np.full(N, NONE, dtype=np.uint32)
    rc, t0 = rt.compute(1, 1, [])                              # step 1: t0
    if rc == 0:
        rc = rt.ensure(t0)                                     # t0 must remain in memory
    tails = []
    while rc == 0 and rt.state()["n"] < N:
        n = rt.state()["n"]
        if len(tails) < B:                                     # t0's B children
            j, p = len(tails), t0
        else:                                                  # the lowest fully evicted path
            fl = rt.tensors()[0]
            resident = np.zeros(B, dtype=bool)
            for t in range(1, n):
                if fl[t] & 1:
                    resident[path_of[t]] = True
            free = np.flatnonzero(~resident)
            assert len(free) > 0, "B paths share B - 1 units: one path has no resident node"
            j = int(free[0])
            p = tails[j]
        rc, t = rt.compute(1, 1, [p])
        if rc != 0:
            break
        parents[t] = p
        path_of[t] = j
        if j == len(tails):
            tails.append(t)
        else:
            tails[j] = t
    return rt.result(), parents, path_of, rt.trace()


def path_lengths(path_of: np.ndarray, B: int) -> np.ndarray:
    p = path_of[path_of != NONE]
    return np.bincount(p.astype(np.int64), minlength=B)


def dynamic_cost_closed_form(lengths) -> int:
    """App. B's cost sum: t0 once, plus sum_j sum_{i=1}^{L_j} i = sum_j L_j (L_j + 1) / 2."""
    return 1 + sum(int(L) * (int(L) + 1) // 2 for L in lengths)


def static_log(parents: np.ndarray, path_of: np.ndarray):
    """The revealed graph in the static path-at-a-time order as a
    log: t0, ENSURE t0, then every path's nodes in path order.  Ids are
    renumbered in that order; returns the log words."""
    from dtr_inputs.logfmt import LogBuilder
    N = len(parents)
    B = int(path_of[path_of != NONE].max()) + 1 if N > 1 else 0
    b = LogBuilder(model_id=0, seed=0)
    new = {0: b.make(1, 1, [])}
    b.ensure(new[0])
    for j in range(B):
        for t in np.flatnonzero(path_of == j):
            t = int(t)
            new[t] = b.make(1, 1, [new[int(parents[t])]])
    return b.build()
