"""Pins of the C oracle against what the paper and mathematics fix (not against itself)."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from dtr_inputs import LogBuilder, LogView, models
import twin as TW

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def build_fixture(O, g, heuristic=0, mems=None):
    rt = O.Runtime(heuristic)
    for i, ps in enumerate(g["parents"]):
        rc, t = rt.compute(mems[i] if mems else 1, 1, ps)
        assert rc == 0 and t == i
    for t in g["evict"]:
        assert rt.debug_evict(t) == 0
    return rt


def frac(nd):
    n, d = nd
    return math.inf if d == 0 else Fraction(n, d)


# ---------------------------------------------------------------- worked examples

def test_worked_example_E_t4_undirected(oracle_mod):
    g = gold("simrd_fig_compheur.json")
    rt = build_fixture(oracle_mod, g)
    for t, exp in g["expect_E"].items():
        assert rt.neighbourhood(int(t)) == exp
    # the directed closure (ancestors+descendants through evicted tensors) differs,
    # so the fixture distinguishes the undirected reading (C-1)
    par = g["parents"]
    ch = [[c for c in range(len(par)) if p in par[c]] for p in range(len(par))]
    ev = set(g["evict"])

    def closure(t, nbr):
        out, st = set(), [t]
        while st:
            x = st.pop()
            for y in nbr[x]:
                if y in ev and y not in out:
                    out.add(y)
                    st.append(y)
        return out
    for t, exp in g["expect_directed_estar"].items():
        d = closure(int(t), par) | closure(int(t), ch)
        assert sorted(d) == exp
        assert sorted(d) != g["expect_E"][t]


def test_worked_example_doc_c_estar(oracle_mod):
    g = gold("dtr_fig1_estar.json")
    rt = build_fixture(oracle_mod, g)
    for t, exp in g["expect_E"].items():
        assert rt.neighbourhood(int(t)) == exp
    for t, exp in g["expect_estar"].items():      # the directed e* of the paper's example
        assert rt.estar(int(t)) == exp


def test_estar_directed_differs_from_undirected(oracle_mod):
    g = gold("simrd_fig_compheur.json")
    rt = build_fixture(oracle_mod, g)
    for t, exp in g["expect_directed_estar"].items():
        assert rt.estar(int(t)) == exp


def test_dtr_full_and_estar_scores_hand(oracle_mod):
    """T_B at clock 7 (la = {t0:3, t2:2, t3:4, t4:4}): directed e*(t0) = {t1, t5, t6}
    (descendants t1 -> t5 -> t6), e*(t2) = {t1}, e*(t3) = {}, e*(t4) = {t1}.
    h_DTR_full = (c + sum e*) / (m * (clock - la(t)));
    h_e* = (c + sum e*) / m = |e*| + 1 under unit costs."""
    g = gold("hdtr_T_B_clock7.json")
    rt = build_fixture(oracle_mod, g, heuristic=oracle_mod.H_DTR_FULL)
    assert {k: frac(v) for k, v in rt.scores().items()} == {0: Fraction(4, 4), 2: Fraction(2, 5),
                                                            3: Fraction(1, 3), 4: Fraction(2, 3)}
    rt = build_fixture(oracle_mod, g, heuristic=oracle_mod.H_ESTAR)
    sc = rt.scores()
    assert {k: frac(v) for k, v in sc.items()} == {0: 4, 2: 2, 3: 1, 4: 2}
    for k in sc:                                    # corollary: |e*| + 1 with unit costs
        assert frac(sc[k]) == len(rt.estar(k)) + 1


def test_hdtr_scores_hand_derived(oracle_mod):
    g = gold("hdtr_T_B_clock7.json")
    for e_mode in (0, 1):
        rt = oracle_mod.Runtime(0, e_mode=e_mode)
        for ps in g["parents"]:
            rt.compute(1, 1, ps)
        for t in g["evict"]:
            rt.debug_evict(t)
        assert rt.state()["clock"] == g["clock"]
        got = {str(k): frac(v) for k, v in rt.scores().items()}
        assert got == {k: frac(v) for k, v in g["expect_scores"].items()}


def test_v2_banish_zero(oracle_mod):
    g = gold("hdtr_T_B_clock7.json")
    rt = build_fixture(oracle_mod, g)
    assert rt.release(3) == 0
    assert frac(rt.scores()[3]) == frac(g["v2_release"]["release_3_expect"]) == 0
    assert rt.release(2) == 0
    assert frac(rt.scores()[2]) == frac(g["v2_release"]["release_2_expect"]) == 4


def test_staleness_zero_and_tiebreak(oracle_mod):
    g = gold("hdtr_T_B_clock7.json")
    s0 = g["staleness0"]
    rt = build_fixture(oracle_mod, g)
    rt.set_budget(s0["budget"])
    rc, t = rt.compute(1, 1, s0["make_parents"])
    assert rc == 0
    tr = rt.trace()
    assert [[int(r["clock"]), int(r["id"])] for r in tr] == s0["expect_trace"]
    assert rt.state()["clock"] == s0["expect_clock"]
    # the tie at clock 9: t0's score equals t4's exactly, and t0 wins on id
    at9 = [r for r in tr if int(r["clock"]) == 9][0]
    assert Fraction(int(at9["num"]), int(at9["den"])) == Fraction(2, 5)


def test_staleness_zero_distinguishing(oracle_mod):
    g = gold("hdtr_T_B_clock7.json")
    d = g["distinguishing"]
    mems = [1] * 7
    mems[2] = d["mem_t2"]
    rt = build_fixture(oracle_mod, g, mems=mems)
    rt.set_budget(rt.state()["M"])
    rt.compute(1, 1, [6])
    tr = rt.trace()
    assert [int(tr[0]["clock"]), int(tr[0]["id"])] == d["expect_first"]


def test_msps_chain_hand(oracle_mod):
    # S1(ev, c=2) -> S2(ev, c=3) -> S3(resident, m=4): h_MSPS(S3) = (1 + 2 + 3) / 4
    rt = oracle_mod.Runtime(oracle_mod.H_MSPS)
    rt.compute(1, 2, [])
    rt.compute(1, 3, [0])
    rt.compute(4, 1, [1])
    rt.debug_evict(0)
    rt.debug_evict(1)
    assert frac(rt.scores()[2]) == Fraction(6, 4)


# ---------------------------------------------------------------- closed forms

ALL_H = ["dtr", "dtr_eq", "lru", "size", "msps", "local", "random", "dtr_full", "estar"]


@pytest.mark.parametrize("model", ["resnet32", "unet", "densenet100"])
def test_unlimited_budget(oracle_mod, model):
    v = LogView(models.CONFIG_MODELS[model]())
    for h in ALL_H:
        r, _ = oracle_mod.replay(v.words, oracle_mod.HEURISTICS[h], v.peak_total)
        assert r["status"] == 0
        assert r["decisions"] == 0 and r["remats"] == 0
        assert r["clock"] == v.base == r["base"]
        assert r["computations"] == v.n


def test_linear_forward_exactly_N(oracle_mod):
    N = 30
    b = LogBuilder()
    t = b.make(1, 1, [])
    for i in range(1, N):
        t = b.make(1, 1, [t])
    w = b.build()
    fo = gold("linear_appendix_a.json")["forward_only"]
    for h in ALL_H:
        for B in (2, 3, 8):
            r, _ = oracle_mod.replay(w, oracle_mod.HEURISTICS[h], B)
            assert r["status"] == 0 and r["computations"] == N and r["remats"] == 0
    # LRU / size: FIFO eviction keeps the last B tensors (closed form)
    for h in ("lru", "size"):
        rt = oracle_mod.Runtime(oracle_mod.HEURISTICS[h], budget=fo["B"])
        t = rt.compute(1, 1, [])[1]
        for i in range(1, fo["N"]):
            t = rt.compute(1, 1, [t])[1]
        fl, *_ = rt.tensors()
        assert [i for i in range(fo["N"]) if fl[i] & 1] == fo["lru_size_resident"]


def test_linear_theorem1_bound(oracle_mod):
    g = gold("linear_appendix_a.json")
    ratios = {}
    for N in g["Ns"]:
        B = 2 * math.ceil(math.sqrt(N))
        r, _ = oracle_mod.replay(models.linear(N), oracle_mod.H_DTR, B, thrash_kill=0)
        assert r["status"] == 0
        ratios[N] = int(r["clock"]) / (2 * N)
    for N in g["Ns"]:
        assert ratios[N] <= g["proxy_factor"] * ratios[64], ratios


def test_oom_closed_form(oracle_mod):
    # B below the largest single op's inputs + output -> OOM.
    w = models.linear(16)
    r, _ = oracle_mod.replay(w, oracle_mod.H_DTR, 2, thrash_kill=0)
    assert r["status"] == oracle_mod.OOM
    r, _ = oracle_mod.replay(w, oracle_mod.H_DTR, 3, thrash_kill=0)
    assert r["status"] == 0
    v = LogView(models.resnet32())
    need = max(sum(int(v.mem[p]) for p in v.parents(t)) + int(v.mem[t]) for t in range(v.n))
    r, _ = oracle_mod.replay(v.words, oracle_mod.H_DTR, need - 1, thrash_kill=0)
    assert r["status"] == oracle_mod.OOM


# ---------------------------------------------------------------- brute force

@pytest.mark.parametrize("N,B,exp_min", [(4, 3, 9), (5, 3, 13), (6, 3, 18)])
def test_bruteforce_linear_lower_bound(oracle_mod, N, B, exp_min):
    w = models.linear(N)
    v = LogView(w)
    best, leaves = TW.brute_force_min_clock(v, B)
    assert best == exp_min
    r, _ = oracle_mod.replay(w, oracle_mod.H_DTR, B, thrash_kill=0)
    assert r["clock"] >= best


def test_bruteforce_random_lower_bound(oracle_mod):
    checked = 0
    for seed in range(40):
        w = models.random_program(8, seed=seed, mem_max=3, cost_max=3, p_release=0.25)
        v = LogView(w)
        B = max(3, v.peak_live * 6 // 10)
        try:
            best, leaves = TW.brute_force_min_clock(v, B, limit_leaves=20000)
        except RuntimeError:
            continue
        for h in ("dtr", "dtr_eq", "lru", "msps"):
            r, tr = oracle_mod.replay(w, oracle_mod.HEURISTICS[h], B, thrash_kill=0, trace_cap=1000)
            if best is None:
                assert r["status"] == oracle_mod.OOM
            elif r["status"] == 0:
                assert r["clock"] >= best
        checked += 1
    assert checked >= 20


# ---------------------------------------------------------------- independent twin (ratio staleness)

TWIN_H = {"dtr": TW.H_DTR, "dtr_eq": TW.H_DTR_EQ, "lru": TW.H_LRU, "size": TW.H_SIZE,
          "msps": TW.H_MSPS, "local": TW.H_LOCAL, "dtr_full": TW.H_DTR_FULL, "estar": TW.H_ESTAR}


@pytest.mark.parametrize("h", list(TWIN_H))
def test_twin_ratio_staleness_agrees(oracle_mod, h):
    """Reading C-2: the ratio form (twin) and the difference form (P:2223,
    oracle) give the same trace."""
    cases = [models.random_program(30, seed=s, p_release=0.3) for s in range(25)]
    cases.append(models.linear(24))
    for w in cases:
        v = LogView(w)
        for frac_b in (0.4, 0.6, 0.8):
            B = max(4, int(v.peak_live * frac_b))
            tw, status = TW.replay_log(v, TWIN_H[h], B)
            r, tr = oracle_mod.replay(w, oracle_mod.HEURISTICS[h], B, thrash_kill=0, trace_cap=100000)
            st = {0: "ok", oracle_mod.OOM: "oom"}[int(r["status"])]
            assert st == status
            assert [(int(x["clock"]), int(x["id"])) for x in tr] == tw.trace
            if status == "ok":
                assert int(r["clock"]) == tw.clock and int(r["remats"]) == tw.remats
                assert int(r["peak_M"]) == tw.peak


def test_e_modes_agree(oracle_mod):
    for s in range(10):
        w = models.random_program(60, seed=100 + s, p_release=0.3)
        v = LogView(w)
        B = max(4, v.peak_live // 2)
        a, ta = oracle_mod.replay(w, 0, B, e_mode=0, trace_cap=10 ** 5)
        b, tb = oracle_mod.replay(w, 0, B, e_mode=1, trace_cap=10 ** 5)
        assert a.tobytes() == b.tobytes() and ta.tobytes() == tb.tobytes()


# ---------------------------------------------------------------- invariants

def step_log(O, w, heuristic, B):
    """Per-record replay through the per-call API, yielding the runtime after each record."""
    from dtr_inputs.logfmt import OP_MAKE, OP_GET, OP_RELEASE, OP_ENSURE, OP_SHIFT, ID_MASK
    v = LogView(w)
    rt = O.Runtime(heuristic, budget=B)
    for word in v.ops:
        op, i = int(word) >> OP_SHIFT, int(word) & ID_MASK
        if op == OP_MAKE:
            rc, _ = rt.compute(int(v.mem[i]), int(v.cost[i]), v.parents(i))
        elif op == OP_GET:
            rc = rt.get(i)
        elif op == OP_RELEASE:
            rc = rt.release(i)
        elif op == OP_ENSURE:
            rc = rt.ensure(i)
        if rc != 0:
            return
        yield rt, v


def test_runtime_audits(oracle_mod):
    """M = sum of material mem; M <= B; pool == {m and l == 0}."""
    for s in range(8):
        w = models.random_program(50, seed=200 + s, p_release=0.3)
        B = max(4, LogView(w).peak_live // 2)
        for rt, v in step_log(oracle_mod, w, 0, B):
            st = rt.state()
            fl, rho, ell, la = rt.tensors()
            n = st["n"]
            mat = fl & 1
            assert st["M"] == int(sum(int(v.mem[t]) for t in range(n) if mat[t]))
            assert st["M"] <= B
            pool = (fl >> 2) & 1
            assert np.array_equal(pool.astype(bool), (mat == 1) & (ell == 0))


def test_uf_conservation_and_prefix_equivalence(oracle_mod):
    """UF: sum of root costs == sum of evicted costs;
    root maxla >= true member max (reading C-9). h_DTR_eq == h_DTR until the
    first completed remat (no phantoms yet) on release-free programs."""
    for s in range(12):
        w = models.random_program(50, seed=300 + s, p_release=0.3)
        B = max(4, LogView(w).peak_live // 2)
        for rt, v in step_log(oracle_mod, w, oracle_mod.H_DTR_EQ, B):
            fl, rho, ell, la = rt.tensors()
            ev = [t for t in range(len(fl)) if (fl[t] & 3) == 2]
            assert rt.uf_root_cost_sum() == sum(int(v.cost[t]) for t in ev)
            root_of, root_cost, root_maxla = rt.uf_roots()
            for t in ev:
                assert root_maxla[t] >= la[t]
    for s in range(12):
        w = models.random_program(50, seed=400 + s, p_release=0.0)
        v = LogView(w)
        B = max(4, v.peak_live // 2)
        tw, _ = TW.replay_log(v, TW.H_DTR, B)
        # decisions made before the first completed remat
        first = None
        for rt, _v in step_log(oracle_mod, w, 0, B):
            st = rt.state()
            if st["remats"] > 0:
                break
            first = st["decisions"]
        D = first or 0
        a, ta = oracle_mod.replay(w, 0, B, trace_cap=10 ** 5)
        b, tb = oracle_mod.replay(w, oracle_mod.H_DTR_EQ, B, trace_cap=10 ** 5)
        assert ta[:D].tobytes() == tb[:D].tobytes()


@pytest.mark.parametrize("h", ALL_H)
def test_metamorphic_scaling(oracle_mod, h):
    """compute x k => same trace ids and clock x k; mem x k with B x k => same trace."""
    for s in range(6):
        b0 = models.random_program(40, seed=500 + s, p_release=0.3)
        v = LogView(b0)
        B = max(4, v.peak_live // 2)
        ref, tr = oracle_mod.replay(b0, oracle_mod.HEURISTICS[h], B, thrash_kill=0, trace_cap=10 ** 5)
        for k in (3, 5):
            w = b0.copy()
            o = 16 + v.n
            w[o:o + v.n] *= k                      # compute x k
            r, t2 = oracle_mod.replay(w, oracle_mod.HEURISTICS[h], B, thrash_kill=0, trace_cap=10 ** 5)
            assert list(t2["id"]) == list(tr["id"]) and r["status"] == ref["status"]
            assert int(r["clock"]) == k * int(ref["clock"])
            w = b0.copy()
            w[16:16 + v.n] *= k                    # mem x k, B x k
            r, t3 = oracle_mod.replay(w, oracle_mod.HEURISTICS[h], B * k, thrash_kill=0, trace_cap=10 ** 5)
            assert list(t3["id"]) == list(tr["id"]) and r["status"] == ref["status"]


def test_argmin_exact_vs_bigint(oracle_mod):
    """The evicted tensor is the exact lexicographic min of (num/den, id) over the
    pool scores, checked with Python big integers (reading C-5)."""
    for s in range(10):
        w = models.random_program(40, seed=600 + s, p_release=0.3, mem_max=50, cost_max=1000)
        v = LogView(w)
        B = max(60, v.peak_live // 2)
        from dtr_inputs.logfmt import OP_MAKE, OP_SHIFT, ID_MASK
        rt = oracle_mod.Runtime(0, budget=B)
        for word in v.ops:
            op, i = int(word) >> OP_SHIFT, int(word) & ID_MASK
            if op != OP_MAKE:
                {2: rt.get, 3: rt.release, 5: rt.ensure}[op](i)
                continue
            before = rt.state()["decisions"]
            sc = rt.scores()
            need = rt.state()["M"] + int(v.mem[i]) > B and not any(
                not (rt.tensors()[0][p] & 1) for p in v.parents(i))
            rc, _ = rt.compute(int(v.mem[i]), int(v.cost[i]), v.parents(i))
            if need and rt.state()["decisions"] > before and sc:
                first = rt.trace()[before]
                # parents were locked before free(): they are not candidates
                cands = {t: nd for t, nd in sc.items() if t not in v.parents(i)}
                best = min(cands, key=lambda t: (frac(cands[t]), t))
                assert int(first["id"]) == best
            if rc != 0:
                break


def test_determinism(oracle_mod):
    w = models.resnet32()
    v = LogView(w)
    for h in ALL_H:
        a, ta = oracle_mod.replay(w, oracle_mod.HEURISTICS[h], v.budget(400), trace_cap=10 ** 6)
        b, tb = oracle_mod.replay(w, oracle_mod.HEURISTICS[h], v.budget(400), trace_cap=10 ** 6)
        assert a.tobytes() == b.tobytes() and ta.tobytes() == tb.tobytes()


# ---------------------------------------------------------------- deallocation policies (NEXT #2)

def test_gap_lemma_estar(oracle_mod):
    """After the forward pass of the linear net with B = 2*ceil(sqrt N), h_e* leaves
    resident tensors no more than 2(N-2)/(B-1) apart; h_DTR_full / LRU do not."""
    g = gold("theorem1_estar_v1.json")
    for N in g["Ns"]:
        B = 2 * math.ceil(math.sqrt(N))
        gaps = {}
        for h in ("estar", "lru"):
            rt = oracle_mod.Runtime(oracle_mod.HEURISTICS[h], budget=B, dealloc=1)
            t = rt.compute(1, 1, [])[1]
            for i in range(2, N + 1):
                t = rt.compute(1, 1, [t])[1]
            fl, *_ = rt.tensors()
            pts = [-1] + [i for i in range(N) if fl[i] & 1]     # the input t0 is always resident
            gaps[h] = max(b - a for a, b in zip(pts, pts[1:]))
        assert gaps["estar"] <= 2 * (N - 2) / (B - 1), (N, gaps)
        if N >= 64:
            assert gaps["lru"] > 2 * (N - 2) / (B - 1)


def test_theorem1_estar_v1(oracle_mod):
    """Theorem 1 with V1 banishing: h_e* needs O(N) operations at
    B = 2*ceil(sqrt N) -- C(N)/2N stays below a constant while LRU grows."""
    g = gold("theorem1_estar_v1.json")
    for N in g["Ns"]:
        B = 2 * math.ceil(math.sqrt(N))
        r, _ = oracle_mod.replay(models.linear(N), oracle_mod.H_ESTAR, B, thrash_kill=0, dealloc=1)
        assert r["status"] == 0 and int(r["clock"]) / (2 * N) <= g["ratio_bound"], (N, int(r["clock"]))
        if N >= g["lru_exceeds_from"]:
            r, _ = oracle_mod.replay(models.linear(N), oracle_mod.H_LRU, B, thrash_kill=0, dealloc=1)
            assert int(r["clock"]) / (2 * N) > g["ratio_bound"]


def test_v1_banish_semantics(oracle_mod):
    """banish_V1: t0 = f(); t1 = f(t0); release(t0) with its only child
    material -> t0 evicted (M drops), t1 pinned (out of the pool), t0 gone from the
    graph; a banished tensor never returns to the pool."""
    rt = oracle_mod.Runtime(oracle_mod.H_DTR, dealloc=1)
    rt.compute(1, 1, [])
    rt.compute(1, 1, [0])
    assert rt.state()["M"] == 2
    assert rt.release(0) == 0
    fl, rho, ell, la = rt.tensors()
    assert rt.state()["M"] == 1
    assert (fl[0] & 1) == 0 and (fl[0] & 4) == 0          # not material, not in pool
    assert (fl[1] & 4) == 0 and ell[1] == 1                # pinned
    rt.compute(1, 1, [1])                                  # t2 = f(t1): t1 stays pinned
    fl, rho, ell, la = rt.tensors()
    assert (fl[1] & 4) == 0 and (fl[2] & 4) == 4
    # not banished while a child is evicted: t3 = f(t2), t4 = f(t3); evict t3; release t2
    rt2 = oracle_mod.Runtime(oracle_mod.H_DTR, dealloc=1)
    for ps in ([], [0], [1]):
        rt2.compute(1, 1, ps)
    rt2.debug_evict(1)
    assert rt2.release(0) == 0
    fl, *_ = rt2.tensors()
    assert fl[0] & 1                                      # kept: child t1 is evicted


def test_v1_banish_inside_release_loop(oracle_mod):
    """get_internal releases every parent it locked, even when the
    first release banishes that parent and removes it from t.P:
    a = f(), b = f(), t = f(a, b); release a, b (t evicted, so neither is banished);
    rematerialize t -> release_internal(a) banishes a, release_internal(b) banishes b.
    Both pin t (l = 2) and only t stays resident (M = 1)."""
    for h in (oracle_mod.H_DTR, oracle_mod.H_DTR_EQ, oracle_mod.H_LRU):
        rt = oracle_mod.Runtime(h, dealloc=1)
        rt.compute(1, 1, [])
        rt.compute(1, 1, [])
        rt.compute(1, 1, [0, 1])
        assert rt.debug_evict(2) == 0
        assert rt.release(0) == 0 and rt.release(1) == 0
        fl, rho, ell, la = rt.tensors()
        assert fl[0] & 1 and fl[1] & 1                     # kept: child t is evicted
        assert rt.rematerialize(2) == 0
        fl, rho, ell, la = rt.tensors()
        assert [int(x) & 1 for x in fl] == [0, 0, 1]
        assert list(map(int, ell)) == [0, 0, 2]
        assert rt.state()["M"] == 1
        assert rt.rematerialize(0) == 2 and rt.ensure(1) == 2  # banished: PRECOND (reading C-22)


def test_v1_lock_balance(oracle_mod):
    """After a V1 replay, every lock is a pin: l(t) = #banished parents of t for every
    tensor still in the graph, pool = {material, l = 0, not banished}, M = sum of material mem."""
    from dtr_inputs.logfmt import OP_SHIFT, ID_MASK, OP_ENSURE
    done = 0
    for s in range(24):
        w = models.random_program(60, seed=900 + s, p_release=0.4, max_parents=4, n_ensure=0)
        v = LogView(w)
        rt = oracle_mod.Runtime(oracle_mod.H_DTR, budget=max(4, v.peak_live * 6 // 10), dealloc=1)
        rc = 0
        for word in v.ops:
            if rc != 0:
                break
            op, i = int(word) >> OP_SHIFT, int(word) & ID_MASK
            if op == 1:
                rc, t = rt.compute(int(v.mem[i]), int(v.cost[i]), v.parents(i))
            elif op == 2:
                rc = rt.get(i)
            elif op == 3:
                rc = rt.release(i)
        if rc == oracle_mod.OOM:
            continue
        assert rc == 0
        done += 1
        fl, rho, ell, la = rt.tensors()
        n = len(fl)
        banished = [bool(fl[t] & 8) for t in range(n)]
        for t in range(n):
            if banished[t]:          # banished => released, not material, computed once
                assert rho[t] == 0 and (fl[t] & 7) == 2
                continue
        for t in range(n):
            if banished[t]:          # its pins depend on which of t and its parent went first
                assert not fl[t] & 4
                continue
            pins = sum(1 for p in v.parents(t) if banished[p])
            assert int(ell[t]) == pins, (s, t)
            assert bool(fl[t] & 4) == (bool(fl[t] & 1) and ell[t] == 0)
        assert rt.state()["M"] == sum(int(v.mem[t]) for t in range(n) if fl[t] & 1)
    assert done >= 8


def test_eager_and_ignore_semantics(oracle_mod):
    """eager eviction: the last release evicts a pool member
    normally (it stays rematerializable); ignore: release changes nothing."""
    rt = oracle_mod.Runtime(oracle_mod.H_DTR, dealloc=2)
    rt.compute(1, 1, [])
    rt.compute(1, 1, [0])
    rt.release(0)
    fl, rho, ell, la = rt.tensors()
    assert (fl[0] & 3) == 2 and rt.state()["M"] == 1      # evicted, computed once
    assert rt.rematerialize(0) == 0 and rt.state()["remats"] == 1
    rt = oracle_mod.Runtime(oracle_mod.H_DTR, dealloc=3)
    rt.compute(1, 1, [])
    before = rt.tensors()[3][0]
    rt.release(0)
    fl, rho, ell, la = rt.tensors()
    assert fl[0] & 1 and la[0] == before and rt.state()["M"] == 1


@pytest.mark.parametrize("dealloc", ["v1", "eager", "ignore"])
def test_twin_agrees_dealloc(oracle_mod, dealloc):
    for h in ("dtr", "dtr_eq", "lru", "dtr_full", "estar"):
        for s in range(12):
            w = models.random_program(40, seed=700 + s, p_release=0.35)
            v = LogView(w)
            B = max(4, v.peak_live * 6 // 10)
            tw, status = TW.replay_log(v, TWIN_H[h], B, dealloc=dealloc)
            r, tr = oracle_mod.replay(w, oracle_mod.HEURISTICS[h], B, thrash_kill=0, trace_cap=10 ** 5,
                                      dealloc=oracle_mod.DEALLOC[dealloc])
            assert {0: "ok", oracle_mod.OOM: "oom"}[int(r["status"])] == status
            assert [(int(x["clock"]), int(x["id"])) for x in tr] == tw.trace, (h, s)


# ---------------------------------------------------------------- D.1 ablation h'(s, m, c) (reading C-23)

def test_ablation_scores_hand(oracle_mod):
    """Hand scores of h'(s,m,c) = c/(m s) on fixture T_B (tests/golden/ablation_T_B_clock7.json).
    EqClass and e* differ on t2 and t4: the union-find set of t1 also holds t5 and t6
    (a phantom connection), the directed e* does not."""
    g = gold("hdtr_T_B_clock7.json")
    a = gold("ablation_T_B_clock7.json")
    for name, exp in a["expect"].items():
        rt = build_fixture(oracle_mod, g, heuristic=oracle_mod.HEURISTICS["abl_" + name])
        got = {str(k): frac(v) for k, v in rt.scores().items()}
        assert got == {k: frac(v) for k, v in exp.items()}, name


def _same_trace(O, w, h1, h2, B):
    r1, t1 = O.replay(w, O.HEURISTICS[h1], B, thrash_kill=0, trace_cap=1 << 20)
    r2, t2 = O.replay(w, O.HEURISTICS[h2], B, thrash_kill=0, trace_cap=1 << 20)
    assert int(r1["status"]) == int(r2["status"])
    assert [(int(x["clock"]), int(x["id"])) for x in t1] == [(int(x["clock"]), int(x["id"])) for x in t2], (h1, h2)
    return int(r1["decisions"])


def test_ablation_reduces_to_named_heuristics(oracle_mod):
    """P:2527-2536 with measures ablated reduces to heuristics pinned elsewhere:
    h'(s,m,e*) = h_DTR_full, h'(no s, m, e*) = h_e* (P:1835-1837),
    h'(s,m,local) = h_DTR_local, h'(s, no m, no c) = LRU,
    h'(no s, m, no c) = largest-first. The eviction sequences match
    (the scores themselves may differ by a constant factor)."""
    pairs = [("abl_estar_ms", "dtr_full"), ("abl_estar_mx", "estar"), ("abl_local_ms", "local"),
             ("abl_no_xs", "lru"), ("abl_no_mx", "size")]
    dec = 0
    for s in range(6):
        w = models.random_program(80, seed=1300 + s, p_release=0.3, max_parents=4)
        v = LogView(w)
        for fr in (0.35, 0.6):
            for h1, h2 in pairs:
                dec += _same_trace(oracle_mod, w, h1, h2, max(3, int(v.peak_live * fr)))
    w = models.resnet32()
    v = LogView(w)
    for h1, h2 in pairs:
        dec += _same_trace(oracle_mod, w, h1, h2, v.budget(400))
    assert dec > 1000


def test_ablation_constant_score_evicts_smallest_id(oracle_mod):
    """h'(no s, no m, no c) = 1 for every candidate: by the id tie-break (C-5) each
    decision takes the smallest id in the pool -- the twin with a min-id chooser."""
    for s in range(8):
        w = models.random_program(60, seed=1400 + s, p_release=0.3)
        v = LogView(w)
        B = max(3, v.peak_live // 2)
        tw, status = TW.replay_log(v, TW.H_SIZE, B, chooser=lambda tw, c: min(c))
        r, tr = oracle_mod.replay(w, oracle_mod.HEURISTICS["abl_no_xx"], B, thrash_kill=0, trace_cap=10 ** 5)
        assert {0: "ok", oracle_mod.OOM: "oom"}[int(r["status"])] == status
        assert [(int(x["clock"]), int(x["id"])) for x in tr] == tw.trace


@pytest.mark.parametrize("c", ["estar", "eqclass", "local", "no"])
def test_ablation_twin_agrees(oracle_mod, c):
    """All 16 variants: the C oracle and the Fraction twin (ratio staleness) agree."""
    for m in "xm":
        for st in "xs":
            name = f"abl_{c}_{m}{st}"
            hid = oracle_mod.HEURISTICS[name]
            for s in range(8):
                w = models.random_program(50, seed=1500 + s, p_release=0.3, max_parents=3)
                v = LogView(w)
                B = max(4, v.peak_live * 5 // 10)
                for dealloc in ("v2", "v1"):
                    tw, status = TW.replay_log(v, hid, B, dealloc=dealloc)
                    r, tr = oracle_mod.replay(w, hid, B, thrash_kill=0, trace_cap=10 ** 5,
                                              dealloc=oracle_mod.DEALLOC[dealloc])
                    assert {0: "ok", oracle_mod.OOM: "oom"}[int(r["status"])] == status
                    assert [(int(x["clock"]), int(x["id"])) for x in tr] == tw.trace, (name, s, dealloc)
