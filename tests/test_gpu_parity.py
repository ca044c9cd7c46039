"""Parity of the CUDA path (through the C ABI) against the CPU oracle.

Bar (north_star): bit-identical eviction traces, rows (status, clock,
decisions, remats, computations, peak M, trace hash) on every config.
Everything here is integer: comparisons are exact equality.
"""
import math

import numpy as np
import pytest

from dtr_inputs import LogView, models

pytestmark = pytest.mark.gpu

ROW_FIELDS = ("status", "records_done", "clock", "base", "decisions", "remats", "computations", "peak_M",
              "trace_hash")
HS = ["dtr", "dtr_eq", "lru", "size", "msps", "local", "random", "dtr_full", "estar"]


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_09616_b200 as P
    return P


def oracle_runs(O, logs, specs, trace=True):
    out = []
    for s in specs:
        r, tr = O.replay(logs[s["log"]], O.HEURISTICS[s["h"]], s["budget"], seed=s.get("seed", 0),
                         thrash_kill=s.get("thrash_kill", 16), max_decisions=s.get("max_decisions", 0),
                         trace_cap=(1 << 22) if trace else 0, dealloc=O.DEALLOC[s.get("dealloc", "v2")])
        out.append((r, tr))
    return out


def gpu_batch(P, logs, specs, engine, trace_caps):
    spec2 = [dict(log=s["log"], budget=s["budget"], heuristic=P.HEURISTICS[s["h"]], seed=s.get("seed", 0),
                  thrash_kill=s.get("thrash_kill", 16), max_decisions=s.get("max_decisions", 0),
                  dealloc=P.DEALLOC[s.get("dealloc", "v2")]) for s in specs]
    b = P.DeviceBatch(logs, spec2, engine=engine, trace_caps=trace_caps)
    b.run()
    import torch
    torch.cuda.synchronize()
    rows = b.result_rows()
    tr = b.traces()
    return rows, [b.cell_trace(i, tr) if tr is not None else None for i in range(len(specs))]


def assert_parity(P, O, logs, specs, engine, check_trace=True):
    ref = oracle_runs(O, logs, specs, trace=check_trace)
    caps = [int(r["decisions"]) + 4 if check_trace else 0 for r, _ in ref]
    rows, trs = gpu_batch(P, logs, specs, engine, caps)
    for i, ((r, tr), g) in enumerate(zip(ref, rows)):
        for f in ROW_FIELDS:
            assert int(g[f]) == int(r[f]), (i, specs[i], f, int(g[f]), int(r[f]))
        if check_trace:
            gt = trs[i][: int(g["n_trace"])]
            assert int(g["n_trace"]) == int(r["decisions"])
            assert gt.tobytes() == tr.tobytes(), (i, specs[i])
    return rows


# ------------------------------------------------------------------ config 1

@pytest.mark.parametrize("engine", [1, 2])
def test_linear_config1(P, oracle_mod, engine):
    N = 64
    B = 2 * math.ceil(math.sqrt(N))
    logs = [models.linear(N)]
    specs = [dict(log=0, h=h, budget=B, thrash_kill=0) for h in HS]
    rows = assert_parity(P, oracle_mod, logs, specs, engine)
    assert int(rows[0]["clock"]) == 177 and int(rows[0]["decisions"]) == 161


# ------------------------------------------------------------------ random programs (edge-heavy)

@pytest.mark.parametrize("engine", [1, 2])
def test_random_programs(P, oracle_mod, engine):
    logs, specs = [], []
    for s in range(24 if engine == 1 else 6):
        w = models.random_program(60, seed=1000 + s, p_release=0.3, max_parents=4)
        logs.append(w)
        v = LogView(w)
        for fr in (0.3, 0.5, 0.8):
            for h in HS:
                specs.append(dict(log=len(logs) - 1, h=h, budget=max(3, int(v.peak_live * fr)), seed=s))
    assert_parity(P, oracle_mod, logs, specs, engine)


def test_random_programs_wide(P, oracle_mod):
    """High fan-in (many distinct adjacent components: exercises the dedup fallback)."""
    logs, specs = [], []
    for s in range(12):
        w = models.random_program(120, seed=2000 + s, p_release=0.2, max_parents=12, window=24)
        logs.append(w)
        v = LogView(w)
        for fr in (0.3, 0.6):
            for h in ("dtr", "dtr_eq", "msps", "dtr_full", "estar"):
                specs.append(dict(log=len(logs) - 1, h=h, budget=max(3, int(v.peak_live * fr))))
    assert_parity(P, oracle_mod, logs, specs, 1)


# ------------------------------------------------------------------ deallocation policies (reading C-22)

@pytest.mark.parametrize("engine", [1, 2])
def test_dealloc_policies_random(P, oracle_mod, engine):
    """V1 banishing / eager eviction / ignore on random programs, every heuristic."""
    logs, specs = [], []
    for s in range(10 if engine == 1 else 3):
        w = models.random_program(70, seed=3000 + s, p_release=0.35, max_parents=4)
        logs.append(w)
        v = LogView(w)
        for dealloc in ("v1", "eager", "ignore"):
            for fr in (0.4, 0.7):
                for h in HS:
                    specs.append(dict(log=len(logs) - 1, h=h, budget=max(3, int(v.peak_live * fr)), seed=s,
                                      dealloc=dealloc))
    rows = assert_parity(P, oracle_mod, logs, specs, engine)
    assert sum(int(r["decisions"]) for r in rows) > 0


@pytest.mark.parametrize("engine", [1, 2])
def test_dealloc_v1_linear_theorem1(P, oracle_mod, engine):
    """linear(N) under V1 (App. A's Theorem 1 setting): h_e* and the baselines."""
    logs, specs = [], []
    for N in (64, 200):
        logs.append(models.linear(N))
        B = 2 * math.ceil(math.sqrt(N))
        for h in HS:
            specs.append(dict(log=len(logs) - 1, h=h, budget=B, thrash_kill=0, dealloc="v1"))
    rows = assert_parity(P, oracle_mod, logs, specs, engine)
    # Theorem 1 for h_e*: total cost O(N) -- C/2N <= 2 (pinned on the oracle)
    for sp, r in zip(specs, rows):
        if sp["h"] == "estar":
            N = 64 if sp["log"] == 0 else 200
            assert int(r["status"]) == 0 and int(r["clock"]) <= 4 * N


def test_dealloc_models(P, oracle_mod):
    """V1 / eager / ignore on the resnet32 log at three budgets."""
    w = models.resnet32()
    v = LogView(w)
    specs = [dict(log=0, h=h, budget=v.budget(pm), dealloc=d)
             for d in ("v1", "eager", "ignore") for h in ("dtr", "dtr_eq", "lru", "estar") for pm in (300, 600, 900)]
    assert_parity(P, oracle_mod, [w], specs, 1)


def test_percall_dealloc_random(P, oracle_mod):
    """Per-call sessions under every policy: the linked child lists, the tensor
    under creation blocking V1, REMAT/ENSURE of banished tensors (PRECOND)."""
    rng = np.random.default_rng(17)
    for dealloc in ("v1", "eager", "ignore"):
        for h in HS:
            for trial in range(3):
                B = int(rng.integers(6, 14))
                g = P.Runtime(P.HEURISTICS[h], budget=B, seed=trial, cap_tensors=256, cap_edges=1024,
                              dealloc=P.DEALLOC[dealloc])
                o = oracle_mod.Runtime(oracle_mod.HEURISTICS[h], budget=B, seed=trial,
                                       dealloc=oracle_mod.DEALLOC[dealloc])
                live = []
                for step in range(80):
                    r = rng.random()
                    if r < 0.55 or not live:
                        k = int(rng.integers(0, min(3, len(live)) + 1))
                        ps = [int(x) for x in rng.choice(live, size=k, replace=False)] if k else []
                        m, c = int(rng.integers(1, 4)), int(rng.integers(1, 5))
                        a, b = g.compute(m, c, ps), o.compute(m, c, ps)
                        assert a == b, (dealloc, h, trial, step)
                        if a[0] == 0:
                            live.append(a[1])
                    elif r < 0.8:
                        t = int(rng.choice(live))
                        assert g.release(t) == o.release(t)
                        live.remove(t)
                    elif r < 0.9:
                        t = int(rng.integers(0, o.state()["n"] + 2))
                        assert g.rematerialize(t) == o.rematerialize(t)
                    else:
                        t = int(rng.integers(0, o.state()["n"] + 1))
                        assert g.ensure(t) == o.ensure(t)
                    gs, os_ = g.stats(), o.result()
                    for f in ("status", "clock", "decisions", "remats", "computations", "peak_M", "trace_hash"):
                        assert int(gs[f]) == int(os_[f]), (dealloc, h, trial, step, f)
                    if int(gs["status"]) != 0:
                        break
                assert g.trace().tobytes() == o.trace().tobytes()


# ------------------------------------------------------------------ D.1 ablation h'(s, m, c) (reading C-23)

ABL = [f"abl_{c}_{m}{s}" for c in ("estar", "eqclass", "local", "no") for m in "xm" for s in "xs"]


@pytest.mark.parametrize("engine", [1, 2])
def test_ablation_random(P, oracle_mod, engine):
    logs, specs = [], []
    for s in range(8 if engine == 1 else 2):
        w = models.random_program(70, seed=4000 + s, p_release=0.3, max_parents=4)
        logs.append(w)
        v = LogView(w)
        for fr in (0.35, 0.7):
            for h in ABL:
                specs.append(dict(log=len(logs) - 1, h=h, budget=max(3, int(v.peak_live * fr)),
                                  dealloc="v1" if s % 2 else "v2"))
    assert_parity(P, oracle_mod, logs, specs, engine)


def test_ablation_models(P, oracle_mod):
    """The 16 variants on resnet32 and unet (the paper's D.1 workloads are these logs)."""
    logs = [models.resnet32(), models.unet()]
    specs = []
    for li, w in enumerate(logs):
        v = LogView(w)
        specs += [dict(log=li, h=h, budget=v.budget(pm)) for h in ABL for pm in (300, 700)]
    assert_parity(P, oracle_mod, logs, specs, 1)


def test_ablation_grid_and_pool_argmin(P, oracle_mod):
    import torch
    w = models.transformer()
    v = LogView(w)
    specs = [dict(log=0, h=h, budget=v.budget(400), max_decisions=300) for h in ABL]
    assert_parity(P, oracle_mod, [w], specs, 2)
    w = models.random_dag(100000, seed=12)
    v = LogView(w)
    for h in ("abl_estar_ms", "abl_eqclass_ms", "abl_eqclass_mx", "abl_local_xs", "abl_no_xx"):
        D = 20
        B = v.peak_total * 97 // 100
        ref, tr = oracle_mod.replay(w, oracle_mod.HEURISTICS[h], B, max_decisions=D + 1, trace_cap=D + 1)
        b = P.DeviceBatch([w], [dict(log=0, budget=B, heuristic=P.HEURISTICS[h], max_decisions=D)],
                          engine=P.ENGINE_GRID)
        b.run()
        out = b.pool_argmin().cpu().numpy().astype(np.uint64)
        torch.cuda.synchronize()
        nxt = tr[D]
        assert (int(out[0]), int(out[1]), int(out[2])) == (int(nxt["num"]), int(nxt["den"]), int(nxt["id"])), h


def test_percall_ablation_fixture(P):
    """Hand scores of tests/golden/ablation_T_B_clock7.json through the per-call API."""
    import json, os
    from fractions import Fraction
    gd = os.path.join(os.path.dirname(__file__), "golden")
    g = json.load(open(os.path.join(gd, "hdtr_T_B_clock7.json")))
    a = json.load(open(os.path.join(gd, "ablation_T_B_clock7.json")))
    for name, exp in a["expect"].items():
        rt = percall_fixture(P, "abl_" + name, g["parents"], g["evict"])
        got = {k: Fraction(n, d) for k, (n, d) in rt.scores().items()}
        assert got == {int(k): Fraction(*v) for k, v in exp.items()}, name


# ------------------------------------------------------------------ config 2 / 3

def sweep_specs(v, hs, permilles, log=0, **kw):
    return [dict(log=log, h=h, budget=v.budget(pm), **kw) for h in hs for pm in permilles]


def test_resnet32_sweep(P, oracle_mod):
    w = models.resnet32()
    v = LogView(w)
    specs = sweep_specs(v, ["dtr", "dtr_eq", "lru", "size", "msps", "dtr_full", "estar"], models.sweep_permilles(30))
    assert_parity(P, oracle_mod, [w], specs, 1)


@pytest.mark.parametrize("model", ["densenet100", "unet"])
def test_config3_subset(P, oracle_mod, model):
    w = models.CONFIG_MODELS[model]()
    v = LogView(w)
    specs = sweep_specs(v, ["dtr", "dtr_eq", "lru", "size", "msps"], [100, 300, 500, 800, 1000])
    assert_parity(P, oracle_mod, [w], specs, 1)


@pytest.mark.parametrize("model", ["transformer", "lstm", "treelstm"])
def test_long_logs_decision_sample(P, oracle_mod, model):
    """Config 4/5 shapes at full size: the first K decisions (bounded sample the
    oracle finishes in seconds), CTA and grid engines."""
    w = models.CONFIG_MODELS[model]()
    v = LogView(w)
    specs = [dict(log=0, h=h, budget=v.budget(pm), max_decisions=300) for h in ("dtr", "dtr_eq", "lru", "msps")
             for pm in (200, 600)]
    assert_parity(P, oracle_mod, [w], specs, 1)
    assert_parity(P, oracle_mod, [w], specs[:4], 2)


def test_stress_pool_grid(P, oracle_mod):
    """Config 5s shape (random locality DAG) on the grid engine, first decisions."""
    w = models.random_dag(200000, seed=3)
    v = LogView(w)
    specs = [dict(log=0, h=h, budget=v.peak_total * 98 // 100, max_decisions=50) for h in ("dtr", "dtr_eq", "lru")]
    assert_parity(P, oracle_mod, [w], specs, 2)


# ------------------------------------------------------------------ edge cases

def test_edge_statuses(P, oracle_mod):
    from dtr_inputs import LogBuilder
    logs, specs = [], []
    w = models.linear(16)
    logs.append(w)
    specs += [dict(log=0, h="dtr", budget=2, thrash_kill=0),          # OOM
              dict(log=0, h="size", budget=4, thrash_kill=2),         # thrash kill
              dict(log=0, h="dtr", budget=4, max_decisions=5)]        # decision cap
    b = LogBuilder()                                                  # empty log
    logs.append(b.build())
    specs.append(dict(log=1, h="dtr", budget=10))
    b = LogBuilder()                                                  # single tensor, budget below its size
    b.make(5, 1, [])
    logs.append(b.build())
    specs.append(dict(log=2, h="dtr", budget=3))
    bad = models.linear(8).copy()                                     # malformed: RELEASE twice -> PRECOND
    v = LogView(bad)
    ops = v.ops.copy()
    rel = [i for i, x in enumerate(ops) if (int(x) >> 29) == 3]
    ops[rel[1]] = ops[rel[0]]
    bad[len(bad) - len(ops):] = ops
    logs.append(bad)
    specs.append(dict(log=3, h="dtr", budget=100))
    rows = assert_parity(P, oracle_mod, logs, specs, 1)
    assert [int(r["status"]) for r in rows] == [3, 4, 8, 0, 3, 2]


def test_host_e2e_entry(P, oracle_mod):
    w = models.resnet32()
    v = LogView(w)
    words, offs = P.pack_logs([w])
    specs = [dict(log=0, budget=v.budget(pm), heuristic=P.HEURISTICS[h]) for h in ("dtr", "lru") for pm in
             (200, 500, 900)]
    cells, _ = P.make_cells(offs, specs)
    rows, _ = P.replay_batch_host(words, cells)
    for i, s in enumerate(specs):
        r, _ = oracle_mod.replay(w, s["heuristic"], s["budget"])
        for f in ROW_FIELDS:
            assert int(rows[i][f]) == int(r[f])


def test_determinism(P):
    w = models.densenet100()
    v = LogView(w)
    specs = [dict(log=0, budget=v.budget(pm), heuristic=P.HEURISTICS[h]) for h in ("dtr", "dtr_eq") for pm in
             (200, 600)]
    words, offs = P.pack_logs([w])
    cells, _ = P.make_cells(offs, specs)
    a, _ = P.replay_batch_host(words, cells)
    b, _ = P.replay_batch_host(words, cells)
    a["wall_ns"] = 0      # device time of the run: the one field that may differ
    b["wall_ns"] = 0
    assert a.tobytes() == b.tobytes()


# ------------------------------------------------------------------ per-call API (fixtures)

def percall_fixture(P, h, parents, evict, mems=None):
    rt = P.Runtime(P.HEURISTICS[h])
    for i, ps in enumerate(parents):
        rc, t = rt.compute(mems[i] if mems else 1, 1, ps)
        assert rc == 0 and t == i
    for t in evict:
        assert rt.debug_evict(t) == 0
    return rt


def test_percall_hand_fixtures(P):
    import json, os
    from fractions import Fraction
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hdtr_T_B_clock7.json")))
    rt = percall_fixture(P, "dtr", g["parents"], g["evict"])
    sc = {str(k): Fraction(n, d) for k, (n, d) in rt.scores().items()}
    assert sc == {k: Fraction(*v) for k, v in g["expect_scores"].items()}
    assert rt.release(3) == 0
    assert rt.scores()[3][0] == 0
    s0 = g["staleness0"]
    rt = percall_fixture(P, "dtr", g["parents"], g["evict"])
    rt.set_budget(s0["budget"])
    rc, t = rt.compute(1, 1, s0["make_parents"])
    assert rc == 0
    tr = rt.trace()
    assert [[int(r["clock"]), int(r["id"])] for r in tr] == s0["expect_trace"]
    assert int(rt.stats()["clock"]) == s0["expect_clock"]
    # MSPS chain
    rt = P.Runtime(P.HEURISTICS["msps"])
    rt.compute(1, 2, [])
    rt.compute(1, 3, [0])
    rt.compute(4, 1, [1])
    rt.debug_evict(0)
    rt.debug_evict(1)
    assert Fraction(*rt.scores()[2]) == Fraction(6, 4)


def test_percall_estar_fixture(P):
    """Directed e* scores on fixture T_B through the per-call API (hand values, see
    tests/test_oracle_pins.py::test_dtr_full_and_estar_scores_hand)."""
    import json, os
    from fractions import Fraction
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hdtr_T_B_clock7.json")))
    rt = percall_fixture(P, "dtr_full", g["parents"], g["evict"])
    assert {k: Fraction(n, d) for k, (n, d) in rt.scores().items()} == {0: 1, 2: Fraction(2, 5), 3: Fraction(1, 3),
                                                                       4: Fraction(2, 3)}
    rt = percall_fixture(P, "estar", g["parents"], g["evict"])
    assert {k: Fraction(n, d) for k, (n, d) in rt.scores().items()} == {0: 4, 2: 2, 3: 1, 4: 2}


def test_percall_vs_oracle_random(P, oracle_mod):
    """Random per-call sessions incl. REMAT of evicted tensors and preconditions."""
    rng = np.random.default_rng(7)
    for h in HS:
        for trial in range(4):
            B = int(rng.integers(6, 14))
            g = P.Runtime(P.HEURISTICS[h], budget=B, seed=trial, cap_tensors=256, cap_edges=1024)
            o = oracle_mod.Runtime(oracle_mod.HEURISTICS[h], budget=B, seed=trial)
            live = []
            for step in range(80):
                r = rng.random()
                if r < 0.55 or not live:
                    k = int(rng.integers(0, min(3, len(live)) + 1))
                    ps = [int(x) for x in rng.choice(live, size=k, replace=False)] if k else []
                    m, c = int(rng.integers(1, 4)), int(rng.integers(1, 5))
                    a, b = g.compute(m, c, ps), o.compute(m, c, ps)
                    assert a == b, (h, trial, step)
                    if a[0] == 0:
                        live.append(a[1])
                elif r < 0.75:
                    t = int(rng.choice(live))
                    assert g.release(t) == o.release(t)
                    live.remove(t)
                elif r < 0.85:
                    t = int(rng.integers(0, o.state()["n"] + 2))
                    assert g.rematerialize(t) == o.rematerialize(t)
                elif r < 0.9:
                    t = int(rng.choice(live))
                    assert g.get(t) == o.get(t)
                    live.append(t)
                else:
                    t = int(rng.choice(live))
                    assert g.release(t) == o.release(t)      # may hit rho == 0 -> PRECOND on both
                    if t in live:
                        live.remove(t)
                gs, os_ = g.stats(), o.result()
                for f in ("status", "clock", "decisions", "remats", "computations", "peak_M", "trace_hash"):
                    assert int(gs[f]) == int(os_[f]), (h, trial, step, f)
                if int(gs["status"]) != 0:
                    break
            assert g.trace().tobytes() == o.trace().tobytes()


def test_pool_argmin_standalone(P, oracle_mod):
    """K3+K4 alone over a stopped grid-engine simulation = the oracle's next decision."""
    import torch
    w = models.random_dag(100000, seed=11)
    v = LogView(w)
    for h in ("dtr", "dtr_eq", "lru", "size", "msps", "local", "dtr_full", "estar"):
        D = 25
        B = v.peak_total * 97 // 100
        ref, tr = oracle_mod.replay(w, oracle_mod.HEURISTICS[h], B, max_decisions=D + 1, trace_cap=D + 1)
        b = P.DeviceBatch([w], [dict(log=0, budget=B, heuristic=P.HEURISTICS[h], max_decisions=D)],
                          engine=P.ENGINE_GRID)
        b.run()
        out = b.pool_argmin().cpu().numpy().astype(np.uint64)
        torch.cuda.synchronize()
        nxt = tr[D]
        assert (int(out[0]), int(out[1]), int(out[2])) == (int(nxt["num"]), int(nxt["den"]), int(nxt["id"])), h
        assert int(out[4]) > 0


@pytest.mark.parametrize("model", ["transformer", "lstm", "densenet100"])
def test_grid_engine_all_heuristics(P, oracle_mod, model):
    """The whole-GPU engine (bitmap pool, paired gathers) on mid-size logs, every heuristic."""
    w = models.CONFIG_MODELS[model]()
    v = LogView(w)
    specs = [dict(log=0, h=h, budget=v.budget(pm), max_decisions=400 if h in ("msps", "dtr_full", "estar") else 1500,
                  seed=3) for h in HS for pm in (250, 900)]
    assert_parity(P, oracle_mod, [w], specs, 2)


def test_config4_lstm_full_size_sample(P, oracle_mod):
    """Config 4 shape at full size (LSTM T=4096, 2 layers, ~3e5 tensors; budget
    sized for a ~1e5-tensor pool): the first 300 decisions, whole-GPU engine."""
    w = models.lstm(T=4096, layers=2)
    v = LogView(w)
    B = v.peak_total * 100000 // v.n
    specs = [dict(log=0, h=h, budget=B, max_decisions=300) for h in ("dtr", "dtr_eq", "lru", "size")]
    assert_parity(P, oracle_mod, [w], specs, 2)


def test_grid_engine_hub_degrees(P, oracle_mod):
    """Hub tensors of degree > 32 (hub_dag): the whole-GPU team's warp-cooperative
    neighbour walk (several 32-neighbour chunks, labels deduplicated across
    chunks) and the per-lane phased walk, on the grid engine and dtr_pool_argmin."""
    import torch
    w = models.hub_dag(20000, seed=5)
    v = LogView(w)
    # the fixture does reach the warp walk: at most decisions a hub of degree > 32 is
    # resident next to an evicted tensor (evicted set read off the oracle's trace)
    nb = [[] for _ in range(v.n)]
    for t in range(v.n):
        for p in v.parents(t):
            nb[p].append(t)
            nb[t].append(p)
    hubs = [x for x in range(v.n) if len(nb[x]) > 32]
    _, tr = oracle_mod.replay(w, oracle_mod.HEURISTICS["dtr"], v.peak_total * 930 // 1000, max_decisions=600,
                              trace_cap=600)
    ev, hits = set(), 0
    for rec in tr:
        hits += any(x not in ev and any(q in ev for q in nb[x]) for x in hubs)
        ev.add(int(rec["id"]))
    assert len(hubs) >= 8 and hits > 300, (len(hubs), hits)
    specs = [dict(log=0, h=h, budget=v.peak_total * pm // 1000, max_decisions=600)
             for h in ("dtr", "dtr_eq", "abl_eqclass_ms") for pm in (930, 970)]
    assert_parity(P, oracle_mod, [w], specs, 2)
    for h in ("dtr", "dtr_eq"):
        D = 300
        B = v.peak_total * 950 // 1000
        ref, tr = oracle_mod.replay(w, oracle_mod.HEURISTICS[h], B, max_decisions=D + 1, trace_cap=D + 1)
        b = P.DeviceBatch([w], [dict(log=0, budget=B, heuristic=P.HEURISTICS[h], max_decisions=D)],
                          engine=P.ENGINE_GRID)
        b.run()
        out = b.pool_argmin().cpu().numpy().astype(np.uint64)
        torch.cuda.synchronize()
        nxt = tr[D]
        assert (int(out[0]), int(out[1]), int(out[2])) == (int(nxt["num"]), int(nxt["den"]), int(nxt["id"])), h


@pytest.mark.parametrize("width", [20, 30, 60])
def test_percall_msps_wide_frontier(P, oracle_mod, width):
    """MSPS with a closure frontier wider than the per-lane heap (24 ids): a
    tensor y of `width` evicted parents (partly chained, so closures overlap) --
    the lane walk overflows and the warp BFS takes over (width 30, 60); width 20
    stays in the lane walk.  y is huge, so it is the first eviction and its exact
    closure sum is in the trace; every decision must match the oracle."""
    _msps_wide(P, oracle_mod, width)


def _msps_wide(P, O, width):
    B0 = 1 << 40
    g = P.Runtime(P.HEURISTICS["msps"], budget=B0, cap_tensors=256, cap_edges=1024)
    o = O.Runtime(O.HEURISTICS["msps"], budget=B0)
    xs = []
    for i in range(width):                          # x_i: cost 50, chained pairwise so closures overlap
        ps = [xs[-1]] if xs and i % 3 else []
        a, b = g.compute(1, 50, ps), o.compute(1, 50, ps)
        assert a == b
        xs.append(a[1])
    a, b = g.compute(1 << 20, 1, xs), o.compute(1 << 20, 1, xs)   # y = f(x_0 .. x_{w-1}), huge: evicted first
    assert a == b
    y = a[1]
    a, b = g.compute(1, 1, [y]), o.compute(1, 1, [y])  # z = f(y)
    assert a == b
    for x in xs:                                    # evict every x (pool members, outside free())
        assert g.debug_evict(x) == o.debug_evict(x)
    st = o.state()
    B = int(st["M"])                                # now at the budget: the next MAKE must evict
    g.set_budget(B)
    o.set_budget(B)
    for k in range(4):                              # nullary MAKEs: y stays an unlocked candidate
        a, b = g.compute(1, 1, []), o.compute(1, 1, [])
        assert a == b, k
    gs, os_ = g.stats(), o.result()
    for f in ("status", "clock", "decisions", "remats", "computations", "peak_M", "trace_hash"):
        assert int(gs[f]) == int(os_[f]), f
    tr = o.trace()
    assert int(tr[0]["id"]) == y and int(tr[0]["num"]) == 1 + 50 * width   # the exact closure sum decided it
    assert g.trace().tobytes() == tr.tobytes()


def test_percall_state_residency_vs_oracle(P, oracle_mod):
    """dtr_debug_state (the App. A residency trace) equals the oracle's
    per-tensor flags after every record: the linear net, N = 64, B = 2 sqrt(N),
    h_e* with V1 banishing (the Theorem 1 setting) and h_DTR with V2."""
    from dtr_inputs.logfmt import OP_GET, OP_MAKE, OP_RELEASE, OP_SHIFT
    O = oracle_mod
    N = 64
    v = LogView(models.linear(N))
    for h, dealloc in (("estar", "v1"), ("dtr", "v2")):
        rt = P.Runtime(P.HEURISTICS[h], budget=16, dealloc=P.DEALLOC[dealloc], cap_tensors=4 * N, cap_edges=8 * N)
        ref = O.Runtime(O.HEURISTICS[h], budget=16, dealloc=O.DEALLOC[dealloc])
        for k, w in enumerate(v.ops):
            op, t = int(w) >> OP_SHIFT, int(w) & ((1 << OP_SHIFT) - 1)
            if op == OP_MAKE:
                a, b = rt.compute(int(v.mem[t]), int(v.cost[t]), v.parents(t)), ref.compute(int(v.mem[t]), int(v.cost[t]), v.parents(t))
                assert a == b
            elif op == OP_GET:
                assert rt.get(t) == ref.get(t) == 0
            elif op == OP_RELEASE:
                assert rt.release(t) == ref.release(t) == 0
            fl = ref.tensors()[0]
            want = [3 if f & 8 else 1 if f & 1 else 2 if f & 2 else 0 for f in fl]
            assert rt.state().tolist() == want, (h, k)
        rt.close()


def test_pool_argmin_bench_1e6_vs_oracle(P, oracle_mod):
    """The bench's roofline_large_pool configuration itself (config-5s stress log, n = 1e6,
    B = 0.98 peak_total, 1000 grid-engine decisions, then dtr_pool_argmin over the ~980 k
    pool) equals the oracle's 1001st decision ("check the bench's 1e6
    dtr_pool_argmin answers against the oracle's next decision")."""
    import torch
    w = models.random_dag(1000000, seed=0, cost_max=200)
    v = LogView(w)
    B = v.peak_total * 98 // 100
    D = 1000
    ref, tr = oracle_mod.replay(w, oracle_mod.HEURISTICS["dtr"], B, max_decisions=D + 1, trace_cap=D + 1)
    b = P.DeviceBatch([w], [dict(log=0, budget=B, heuristic=0, max_decisions=D)], engine=P.ENGINE_GRID)
    b.run()
    out = b.pool_argmin().cpu().numpy().astype(np.uint64)
    torch.cuda.synchronize()
    row = b.result_rows()[0]
    assert int(row["decisions"]) == D
    nxt = tr[D]
    assert (int(out[0]), int(out[1]), int(out[2])) == (int(nxt["num"]), int(nxt["den"]), int(nxt["id"]))
