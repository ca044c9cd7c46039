"""Parity of the on-device Theorem 2 adversary (K8, dtr_adversary_batch) with the
oracle-driven construction (oracle/adversary.py): identical revealed graphs,
result rows and eviction traces; Theorem 2's bound on the GPU runs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("status", "clock", "decisions", "remats", "computations", "peak_M", "trace_hash", "n_trace")


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_09616_b200 as P
    return P


def run_both(P, O, A, runs):
    ab = P.AdversaryBatch([dict(r, heuristic=P.HEURISTICS[r["h"]]) for r in runs])
    ab.run()
    import torch
    torch.cuda.synchronize()
    rows = ab.result_rows()
    allp = ab.parents.cpu().numpy().view(np.uint32)
    for i, r in enumerate(runs):
        ref, parents, path_of, tr = A.run_adversary(r["n"], r["budget"], O.HEURISTICS[r["h"]], seed=r.get("seed", 0),
                                                    trace_cap=r.get("trace_cap", 0))
        g = rows[i]
        assert int(g["status"]) == int(ref["status"]), (i, r)
        for f in FIELDS:
            if f == "n_trace":
                assert int(g[f]) == min(int(ref["decisions"]), r.get("trace_cap", 0)), (i, r)
            else:
                assert int(g[f]) == int(ref[f]), (i, r, f, int(g[f]), int(ref[f]))
        assert np.array_equal(ab.run_parents(i, allp), parents), (i, r)
        if r.get("trace_cap"):
            gt = ab.run_trace(i)[: int(g["n_trace"])]
            assert gt.tobytes() == tr.tobytes(), (i, r)
    return rows


def test_adversary_parity_small(P, oracle_mod):
    from oracle import adversary as A
    runs = []
    for h in ("estar", "lru", "local", "dtr", "dtr_eq", "size", "msps", "dtr_full", "random", "abl_eqclass_ms"):
        for N, B in ((40, 3), (97, 5), (160, 8)):
            runs.append(dict(n=N, budget=B, h=h, seed=5, trace_cap=1 << 14))
    run_both(P, oracle_mod, A, runs)


def test_adversary_theorem2_bound(P, oracle_mod):
    """SPEC's primary Theorem 2 setting on the device: N = 512, B in {8, 16, 32},
    h in {h_e*, LRU, h_DTR_local}; C / N >= N / (4B) and C = 1 + sum L_j (L_j + 1) / 2."""
    from oracle import adversary as A
    runs = [dict(n=512, budget=B, h=h) for h in ("estar", "lru", "local") for B in (8, 16, 32)]
    rows = run_both(P, oracle_mod, A, runs)
    for r, row in zip(runs, rows):
        C = int(row["computations"])
        assert C / 512 >= 512 / (4 * r["budget"])


def test_adversary_global_memory_path(P, oracle_mod):
    """Runs too large for shared memory use the workspace region (Sim<false>)."""
    from oracle import adversary as A
    runs = [dict(n=6000, budget=40, h="lru"), dict(n=5000, budget=16, h="dtr_eq")]
    run_both(P, oracle_mod, A, runs)


def test_adversary_edges(P, oracle_mod):
    from oracle import adversary as A
    run_both(P, oracle_mod, A, [dict(n=1, budget=3, h="lru"), dict(n=2, budget=3, h="lru"),
                                dict(n=9, budget=8, h="estar"), dict(n=9, budget=9, h="size")])
