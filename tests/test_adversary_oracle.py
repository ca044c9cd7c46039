"""Pins of the Theorem 2 adversary (App. B) on the CPU oracle.

* the construction's own cost sum, exactly: C = 1 + sum_j L_j (L_j + 1) / 2
  (P:2083-2088), because every reveal after the first B lands on an entirely
  evicted path of length L and costs L rematerializations plus one computation;
* Theorem 2's bound: C / N >= N / (4B) (SPEC S:465-473's factor-2 slack on
  C >= N^2 / (2B) from equal L_j);
* the static path-at-a-time baseline replays in exactly N computations
  (P:2093-2096), with no rematerialization;
* B = N - 1: one node per path, C = N;
* the revealed graph is well formed: B paths from t0, sum L_j = N - 1.
"""
import numpy as np
import pytest

from oracle import adversary as A

H_SET = ["estar", "lru", "local", "dtr", "dtr_eq", "size", "dtr_full", "msps"]


@pytest.mark.parametrize("h", H_SET)
def test_cost_sum_closed_form(oracle_mod, h):
    for N, B in ((64, 3), (97, 5), (200, 8)):
        r, parents, path_of, _ = A.run_adversary(N, B, oracle_mod.HEURISTICS[h])
        assert int(r["status"]) == 0
        L = A.path_lengths(path_of, B)
        assert L.sum() == N - 1 and (L > 0).all()
        assert int(r["computations"]) == A.dynamic_cost_closed_form(L), (h, N, B)
        assert int(r["clock"]) == int(r["computations"])          # unit costs
        assert int(r["remats"]) == int(r["computations"]) - N
        # well formed: t0 has B children; every other node has exactly one child except path ends
        kids = np.bincount(parents[parents != A.NONE].astype(np.int64), minlength=N)
        assert kids[0] == B and (kids[1:] <= 1).all()


@pytest.mark.parametrize("h", ["estar", "lru", "local"])
@pytest.mark.parametrize("B", [8, 16, 32])
def test_theorem2_ratio(oracle_mod, h, B):
    """SPEC's primary Theorem 2 check: N = 512, ratio = C / N >= N / (4B), static = N."""
    N = 512
    r, parents, path_of, _ = A.run_adversary(N, B, oracle_mod.HEURISTICS[h])
    assert int(r["status"]) == 0
    C = int(r["computations"])
    assert C / N >= N / (4 * B), (h, B, C)
    words = A.static_log(parents, path_of)
    s, _ = oracle_mod.replay(words, oracle_mod.HEURISTICS[h], B, thrash_kill=0)
    assert int(s["status"]) == 0 and int(s["computations"]) == N and int(s["remats"]) == 0


def test_one_node_per_path(oracle_mod):
    for N in (8, 33):
        r, parents, path_of, _ = A.run_adversary(N, N - 1, oracle_mod.H_LRU)
        assert int(r["computations"]) == N and int(r["remats"]) == 0
        assert (A.path_lengths(path_of, N - 1) == 1).all()


def test_adversary_picks_a_fully_evicted_path(oracle_mod):
    """Replaying the revealed graph in reveal order through the oracle reproduces
    the run (determinism), and at every reveal after the first B the chosen
    path had no resident node -- checked by re-running step by step."""
    N, B = 60, 4
    r, parents, path_of, tr = A.run_adversary(N, B, oracle_mod.H_ESTAR, trace_cap=1 << 16)
    rt = oracle_mod.Runtime(oracle_mod.H_ESTAR, budget=B, trace_cap=1 << 16)
    rt.compute(1, 1, [])
    rt.ensure(0)
    for t in range(1, N):
        if t > B:
            fl = rt.tensors()[0]
            j = path_of[t]
            assert not any(fl[x] & 1 for x in range(1, t) if path_of[x] == j)
            # ... and it is the lowest such path
            for k in range(j):
                assert any(fl[x] & 1 for x in range(1, t) if path_of[x] == k)
        rt.compute(1, 1, [int(parents[t])])
    assert rt.trace().tobytes() == tr.tobytes()
    assert int(rt.result()["trace_hash"]) == int(r["trace_hash"])
