"""Pins for h_random (h_rand(t) = X ~ U(0,1), "a random
baseline ... using no metadata whatsoever"; reading C-15 fixes the draw as
splitmix64(seed ^ decision << 32 ^ id) so both sides are reproducible).

What the paper fixes, and what a wrong draw would break:
  * the evicted tensor is a UNIFORM choice over the pool, independent of the
    tensor id (chi-square of the evicted member's id-rank within the pool, and
    of its creation-age rank, over 2*10^4 decisions);
  * draws are independent across decisions (chi-square of consecutive ranks);
  * the recorded score is the MINIMUM of the pool's U(0,1) draws: with k
    members its mean is 1/(k+1) and P(X <= x) = 1 - (1-x)^k (Kolmogorov-Smirnov);
  * the decision never depends on cost, size or staleness (metamorphic: a log
    with random costs/sizes of one unit scale gives the same ranks as unit ones).
A hash correlated with the id (e.g. x = id) fails the rank chi-square; one that
ignores the decision index fails the consecutive-rank test and the minimum law.
"""
import math

import numpy as np
import pytest

from dtr_inputs.logfmt import LogBuilder

K = 8            # pool size at every decision
D = 20000        # decisions


def _fixture(k=K, d=D, mems=None, costs=None):
    """k independent unit tensors fill the budget B = k; every later MAKE (no
    parents) must evict exactly one pool member (the new tensor is locked while
    it is computed), so every decision sees a pool of exactly k tensors."""
    b = LogBuilder()
    for i in range(k + d):
        b.make(1 if mems is None else int(mems[i]), 1 if costs is None else int(costs[i]), [])
    return b.build()


def _ranks(trace, k=K):
    resident = list(range(k))
    ranks, ages = [], []
    for j, rec in enumerate(trace):
        e = int(rec["id"])
        assert e in resident
        srt = sorted(resident)
        ranks.append(srt.index(e))
        ages.append(srt[::-1].index(e))   # 0 = newest
        resident.remove(e)
        resident.append(k + j)
    return np.array(ranks), np.array(ages)


def _chi2_p(counts):
    """Upper-tail p-value of Pearson's chi-square against uniform (Wilson-Hilferty)."""
    counts = np.asarray(counts, dtype=np.float64)
    exp = counts.sum() / len(counts)
    x2 = float(((counts - exp) ** 2 / exp).sum())
    df = len(counts) - 1
    z = ((x2 / df) ** (1 / 3) - (1 - 2 / (9 * df))) / math.sqrt(2 / (9 * df))
    return 0.5 * math.erfc(z / math.sqrt(2))


@pytest.fixture(scope="module")
def run(oracle_mod):
    O = oracle_mod
    w = _fixture()
    r, tr = O.replay(w, O.H_RANDOM, K, seed=12345, thrash_kill=0, trace_cap=D + 1)
    assert int(r["status"]) == 0 and int(r["decisions"]) == D
    return tr


def test_random_choice_is_uniform_over_the_pool(run):
    ranks, ages = _ranks(run)
    assert _chi2_p(np.bincount(ranks, minlength=K)) > 1e-4
    assert _chi2_p(np.bincount(ages, minlength=K)) > 1e-4
    # an id-correlated draw would pick the smallest id (rank 0) far more often
    assert abs(np.mean(ranks) - (K - 1) / 2) < 0.1


def test_random_draws_independent_across_decisions(run):
    ranks, _ = _ranks(run)
    pairs = ranks[:-1] * K + ranks[1:]
    assert _chi2_p(np.bincount(pairs, minlength=K * K)) > 1e-4


def test_random_score_is_min_of_uniform_draws(run):
    x = np.array([int(v) for v in run["num"]], dtype=np.float64) / 2.0 ** 64
    assert np.all(run["den"] == 1)
    assert abs(x.mean() - 1.0 / (K + 1)) < 0.004       # E[min of K U(0,1)] = 1/(K+1); sd/sqrt(D) ~ 7e-4
    xs = np.sort(x)
    cdf = 1.0 - (1.0 - xs) ** K
    emp = np.arange(1, len(xs) + 1) / len(xs)
    ks = float(np.max(np.abs(emp - cdf)))
    assert ks < 1.95 / math.sqrt(len(xs))               # KS at ~0.1 %


def test_random_ignores_cost_size_and_staleness(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(7)
    n = K + 2000
    a = _fixture(d=2000)
    b = _fixture(d=2000, mems=np.ones(n), costs=rng.integers(1, 1000, n))
    ra, ta = O.replay(a, O.H_RANDOM, K, seed=99, thrash_kill=0, trace_cap=2001)
    rb, tb = O.replay(b, O.H_RANDOM, K, seed=99, thrash_kill=0, trace_cap=2001)
    assert np.array_equal(ta["id"], tb["id"]) and np.array_equal(ta["num"], tb["num"])
    # a different seed gives a different (still valid) choice sequence
    rc, tc = O.replay(a, O.H_RANDOM, K, seed=100, thrash_kill=0, trace_cap=2001)
    assert not np.array_equal(ta["id"], tc["id"])
