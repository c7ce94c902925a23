"""Pins for the oracle's random-number protocol and sampler (Alg. 2 l.5,
P:403; Eq. 2.2; reading R6-R8)."""
import itertools

import numpy as np
import pytest
import scipy.stats

from oracle import philox
from oracle import rbrp as O
from oracle import referee as R


def test_philox_known_answers(golden):
    rows = golden("philox4x32_10_kat.txt")["_rows"]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        assert philox.philox4x32_10(v[0:4], v[4:6]) == tuple(v[6:10])


def test_u53_range_and_mapping():
    # all-zero words -> 0; all-one words -> 1 - 2^-53 (never 1)
    assert philox.u53((0, 0)) == 0.0
    assert philox.u53((0xFFFFFFFF, 0xFFFFFFFF)) == 1.0 - 2.0 ** -53
    # only the top 53 bits of (w1 << 32 | w0) matter
    assert philox.u53((0x7FF, 0)) == 0.0
    assert philox.u53((0x800, 0)) == 2.0 ** -53
    u = philox.uniforms(7, 3, 0, 2000)
    assert u.min() >= 0 and u.max() < 1
    assert abs(u.mean() - 0.5) < 0.03
    # counter layout (j, t, 0, 0), key = (seed_lo, seed_hi)
    w = philox.philox4x32_10((5, 3, 0, 0), (7, 0))
    assert philox.uniforms(7, 3, 5, 1)[0] == philox.u53(w)


def _successive_law(w, b):
    """Exact law of successive sampling without replacement (ordered tuples)."""
    W = sum(w)
    probs = {}
    for tup in itertools.permutations(range(len(w)), b):
        p, rem = 1.0, W
        for i in tup:
            if w[i] == 0:
                p = 0.0
                break
            p *= w[i] / rem
            rem -= w[i]
        if p > 0:
            probs[tup] = p
    return probs


@pytest.mark.parametrize("w,b", [([1.0, 2.0, 3.0, 4.0], 2), ([5.0, 0.0, 1.0, 2.0, 0.5], 3)])
def test_sampler_law_matches_enumeration(w, b):
    """Brute-force enumeration of the successive-sampling law vs the oracle
    sampler's empirical frequencies (chi-square)."""
    w = np.array(w)
    law = _successive_law(list(w), b)
    T = 12000
    counts = {k: 0 for k in law}
    for t in range(1, T + 1):
        S, f = O.sample_block(w, b, seed=11, t=t)
        assert f == 0 and len(S) == b and len(set(S)) == b
        assert all(w[i] > 0 for i in S)
        counts[tuple(S)] += 1
    keys = sorted(law)
    obs = np.array([counts[k] for k in keys], dtype=float)
    exp = np.array([law[k] for k in keys]) * T
    assert obs.sum() == T
    assert scipy.stats.chisquare(obs, exp).pvalue > 1e-4


def test_example_2_3_first_draw_marginals(golden):
    """Example 2.3: group probabilities alpha/((alpha+beta) r)
    and 1/((alpha+beta) r) under Eq. 2.2 (first draw of a block)."""
    g = golden("example_2_3.txt")
    alpha, beta, r, k = g["alpha"], g["beta"], int(g["r"]), int(g["k"])
    m = 5                                    # rows per group (n/k)
    d = np.array([alpha if grp < r else 1.0 for grp in range(k) for _ in range(m)])
    T = 20000
    cnt = np.zeros(k)
    for t in range(1, T + 1):
        S, _ = O.sample_block(d, 1, seed=3, t=t)
        cnt[S[0] // m] += 1
    p = np.array([g["p_heavy"]] * r + [g["p_light"]] * (k - r))
    assert abs(p.sum() - 1) < 1e-12
    assert scipy.stats.chisquare(cnt, p * T).pvalue > 1e-4
    # eta_r of the Example 2.3 matrix through the referee
    X = np.zeros((k * m, k))
    for grp in range(k):
        X[grp * m:(grp + 1) * m, grp] = np.sqrt(alpha) if grp < r else 1.0
    assert abs(R.eta(X, r) - g["eta_r"]) < 1e-14
    assert abs(g["eta_r"] - beta / (alpha + beta)) < 1e-15


def test_sampler_zero_weight_and_support():
    d = np.array([0.0, 3.0, 0.0, 1.0, 0.0])
    for t in range(1, 200):
        S, f = O.sample_block(d, 1, 5, t)
        assert S[0] in (1, 3)
    S, f = O.sample_block(d, 2, 5, 1)
    assert S == [1, 3] and f == O.F_SUPPORT_EXHAUSTED
    S, f = O.sample_block(d, 5, 5, 1)
    assert S == [1, 3] and f == O.F_SUPPORT_EXHAUSTED
    S, f = O.sample_block(np.zeros(4), 2, 5, 1)
    assert S == [] and f == O.F_SUPPORT_EXHAUSTED


def test_sampler_inverse_cdf_rule():
    """The row is the smallest i with C(i) > u C(n-1) (reading R8)."""
    d = np.array([1.0, 0.0, 2.0, 5.0, 0.5, 0.0, 1.5])
    C = np.cumsum(d)
    for t in range(1, 50):
        S, _ = O.sample_block(d, 3, 9, t)
        us = philox.uniforms(9, t, 0, 64)
        expect = []
        for u in us:
            i = next(i for i in range(len(d)) if C[i] > u * C[-1])
            if i not in expect:
                expect.append(i)
            if len(expect) == 3:
                break
        assert S == expect


def test_greedy_block_topb():
    d = np.array([1.0, 5.0, 5.0, 0.0, 2.0])
    assert O.top_block(d, 3) == [1, 2, 4]
    assert O.top_block(d, 5) == [1, 2, 4, 0]
