"""Pins for the oracle's RBRP loop (Alg. 2), SRP (Alg. 1), W
(Alg. 3) and the referee (Eq. 1.2, 1.3)."""
import math

import numpy as np
import pytest
import scipy.linalg

from oracle import rbrp as O
from oracle import referee as R
from workloads import CONFIGS, make, small_config


def _lowrank(n, d, r, seed, noise=0.0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, r)) @ rng.standard_normal((r, d))
    return X + noise * rng.standard_normal((n, d))


def test_row_norms_examples():
    assert list(O.row_sq_norms(np.array([[1.0, 0.0], [0.0, 2.0]]))) == [1.0, 4.0]
    assert list(O.row_sq_norms(np.eye(2))) == [1.0, 1.0]


@pytest.mark.parametrize("form", ["residual", "paper"])
def test_trace_equals_errskel_every_block(form):
    """Prop. 5.1 proof: ||d^(t)||_1 = errskel(X; S) after every block,
    checked against the independent referee (pseudoinverse projection)."""
    X = make(CONFIGS["c1"]).numpy()
    tau = 1.1 * R.eta(X, 20)
    res = O.rbrp(X, tau=tau, b=16, seed=0, form=form)
    assert res.blocks and res.rho <= tau
    S = []
    for blk in res.blocks:
        S += [blk.S_t[p] for p in blk.piv[:blk.b_prime]]
        es = R.errskel(X, S)
        assert abs(blk.rho * res.D0 - es) <= 1e-10 * res.D0
    assert S == res.S
    # before the last block the tolerance was not yet met (l.3)
    if len(res.blocks) > 1:
        assert res.blocks[-2].rho > tau


def test_exact_rank_recovery():
    """Exactly rank-r X: |S| = r and relative errskel <= 1e-24 (fp64)."""
    X = _lowrank(1500, 120, 16, 0)
    res = O.rbrp(X, tau=1e-14, b=8, seed=2)
    assert res.k == 16
    assert R.errskel(X, res.S) / res.D0 <= 1e-24
    # c2-like: rank 24 + 1e-8 noise, tau = 1e-12 stops at |S| = rank exactly
    cfg = small_config("c2", n=6000, d=260, rank=24, b=8)
    Xc = make(cfg).numpy()
    res = O.rbrp(Xc, tau=1e-12, b=8, seed=0)
    assert res.k == 24 and res.rho <= 1e-12


def test_residual_rows_orthogonal_to_skeleton_span():
    """Residual X - L Q^T is orthogonal to span(X_S) (north_star invariant);
    and L Q^T = X X_S^+ X_S (Prop. 5.1 proof)."""
    X = make(CONFIGS["c1"]).numpy()
    res = O.rbrp(X, k=40, b=16, seed=1)
    E = X - res.L @ res.Q.T
    Xs = X[res.S]
    assert np.linalg.norm(E @ Xs.T) <= 1e-12 * np.linalg.norm(X) * np.linalg.norm(Xs)
    P = X @ np.linalg.pinv(Xs) @ Xs
    assert np.linalg.norm(res.L @ res.Q.T - P) <= 1e-11 * np.linalg.norm(X)
    assert np.allclose(res.Q.T @ res.Q, np.eye(res.k), atol=1e-12)


@pytest.mark.parametrize("method", ["pinv", "trsm"])
def test_W_is_optimal_interpolation(method):
    """Alg. 3 / Prop. 5.1: W = L L_1^{-1} = X X_S^+ (Eq. 5.1) vs lstsq;
    W(S,:) = I exactly; normal equations; errid = errskel."""
    X = make(CONFIGS["c1"]).numpy()
    tau = 1.1 * R.eta(X, 20)
    res = O.rbrp(X, tau=tau, b=16, seed=0)
    W, kappa, clipped = O.form_W(res.L, res.S, method=method)
    assert not clipped
    Xs = X[res.S]
    Wls = np.linalg.lstsq(Xs.T, X.T, rcond=None)[0].T
    assert np.linalg.norm(W - Wls) <= 1e-10 * np.linalg.norm(Wls)
    assert np.array_equal(W[res.S], np.eye(res.k))
    G = (X - W @ Xs) @ Xs.T
    assert np.linalg.norm(G) <= 1e-12 * np.linalg.norm(X) * np.linalg.norm(Xs)
    eid, esk = R.errid(X, res.S, W), R.errskel(X, res.S)
    assert abs(eid - esk) <= 1e-10 * res.D0
    # (r, eps)-ID bound, Eq. 1.1 with tau = (1+eps) eta_r
    assert eid <= 1.1 * R.tail(X, 20) * (1 + 1e-12)
    # L_1 = L(S,:) is exactly lower-triangular in selection order (reading R13)
    L1 = res.L[res.S]
    assert np.all(np.triu(L1, 1) == 0)


def test_b1_reduces_to_srp():
    """RBRP with b = 1 is SRP (Alg. 1) step for step (shared draws)."""
    X = make(small_config("c1", n=400, d=60)).numpy()
    for seed in range(3):
        res = O.rbrp(X, k=25, b=1, seed=seed)
        S, L, d = O.srp(X, k=25, seed=seed)
        assert res.S == S
        assert np.allclose(res.L, L, atol=1e-10 * np.abs(L).max())
        assert all(blk.b_prime == 1 for blk in res.blocks)


def test_greedy_b1_is_cpqr_on_Xt():
    """RBGP with b = 1 is greedy pivoting = CPQR on X^T (reading
    A18): the first k pivots equal LAPACK geqp3's."""
    rng = np.random.default_rng(7)
    X = rng.standard_normal((80, 30)) * np.linspace(3, 0.2, 80)[:, None]
    res = O.rbrp(X, k=20, b=1, greedy=True)
    _, _, P = scipy.linalg.qr(X.T, mode="economic", pivoting=True)
    assert res.S == list(P[:20])


def test_residual_form_equals_paper_form():
    """Right-looking residual form (P:523 footnote) = Alg. 2 literal form:
    same S and per-block rho within 1e-12 (Q_b orthogonal to earlier Q)."""
    X = make(CONFIGS["c1"]).numpy()
    a = O.rbrp(X, k=64, b=16, seed=4, form="residual")
    p = O.rbrp(X, k=64, b=16, seed=4, form="paper")
    assert a.S == p.S
    for x, y in zip(a.blocks, p.blocks):
        assert abs(x.rho - y.rho) <= 1e-12


def test_fixed_rank_block_shrinks():
    """l.4: b <- min(b, k - |S|); |S| = k exactly in fixed-rank mode."""
    X = make(CONFIGS["c1"]).numpy()
    res = O.rbrp(X, k=37, b=16, seed=0)
    assert res.k == 37
    assert all(blk.b_t <= 16 for blk in res.blocks)
    assert sum(blk.b_prime for blk in res.blocks) == 37


def test_brute_force_best_subset_and_bounds():
    """errskel pinned by brute force on tiny inputs: the best subset is no
    worse than RBRP's and obeys the k-DPP existence bound
    min_{|S|=k} errskel <= (k+1)/(k-r+1) ||X - [X]_r||^2."""
    rng = np.random.default_rng(8)
    for trial in range(3):
        X = rng.standard_normal((11, 7)) @ np.diag([3, 2, 1, 0.5, 0.2, 0.1, 0.05])
        for k in (2, 3, 4):
            best, arg = R.best_subset(X, k)
            res = O.rbrp(X, k=k, b=2, seed=trial)
            assert best <= R.errskel(X, res.S) * (1 + 1e-12)
            for r in range(1, k + 1):
                assert best <= (k + 1) / (k - r + 1) * R.tail(X, r) * (1 + 1e-12)
            # monotone under inclusion
            assert R.errskel(X, list(arg) + [int(j) for j in range(11) if j not in arg][:1]) <= best * (1 + 1e-12)
            # errskel = min_W ||X - W X_S||^2 (Eq. 1.2) via lstsq
            Xs = X[list(arg)]
            Wls = np.linalg.lstsq(Xs.T, X.T, rcond=None)[0].T
            assert abs(R.errid(X, arg, Wls) - best) <= 1e-12 * (X ** 2).sum()


def test_eta_gaussian_exp_closed_form(golden):
    """Gaussian-exp: eta_100 from the spectrum vs the referee's SVD."""
    g = golden("gaussian_exp_eta.txt")
    n = 1000
    rng = np.random.default_rng(0)
    U, _ = np.linalg.qr(rng.standard_normal((n, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    sig = np.array([1.0 if i <= 100 else max(0.8 ** (i - 100), 1e-5) for i in range(1, n + 1)])
    X = (U * sig) @ V.T
    closed = math.fsum(s * s for s in sig[100:]) / math.fsum(s * s for s in sig)
    assert abs(R.eta(X, 100) - closed) <= 1e-11
    assert abs(closed - g["eta_100"]) <= 5e-7
    assert abs((X ** 2).sum() - g["fro2"]) <= 1e-4


def test_eta_c4_spectrum_closed_form():
    """c4's sigma_i = i^-1.5 (BASELINE configs): eta_r = sum_{i>r} i^-3 / sum i^-3."""
    cfg = small_config("c4", n=8192, d=256)
    X = make(cfg).numpy().astype(np.float64)
    for r in (5, 20):
        closed = math.fsum(i ** -3.0 for i in range(r + 1, 257)) / math.fsum(i ** -3.0 for i in range(1, 257))
        assert abs(R.eta(X, r) - closed) <= 1e-5 * closed


def test_example_2_3_rbrp_vs_brp(golden):
    """Example 2.3 adversary: RBRP's filter rejects duplicate directions and
    recovers X exactly with |S| = k; plain BRP (tau_b = 0) keeps duplicates."""
    g = golden("example_2_3.txt")
    alpha, r, k = g["alpha"], int(g["r"]), int(g["k"])
    m = 30
    X = np.zeros((k * m, 16))
    for grp in range(k):
        X[grp * m:(grp + 1) * m, grp] = np.sqrt(alpha) if grp < r else 1.0
    res = O.rbrp(X, tau=1e-12, b=8, seed=0)
    assert res.k == k and res.rho <= 1e-12
    brp = O.rbrp(X, k=k, b=8, seed=0, tau_b=0.0)
    assert R.errskel(X, brp.S) > 0.5 * R.errskel(X, res.S) + 1e-6


def test_gmm_example_4_1_robustness():
    """Example 4.1 GMM, small: RBRP reaches a lower errskel than
    plain BRP at the same fixed rank, averaged over seeds (Fig. 1 trend)."""
    kc, m, dd = 40, 25, 64
    rng = np.random.default_rng(1)
    X = np.zeros((kc * m, dd))
    for j in range(kc):
        mu = np.zeros(dd)
        mu[j] = 10.0 * (j + 1)
        X[j * m:(j + 1) * m] = mu + rng.standard_normal((m, dd))
    e_rbrp = np.mean([R.errskel(X, O.rbrp(X, k=kc, b=20, seed=s).S) for s in range(4)])
    e_brp = np.mean([R.errskel(X, O.rbrp(X, k=kc, b=20, seed=s, tau_b=0.0).S) for s in range(4)])
    assert e_rbrp < e_brp


def test_c3_small_filter_rejects_duplicates():
    """c3 construction (duplicate heavy rows): no two skeletons share a
    heavy direction."""
    cfg = small_config("c3", n=12000, d=64, n_heavy_dirs=20, n_heavy_rows=6000, b=16)
    X = make(cfg).numpy()
    tau = 1.2 * R.eta(X, 40)
    res = O.rbrp(X, tau=tau, b=16, seed=0)
    heavy = [s % 20 for s in res.S if s < 6000]
    assert len(heavy) == len(set(heavy)) == 20
    assert res.rho <= tau


def test_fp32_config_runs_in_fp32():
    cfg = small_config("c4", n=4096, d=128, b=16)
    X = make(cfg).numpy()
    assert X.dtype == np.float32
    res = O.rbrp(X, tau=1e-3, b=16, seed=0)
    assert res.L.dtype == np.float32 and res.rho <= 1e-3
    assert abs(R.errskel(X, res.S) / res.D0 - res.rho) <= 1e-4
