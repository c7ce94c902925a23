"""Pins for the sketchy-pivoting oracle: LUPP on the sketch,
OSID (Alg. 4 / Eq. 5.3) and the Gaussian embedding (reading R25).

Each check ties oracle/sketch.py to something other than itself: LAPACK getrf's pivot
sequence, permutation and diagonally dominant inputs, LU reconstruction, least-squares
W when the embedding is invertible, exact recovery at exact rank, the closed form of
Eq. 5.2 at l = k, and normal-sample statistics for the embedding."""
import numpy as np
import pytest
import scipy.linalg
import scipy.stats

from oracle import referee as R
from oracle import sketch as K


def _lapack_pivots(Y, k):
    """Original row ids of the first k pivots of LAPACK getrf (row swaps applied)."""
    _, ipiv = scipy.linalg.lu_factor(Y)
    perm = np.arange(Y.shape[0])
    for i, p in enumerate(ipiv):
        perm[i], perm[p] = perm[p], perm[i]
    return [int(v) for v in perm[:k]]


@pytest.mark.parametrize("shape,k", [((200, 30), 30), ((64, 64), 40), ((500, 24), 12)])
def test_lupp_matches_lapack_getrf(shape, k):
    Y = np.random.default_rng(shape[0]).standard_normal(shape)
    f = K.lupp(Y, k)
    assert f.piv == _lapack_pivots(Y, k)
    assert f.pcol == list(range(k)) and not f.short


def test_lupp_reconstruction():
    """Full LU (k = l): Y(piv,:) = L(piv,:) U with L unit lower triangular in pivot order,
    and every non-pivot row reproduced by its multipliers (Y = L U + 0 after l steps)."""
    rng = np.random.default_rng(3)
    Y = rng.standard_normal((80, 12))
    f = K.lupp(Y, 12)
    Lp = f.L[f.piv]
    Lp = Lp + np.eye(12)                                  # unit diagonal (pivot rows)
    assert np.allclose(np.triu(Lp, 1), 0)
    assert np.linalg.norm(Y[f.piv] - Lp @ f.U) <= 1e-13 * np.linalg.norm(Y)
    rest = np.setdiff1d(np.arange(80), f.piv)
    assert np.linalg.norm(Y[rest] - f.L[rest] @ f.U) <= 1e-13 * np.linalg.norm(Y)
    assert np.all(np.abs(f.L) <= 1.0)                     # partial pivoting: |l| <= 1


def test_lupp_permutation_and_dominant():
    P = np.eye(9)[[4, 0, 7, 2, 8, 1, 3, 6, 5]]            # row i of P = e_perm[i]
    f = K.lupp(P, 9)
    assert [int(np.argmax(P[p])) for p in f.piv] == list(range(9))
    D = np.diag(np.arange(20, 0, -1.0)) + 0.01 * np.random.default_rng(0).standard_normal((20, 20))
    assert K.lupp(D, 15).piv == list(range(15))


def test_lupp_zero_column_skip_ties_and_duplicates():
    rng = np.random.default_rng(5)
    Y = rng.standard_normal((30, 6))
    Y[:, 0] = 0.0                                          # exactly zero active column
    f = K.lupp(Y, 4)
    assert f.pcol == [1, 2, 3, 4]
    assert f.piv == K.lupp(Y[:, 1:], 4).piv
    T = np.array([[1.0, 2.0], [-1.0, 3.0], [1.0, 5.0], [0.5, 1.0]])
    assert K.lupp(T, 1).piv == [0]                         # |1| ties: lowest row
    Dup = np.vstack([rng.standard_normal((5, 8))] * 3)     # rows r, r+5, r+10 identical
    fd = K.lupp(Dup, 5)
    assert len({p % 5 for p in fd.piv}) == 5               # no duplicate of a pivot is chosen
    short = K.lupp(Dup, 8)                                 # rank 5 < 8: duplicates become
    assert short.short and len(short.piv) == 5             # exact zeros, columns run out


def test_osid_least_squares_when_embedding_orthogonal():
    """l = d with an orthogonal Omega: (X_S Omega)^+ = Omega^T X_S^+, so Eq. 5.3 gives
    W = X X_S^+, the least-squares interpolation."""
    rng = np.random.default_rng(7)
    X = rng.standard_normal((120, 30))
    Om = np.linalg.qr(rng.standard_normal((30, 30)))[0] * 0.7
    f, W, _ = K.sketchy_id(X, 10, Om)
    Wls = np.linalg.lstsq(X[f.piv].T, X.T, rcond=None)[0].T
    assert np.abs(W - Wls).max() <= 1e-10
    assert np.array_equal(W[f.piv], np.eye(10))


def test_osid_at_l_equal_k_is_eq_5_2():
    """Without oversampling, W = Y Y_S^{-1} (Eq. 5.2) for a square Y_S."""
    rng = np.random.default_rng(8)
    X = rng.standard_normal((90, 25))
    Om = rng.standard_normal((25, 8)) / np.sqrt(8)
    Y = K.sketch(X, Om)
    S = K.lupp(Y, 8).piv
    W = K.osid_w(Y, S)
    Wref = np.linalg.solve(Y[S].T, Y.T).T
    assert np.abs(W - Wref).max() <= 1e-10 * np.abs(Wref).max()


def test_sketchy_id_exact_rank_recovery():
    """X of rank r, k = r, l = 3k: Y_S spans the sketched row space, W X_S = X exactly
    (SPEC sketchy_select example 2; Prop. 5.3 with errskel = 0)."""
    rng = np.random.default_rng(9)
    X = rng.standard_normal((300, 12)) @ rng.standard_normal((12, 60))
    Om = rng.standard_normal((60, 36)) / 6.0
    f, W, _ = K.sketchy_id(X, 12, Om)
    assert R.errskel(X, f.piv) <= 1e-20 * (X * X).sum()
    assert R.errid(X, f.piv, W) <= 1e-18 * (X * X).sum()


def test_osid_gamma_revealing_statistics():
    """Prop. 5.3: with l = 3k, errid <= gamma errskel with gamma =
    (1 + O(sqrt(k/l)))^2 with constant probability; checked as median over seeds <= 2.5
    on a Gaussian-exp matrix (the oversampling the paper uses)."""
    rng = np.random.default_rng(11)
    n, d, k = 400, 80, 10
    X = rng.standard_normal((n, d)) * np.exp(-np.arange(d) / 8.0)
    ratios = []
    for s in range(9):
        Om = np.random.default_rng(100 + s).standard_normal((d, 3 * k)) / np.sqrt(3 * k)
        f, W, _ = K.sketchy_id(X, k, Om)
        ratios.append(R.errid(X, f.piv, W) / R.errskel(X, f.piv))
    assert min(ratios) >= 1.0 - 1e-12                     # errskel is the minimum (Eq. 1.2)
    assert np.median(ratios) <= 2.5


def test_gaussian_embedding_statistics_and_determinism():
    Om = K.gaussian_embedding(40, 30, seed=7)
    assert Om.shape == (40, 30)
    assert np.array_equal(Om, K.gaussian_embedding(40, 30, seed=7))
    assert not np.array_equal(Om, K.gaussian_embedding(40, 30, seed=8))
    z = Om.ravel() * np.sqrt(30)
    assert abs(z.mean()) <= 4 / np.sqrt(z.size)
    assert abs(z.var() - 1) <= 0.12
    assert scipy.stats.kstest(z, "norm").pvalue > 1e-3
    x = np.random.default_rng(0).standard_normal(40)       # isotropy: E||Omega^T x||^2 = ||x||^2
    vals = [np.sum((K.gaussian_embedding(40, 30, seed=s).T @ x) ** 2) for s in range(40)]
    assert abs(np.mean(vals) / (x @ x) - 1) <= 0.1
