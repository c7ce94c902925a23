"""Pins for the oracle's local CPQR (Alg. 2 l.7; Eq. 2.1)
and robust filter (l.8; Remark 4.1; toy cases P:529-533)."""
import numpy as np
import pytest
import scipy.linalg

from oracle import rbrp as O


def _check_factorization(V, qr):
    d, b = V.shape
    s = min(d, b)
    assert np.allclose(qr.Q.T @ qr.Q, np.eye(s), atol=1e-13)
    assert np.all(np.tril(qr.R, -1)[:, :s] == 0)
    dg = np.diagonal(qr.R)
    assert np.all(dg >= 0)
    assert np.all(np.diff(dg) <= 1e-12 * dg[0])            # non-increasing
    Vp = V[:, qr.piv]
    assert np.linalg.norm(Vp - qr.Q @ qr.R) <= 1e-12 * np.linalg.norm(V)
    assert sorted(qr.piv) == list(range(b))
    # trailing-mass identity (Remark 4.1): after j pivots the
    # truncation error equals ||R(j:, j:)||_F^2 = mass[j]
    for j in range(b):
        E = Vp - qr.Q[:, :j] @ qr.R[:j, :]
        assert abs((E * E).sum() - qr.mass[j]) <= 1e-10 * qr.mass[0]


@pytest.mark.parametrize("shape", [(200, 40), (37, 37), (20, 32), (512, 64)])
def test_cpqr_factorization_and_mass(shape):
    rng = np.random.default_rng(1)
    V = rng.standard_normal(shape) * np.logspace(0, -3, shape[1])
    qr = O.cpqr(V)
    _check_factorization(V, qr)


@pytest.mark.parametrize("seed", range(5))
def test_cpqr_pivots_match_lapack_geqp3(seed):
    """Greedy max-residual-norm pivoting = LAPACK geqp3 pivot order on
    inputs without near-ties (scipy.linalg.qr(pivoting=True) calls geqp3)."""
    rng = np.random.default_rng(seed)
    V = rng.standard_normal((150, 30)) @ np.diag(rng.uniform(0.1, 3, 30))
    qr = O.cpqr(V)
    _, R, P = scipy.linalg.qr(V, mode="economic", pivoting=True)
    assert list(P) == list(qr.piv)
    assert np.allclose(np.abs(np.diagonal(R)), np.diagonal(qr.R), rtol=1e-10)


def test_cpqr_orthogonal_columns_order():
    """Orthogonal columns with norms [3,1,2] -> pivot order (0,2,1)."""
    V = np.zeros((5, 3))
    V[0, 0], V[1, 1], V[2, 2] = 3.0, 1.0, 2.0
    assert list(O.cpqr(V).piv) == [0, 2, 1]


def test_cpqr_tie_break_draw_order():
    """Exactly equal residual norms -> lowest original position (R9)."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal(8)
    y = rng.standard_normal(8)
    y *= np.linalg.norm(x) / np.linalg.norm(y)
    V = np.stack([0.5 * y, x, x, 0.1 * x + 0.01 * y], axis=1)
    qr = O.cpqr(V)
    assert qr.piv[0] == 1          # columns 1 and 2 tie exactly; 1 first


def test_filter_orthogonal_equal_norm_keeps_all():
    """orthogonal, equal-norm V -> ||R(i:b,i:b)||^2 = (b-i+1)/b ||V||^2,
    so the last step sits exactly on the threshold (b' = b in exact
    arithmetic; rounding decides the tie, so b' in {b-1, b})."""
    for b in (1, 4, 16):
        Qm, _ = np.linalg.qr(np.random.default_rng(b).standard_normal((64, b)))
        qr = O.cpqr(2.5 * Qm)
        tot = 6.25 * b
        assert np.allclose(qr.mass, [(b - i) / b * tot for i in range(b)], rtol=1e-13)
        assert O.filter_rank(qr.mass, 1.0 / b) >= b - 1
        # strictly inside the threshold -> all kept
        assert O.filter_rank(qr.mass, 0.999 / b) == b


def test_filter_rank_deficient():
    """rank(V) = b'' < b -> b' <= b''."""
    rng = np.random.default_rng(4)
    for rank in (1, 3, 7):
        V = rng.standard_normal((50, rank)) @ rng.standard_normal((rank, 12))
        qr = O.cpqr(V)
        bp = O.filter_rank(qr.mass, 1.0 / 12)
        assert 1 <= bp <= rank
        # the l.8 rule re-checked directly from R: kept mass >= tau_b ||V||^2
        R = qr.R
        tail = lambda i: (R[i:, i:] ** 2).sum()
        assert tail(bp - 1) >= (1 / 12) * (V ** 2).sum() * (1 - 1e-12)
        if bp < 12:
            assert tail(bp) < (1 / 12) * (V ** 2).sum()


def test_filter_drops_duplicates():
    """Ex. 4.1 / Remark 4.1: duplicated candidates are never both kept."""
    rng = np.random.default_rng(5)
    base = rng.standard_normal((40, 6)) * 10
    V = np.concatenate([base, base[:, [0, 2, 2, 5]]], axis=1)
    qr = O.cpqr(V)
    bp = O.filter_rank(qr.mass, 1.0 / V.shape[1])
    kept = [int(p) for p in qr.piv[:bp]]
    groups = [p if p < 6 else [0, 2, 2, 5][p - 6] for p in kept]
    assert len(set(groups)) == len(groups)
    assert bp == 6


def test_filter_b1_and_zero():
    qr = O.cpqr(np.ones((4, 1)))
    assert O.filter_rank(qr.mass, 1.0) == 1
    assert O.filter_rank(np.zeros(3), 0.5) == 0
    assert O.filter_rank(np.array([4.0, 1.0, 0.5]), 0.25) == 2
    assert O.filter_rank(np.array([4.0, 1.0, 0.5]), 0.0) == 3     # BRP keeps all


def test_forced_pivots_replay():
    rng = np.random.default_rng(6)
    V = rng.standard_normal((30, 8))
    forced = [3, 1, 7, 0, 2, 6, 5, 4]
    qr = O.cpqr(V, forced=forced)
    assert list(qr.piv) == forced
    _check_factorization_no_order(V, qr)


def _check_factorization_no_order(V, qr):
    assert np.linalg.norm(V[:, qr.piv] - qr.Q @ qr.R) <= 1e-12 * np.linalg.norm(V)
