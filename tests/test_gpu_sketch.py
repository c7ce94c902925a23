"""SkLUPP-OSID on the GPU against the oracle, through the C ABI
(include/rbrp_sketch.h).

  * embedding: rbrp_gaussian_embedding vs oracle.sketch.gaussian_embedding (reading R25;
    same Philox blocks, libm differences only: rtol 1e-13);
  * LUPP: bit-for-bit -- pivots, pivot columns and every multiplier equal the oracle's on
    the same Y (reading R26: updates a - l*u in pivot order, no FMA), over several panels,
    ragged row splits, fewer rows than SMs, a skipped zero column, duplicate rows and a
    short (rank-deficient) case;
  * sketch_id: S equal to the oracle's; W = Y Y_S^+ within 1e-9 relative (CholQR2 on the
    GPU vs Householder QR in the oracle); W(S,:) = I exactly; exact-rank recovery;
  * full size (c2, k = 128, l = 3k; Table 3's GMM at k = 472, l = 1416 > d): outputs
    computed row by row on the host (W rows from Y(i,:) Y_S^+), W(S,:) = I, the
    skeletonization error, and |L| <= 1 for the exported multipliers.
"""
import numpy as np
import pytest
import torch

from oracle import referee as R
from oracle import sketch as K
from workloads import CONFIGS, make

pytestmark = pytest.mark.gpu
cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")


def _sk():
    from paper_2309_16002_b200 import sketch as sk
    return sk


@cuda
def test_embedding_matches_oracle():
    for d, l, seed in [(24, 18, 5), (40, 7, 123456789)]:
        got = _sk().gaussian_embedding(d, l, seed).cpu().numpy()          # Omega^T (l x d)
        ref = K.gaussian_embedding(d, l, seed).T
        assert got.shape == ref.shape
        assert np.allclose(got, ref, rtol=1e-13, atol=1e-15)


def _lupp_case(Y, k):
    Yt = torch.as_tensor(Y, device="cuda")
    g = _sk().lupp(Yt, k, with_L=True)
    o = K.lupp(Y, k)
    assert g.piv == o.piv
    assert g.pcol == o.pcol
    assert np.array_equal(g.L.cpu().numpy(), o.L)        # every multiplier, bit for bit
    return g, o


@cuda
@pytest.mark.parametrize("n,l,k", [(3000, 96, 70), (777, 40, 40), (100, 50, 33), (60000, 48, 40),
                                   (148 * 3 + 5, 64, 64)])
def test_lupp_bitwise(n, l, k):
    rng = np.random.default_rng(n + l)
    Y = rng.standard_normal((n, l)) * np.exp(-np.arange(l) / 30.0)
    _lupp_case(Y, k)


@cuda
@pytest.mark.parametrize("pw", [16, 8])
def test_lupp_bitwise_narrow_panels(pw, monkeypatch):
    """the 16- and 8-column panel variants (chosen when the rows of a CTA and the U rows
    of k pivots do not fit 32 columns in shared memory), forced by the test knob"""
    monkeypatch.setenv("RBRP_LUPP_PW", str(pw))
    rng = np.random.default_rng(pw)
    Y = rng.standard_normal((3000, 96)) * np.exp(-np.arange(96) / 30.0)
    _lupp_case(Y, 70)


@cuda
def test_lupp_bitwise_large_k():
    """k = 300 pivots (about ten 32-column panels, 300 grid barriers)"""
    rng = np.random.default_rng(300)
    Y = rng.standard_normal((8000, 320)) * np.exp(-np.arange(320) / 100.0)
    _lupp_case(Y, 300)


@cuda
def test_lupp_zero_column_duplicates_and_short():
    rng = np.random.default_rng(4)
    Y = rng.standard_normal((900, 40))
    Y[:, 3] = 0.0
    Y[450:] = Y[:450]                                     # every row duplicated
    g, o = _lupp_case(Y, 39)
    assert 3 not in g.pcol
    base = rng.standard_normal((12, 30))
    D = np.vstack([base] * 40)                            # rank 12, 480 rows
    g, o = _lupp_case(D, 20)
    assert len(g.piv) == 12 and o.short


@cuda
@pytest.mark.parametrize("seeded", [False, True])
def test_sketch_id_matches_oracle(seeded):
    rng = np.random.default_rng(21)
    n, d, k = 4000, 128, 40
    l = 3 * k
    X = rng.standard_normal((n, d)) * np.exp(-np.arange(d) / 20.0)
    if seeded:
        Om = K.gaussian_embedding(d, l, seed=9)
        res = _sk().sketch_id(torch.as_tensor(X, device="cuda"), k, l, seed=9)
    else:
        Om = rng.standard_normal((d, l)) / np.sqrt(l)
        res = _sk().sketch_id(torch.as_tensor(X, device="cuda"), k, l,
                              omega_T=torch.as_tensor(Om.T.copy(), device="cuda"))
    f, W, _ = K.sketchy_id(X, k, Om)
    assert res.S.tolist() == f.piv
    Wg = res.W.cpu().numpy()
    assert np.array_equal(Wg[f.piv], np.eye(k))
    assert np.linalg.norm(Wg - W) <= 1e-9 * np.linalg.norm(W)
    e_g, e_o = R.errid(X, f.piv, Wg), R.errid(X, f.piv, W)
    assert abs(e_g - e_o) <= 1e-9 * e_o


@cuda
def test_sketch_id_large_k_blocked_cholesky():
    """k = 200 > 160: the OSID Cholesky factorizations take the blocked multi-CTA path;
    the sketch is wider than X (l > d)"""
    rng = np.random.default_rng(23)
    n, d, k = 6000, 512, 200              # l = 600 > d (as at Table 3 ranks k > d/3)
    l = 3 * k
    X = rng.standard_normal((n, d)) * np.exp(-np.arange(d) / 150.0)
    Om = rng.standard_normal((d, l)) / np.sqrt(l)
    res = _sk().sketch_id(torch.as_tensor(X, device="cuda"), k, l,
                          omega_T=torch.as_tensor(Om.T.copy(), device="cuda"))
    f, W, _ = K.sketchy_id(X, k, Om)
    assert res.S.tolist() == f.piv
    Wg = res.W.cpu().numpy()
    assert np.array_equal(Wg[f.piv], np.eye(k))
    assert np.linalg.norm(Wg - W) <= 1e-9 * np.linalg.norm(W)


@cuda
def test_sketch_id_exact_rank_and_ragged():
    rng = np.random.default_rng(22)
    n, d, r = 5001, 64, 24
    X = rng.standard_normal((n, r)) @ rng.standard_normal((r, d))
    res = _sk().sketch_id(torch.as_tensor(X, device="cuda"), r, 2 * r + 3, seed=1)
    S = res.S.tolist()
    assert len(set(S)) == r and res.k == r and res.flags == 0
    fro = (X * X).sum()
    assert R.errskel(X, S) <= 1e-20 * fro
    assert R.errid(X, S, res.W.cpu().numpy()) <= 1e-18 * fro


@cuda
def test_sketch_id_full_c2():
    """c2 at full size (65536 x 1024, exact rank 128 + 1e-8 noise), k = 128, l = 384:
    sampled W rows equal Y(i,:) Y_S^+ computed on the host from the same Omega, W(S,:) = I,
    and the skeleton captures the rank (errskel at the noise level)."""
    cfg = CONFIGS["c2"]
    X = make(cfg, device="cuda")
    k, l = 128, 384
    OmT = _sk().gaussian_embedding(cfg.d, l, seed=3)
    res = _sk().sketch_id(X, k, l, omega_T=OmT, profile=True)
    S = res.S.tolist()
    assert res.k == k and len(set(S)) == k
    Om = OmT.T.cpu().numpy()
    Xs = X[res.S.cuda()].cpu().numpy()
    Ys = Xs @ Om
    M = np.linalg.pinv(Ys)
    rows = np.random.default_rng(5).choice(cfg.n, 48, replace=False)
    Yr = X[torch.as_tensor(rows, device="cuda")].cpu().numpy() @ Om
    Wr = res.W[torch.as_tensor(rows, device="cuda")].cpu().numpy()
    ref = Yr @ M
    assert np.linalg.norm(Wr - ref) <= 1e-8 * np.linalg.norm(ref)
    assert np.array_equal(res.W[res.S.cuda()].cpu().numpy(), np.eye(k))
    # exact rank 128: the 128 skeleton rows span the row space up to the 1e-8 noise
    Xd = X.double()
    B = torch.linalg.qr(Xd[res.S.cuda()].T)[0]
    resid = float((Xd - (Xd @ B) @ B.T).pow(2).sum() / Xd.pow(2).sum())
    assert resid <= 1e-12
    assert set(res.ms_phase) == {"embedding", "sketch", "lupp", "osid"}


@cuda
def test_sketch_id_table3_full_rank_472():
    """Table 3's GMM (1e5 x 1e3, 100 clusters) at its largest rank k = 472, l = 3k = 1416 > d
    (the blocked Cholesky, 16-column LUPP panels and the l > d sketch at full size): W(S,:) =
    I, sampled rows of W equal Y(i,:) Y_S^+ from a host pseudo-inverse of the same sketch,
    and every LUPP multiplier has |l| <= 1 (partial pivoting)."""
    cfg = CONFIGS["t3"]
    X = make(cfg, device="cuda")
    k, l = 472, 1416
    OmT = _sk().gaussian_embedding(cfg.d, l, seed=7)
    res = _sk().sketch_id(X, k, l, omega_T=OmT)
    S = res.S.tolist()
    assert res.k == k and len(set(S)) == k
    Sd = res.S.cuda()
    assert torch.equal(res.W[Sd], torch.eye(k, dtype=torch.float64, device="cuda"))
    Om = OmT.T.cpu().numpy()
    Ys = X[Sd].cpu().numpy() @ Om
    M = np.linalg.pinv(Ys)
    rows = np.random.default_rng(8).choice(cfg.n, 32, replace=False)
    Yr = X[torch.as_tensor(rows, device="cuda")].cpu().numpy() @ Om
    ref = Yr @ M
    Wr = res.W[torch.as_tensor(rows, device="cuda")].cpu().numpy()
    assert np.linalg.norm(Wr - ref) <= 1e-7 * np.linalg.norm(ref)
    g = _sk().lupp(X @ OmT.T, k, with_L=True)    # a cuBLAS sketch: pivots may differ on ties
    assert len(g.piv) == k and float(g.L.abs().max()) <= 1.0
