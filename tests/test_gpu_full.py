"""BASELINE.json's configs c3, c4, c5 at FULL size through the C ABI.

The oracle cannot run these sizes end to end, so the checks are the ones the task allows
at any size:
  * outputs the oracle computes one by one: sampled rows of W against the least-squares
    interpolation X(i,:) X_S^+ (Eq. 5.1; numpy lstsq on the k x d system), and
    W(S,:) = I exactly (Alg. 3 l.2);
  * properties of the method: the stop rule rho <= tau (Alg. 2 l.3, Remark 1.1), the
    (r, eps) bound from the referee's errskel (Eq. 1.2) where the matrix fits the
    host, the robust filter's duplicate rejection on the adversary (Remark 4.1).
tau comes from the spectrum of the Gram matrix (harness arithmetic, Eq. 1.3), never from
the CUDA path.
"""
import numpy as np
import pytest
import torch

from oracle import referee as R
from workloads import CONFIGS, make

pytestmark = pytest.mark.gpu

cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")


def _rb():
    import paper_2309_16002_b200 as rb
    return rb


def _gram_tau(cfg, X, chunk=1 << 18):
    """tau = (1 + eps) eta_r from the eigenvalues of X^T X accumulated in fp64."""
    d = X.shape[1]
    G = torch.zeros((d, d), dtype=torch.float64, device=X.device)
    for a in range(0, X.shape[0], chunk):
        Xc = X[a:a + chunk].double()
        G += Xc.T @ Xc
    ev = torch.linalg.eigvalsh(G).flip(0).clamp_min(0)
    return float((1 + cfg.eps) * ev[cfg.r:].sum() / ev.sum())


def _check_W_rows(Wt, S, rows, xs_rows, XS, rtol):
    """W(i,:) = x_i X_S^+ for sampled rows i (least squares, Eq. 5.1); W(S,:) = I.
    Wt: the device W (only the sampled rows and the skeleton rows are copied back)."""
    Wls = np.linalg.lstsq(XS.T, xs_rows.T, rcond=None)[0].T
    Wr = Wt[torch.as_tensor(rows, device=Wt.device)].double().cpu().numpy()
    assert np.linalg.norm(Wr - Wls) <= rtol * np.linalg.norm(Wls)
    WS = Wt[torch.as_tensor(S, device=Wt.device)].double().cpu().numpy()
    assert np.array_equal(WS, np.eye(len(S)))


@cuda
def test_full_c3_adversarial_duplicates():
    """c3 (131072 x 512 fp64, 100 heavy directions each repeated 500x): the robust filter
    never keeps two copies of a heavy direction, every heavy direction is captured, and
    the (r, eps) = (200, 0.2) bound holds by the referee's errskel."""
    cfg = CONFIGS["c3"]
    X = make(cfg, device="cuda")
    Xnp = X.cpu().numpy()
    tau = (1 + cfg.eps) * R.eta(Xnp, cfg.r)
    res = _rb().id(X, tol=tau, b=cfg.b, seed=0)
    S = res.S.tolist()
    assert res.resid_rel <= tau
    e = R.errskel(Xnp, S) / res.fro2
    assert e <= tau and abs(e - res.resid_rel) <= 1e-10
    heavy = [s % cfg.n_heavy_dirs for s in S if s < cfg.n_heavy_rows]
    assert len(heavy) == len(set(heavy))                  # no duplicate kept (Remark 4.1)
    assert set(heavy) == set(range(cfg.n_heavy_dirs))     # each carries ~1% of ||X||^2 >> tau
    rows = np.random.default_rng(1).choice(cfg.n, 64, replace=False)
    _check_W_rows(res.W, S, rows, Xnp[rows], Xnp[S], 1e-8)


@cuda
def test_full_c4_fp32_rows_sharded_form():
    """c4 (1048576 x 2048 fp32, sigma_i = i^-1.5): tau = 1e-3 (reading R2) is met, the
    skeleton is of the size the spectrum allows, and sampled W rows match least squares
    to fp32 accuracy (reading R19: X, L, W fp32; norms and factorizations fp64)."""
    cfg = CONFIGS["c4"]
    X = make(cfg, device="cuda")
    res = _rb().id(X, tol=cfg.tau, b=cfg.b, seed=0)
    S = res.S.tolist()
    assert 20 <= res.k <= 256                             # optimal SVD rank is 20 at tau = 1e-3
    assert res.resid_rel <= cfg.tau
    # residual of the selection computed independently in fp64 (harness): ||X||^2 -
    # ||X B||^2 with B an orthonormal basis of the row space of X_S
    XS = X[S].double()
    B = torch.linalg.qr(XS.T)[0]
    tot = proj = 0.0
    for a in range(0, cfg.n, 1 << 17):
        Xc = X[a:a + (1 << 17)].double()
        tot += float((Xc * Xc).sum())
        P = Xc @ B
        proj += float((P * P).sum())
    assert abs((tot - proj) / tot - res.resid_rel) <= 1e-4   # R23 fp32 tolerance
    rows = np.random.default_rng(2).choice(cfg.n, 64, replace=False)
    rows_t = torch.as_tensor(rows, device=X.device)
    _check_W_rows(res.W, S, rows, X[rows_t].double().cpu().numpy(), XS.cpu().numpy(), 1e-4)


def _referee_fp64(X, S, W=None, chunk=1 << 18):
    """Independent referee in fp64 (harness arithmetic, torch on the device; never the
    CUDA path): errskel(X; S) = ||X||^2 - ||X B||^2 with B an orthonormal basis of the row
    space of X_S (Eq. 1.2), and, given W, errid = ||X - W X_S||_F^2 (Eq. 1.1)."""
    XS = X[torch.as_tensor(S, device=X.device)].double()
    B = torch.linalg.qr(XS.T)[0]
    tot = proj = eid = 0.0
    for a in range(0, X.shape[0], chunk):
        Xc = X[a:a + chunk].double()
        tot += float((Xc * Xc).sum())
        P = Xc @ B
        proj += float((P * P).sum())
        if W is not None:
            E = Xc - W[a:a + chunk].double() @ XS
            eid += float((E * E).sum())
    return tot, (tot - proj) / tot, (eid / tot if W is not None else None)


@cuda
def test_full_c5_gmm_referee():
    """c5 (4194304 x 1024 fp64 GMM, 34 GB; X, the residual, L and W all resident: about
    120 GB of the 180 GB HBM): the (r, eps) = (256, 0.1) bound is certified by an
    independent fp64 referee -- errskel from an orthonormal basis of X_S's row space
    (not the GPU's own resid_rel) and errid of the GPU's W (Eq. 1.1, reading R24) --
    and sampled W rows equal least squares (Eq. 5.1)."""
    cfg = CONFIGS["c5"]
    X = make(cfg, device="cuda")
    tau = _gram_tau(cfg, X)
    res = _rb().id(X, tol=tau, b=cfg.b, seed=0, k_max=768)
    S = res.S.tolist()
    assert cfg.r <= res.k <= 768
    tot, eskel, eid = _referee_fp64(X, S, res.W)
    assert abs(tot - res.fro2) <= 1e-10 * tot
    assert eskel <= tau                                    # (r, eps) met: errskel <= (1+eps) eta_r
    assert abs(eskel - res.resid_rel) <= 1e-10             # rho = errskel / ||X||^2
    assert eid <= tau * (1 + 1e-9) and abs(eid - eskel) <= 1e-10   # errid(W_gpu) = errskel
    rows = np.random.default_rng(3).choice(cfg.n, 32, replace=False)
    rows_t = torch.as_tensor(rows, device=X.device)
    _check_W_rows(res.W, S, rows, X[rows_t].cpu().numpy(), X[torch.as_tensor(S, device=X.device)].cpu().numpy(),
                  1e-7)
