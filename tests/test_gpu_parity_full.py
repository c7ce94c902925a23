"""GPU parity on the paths the full-size configs take ("What's weak" 1).

* Same seed, c2 at BASELINE size (65536 x 1024, 16 sampling chunks): the multi-chunk
  sampler's block-1 candidates equal the oracle's, and the whole run (S, b', rho_t)
  agrees on >= 8 of 10 seeds (SURVEY §8(c) contract; Alg. 2 l.5).
* NEAR_TIE rule: replay of the oracle's candidate blocks WITHOUT forcing
  the pivots, except on blocks whose logged pivot gap is below delta = 1e-9 (fp64) --
  the GPU's own pivoted Cholesky must then choose the oracle's Householder pivots (Alg. 2
  l.7-8) at b = 40, 64, 96, 128.
* Element-wise: the final residual norms d (|d_gpu(i) - d_oracle(i)| <= 1e-10 d0(i),
  Alg. 2 l.16) and W (max-abs error <= max(1e-10, 10 kappa(L_1) u) max|W|).
* Alg. 3 on its own (rbrp_form_w) against oracle.form_W, including the Remark 5.2
  clipped-SVD fallback (reading R17) on an ill-conditioned L_1.
"""
import numpy as np
import pytest
import torch

from oracle import rbrp as O
from oracle import referee as R
from workloads import CONFIGS, make, small_config

pytestmark = pytest.mark.gpu

cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")

DELTA = {np.float64: 1e-9, np.float32: 1e-3}   # NEAR_TIE margin
TOL = {np.float64: 1e-10, np.float32: 1e-4}    # north_star: rho_t, W


def _rb():
    import paper_2309_16002_b200 as rb
    return rb


def _check_d(res, ores, Xnp, dtype):
    d0 = O.row_sq_norms(Xnp)
    dg = res.d.cpu().numpy()
    assert dg.shape == ores.d.shape
    assert np.all(np.abs(dg - ores.d) <= TOL[dtype] * d0 + 1e-300)
    assert np.all(dg[res.S.numpy()] == 0.0)


def _check_W_elementwise(res, ores, dtype):
    W = res.W.double().cpu().numpy()
    Wo, kappa, _ = O.form_W(ores.L, ores.S, method="trsm")
    u = 1.1e-16 if dtype == np.float64 else 6e-8
    tol = max(TOL[dtype], 10 * kappa * u)
    assert np.max(np.abs(W - Wo)) <= tol * max(1.0, np.max(np.abs(Wo)))
    assert np.array_equal(W[res.S.numpy()], np.eye(len(res.S)))


def replay_near_tie(Xnp, ores, dtype, b, **kw):
    """Replay the oracle's candidate blocks; force the pivots only where the oracle's
    pivot gap is below delta (NEAR_TIE); everything else is the GPU's own choice."""
    rb = _rb()
    blocks = [blk.S_t for blk in ores.blocks]
    piv = [blk.piv if blk.pivot_gap < DELTA[dtype] else [-1] * len(blk.S_t) for blk in ores.blocks]
    nforced = sum(1 for blk in ores.blocks if blk.pivot_gap < DELTA[dtype])
    X = torch.from_numpy(Xnp).cuda()
    res = rb.id(X, k=ores.k, b=b, replay_blocks=blocks, replay_pivots=piv, return_d=True, **kw)
    assert bool(res.flags & rb.rbrp.F_NEAR_TIE) == (nforced > 0)
    assert res.S.tolist() == ores.S
    assert res.b_prime == [blk.b_prime for blk in ores.blocks]
    assert [p[:bp] for p, bp in zip(res.pivots, res.b_prime)] == \
        [blk.piv[:blk.b_prime] for blk in ores.blocks]
    for a, blk in zip(res.rho, ores.blocks):
        assert abs(a - blk.rho) <= TOL[dtype]
    _check_d(res, ores, Xnp, dtype)
    _check_W_elementwise(res, ores, dtype)
    return res, nforced


@cuda
def test_c2_full_same_seed_multichunk_sampler():
    """c2 full size (16 chunks of 4096 rows): block-1 candidates equal the oracle's for
    every seed; the whole run agrees on >= 8/10 seeds (identical S and b', rho_t within
    1e-10, d element-wise); |S| = 128 on every seed (exact rank)."""
    cfg = CONFIGS["c2"]
    X = make(cfg)
    Xnp = X.numpy()
    Xd = X.cuda()
    rb = _rb()
    same = 0
    for seed in range(10):
        ores = O.rbrp(Xnp, tau=cfg.tau, b=cfg.b, seed=seed)
        res = rb.id(Xd, tol=cfg.tau, b=cfg.b, seed=seed, return_d=True)
        assert res.blocks[0] == ores.blocks[0].S_t, seed        # multi-chunk CDF search
        assert res.k == ores.k == 128
        assert abs(res.k - ores.k) <= cfg.b
        assert res.resid_rel <= cfg.tau and ores.rho <= cfg.tau
        if res.S.tolist() == ores.S:
            same += 1
            assert res.b_prime == [blk.b_prime for blk in ores.blocks]
            for a, blk in zip(res.rho, ores.blocks):
                assert abs(a - blk.rho) <= 1e-10
            _check_d(res, ores, Xnp, np.float64)
    assert same >= 8, same


@cuda
def test_c2_full_candidates_later_blocks():
    """Every block's candidates equal the oracle's on seed 0 (the later blocks draw from
    the updated multi-chunk CDF, Alg. 2 l.16 -> l.5)."""
    cfg = CONFIGS["c2"]
    X = make(cfg)
    ores = O.rbrp(X.numpy(), tau=cfg.tau, b=cfg.b, seed=0)
    res = _rb().id(X.cuda(), tol=cfg.tau, b=cfg.b, seed=0)
    assert res.blocks == [blk.S_t for blk in ores.blocks]


@cuda
def test_near_tie_t3_b40():
    """Table 3's GMM (Example 4.1) at full size, b = 40, k = 100: unforced pivots."""
    cfg = CONFIGS["t3"]
    Xnp = make(cfg).numpy()
    ores = O.rbrp(Xnp, k=100, b=cfg.b, seed=0)
    replay_near_tie(Xnp, ores, np.float64, cfg.b)


@cuda
def test_near_tie_c3_full_b64():
    """c3 at full size (131072 x 512, b = 64): the heavy rows all have norm 100, so block
    1's first pivot is a rounding-level tie (forced by the NEAR_TIE rule); the other
    blocks use the GPU's own pivots.  The filter's duplicate rejection is exact."""
    cfg = CONFIGS["c3"]
    Xnp = make(cfg).numpy()
    tau = (1 + cfg.eps) * R.eta(Xnp, cfg.r)
    ores = O.rbrp(Xnp, tau=tau, b=cfg.b, seed=0)
    res, nforced = replay_near_tie(Xnp, ores, np.float64, cfg.b)
    assert nforced < len(ores.blocks)


@cuda
@pytest.mark.parametrize("kw", [
    dict(n=12000, d=200, n_centres=150, b=96),      # register-resident filter, 3 parts
    dict(n=24000, d=320, n_centres=260, b=128),     # c5's block size
])
def test_near_tie_c5_like_large_blocks(kw):
    cfg = small_config("c5", **kw)
    Xnp = make(cfg).numpy()
    tau = (1 + cfg.eps) * R.eta(Xnp, min(cfg.r, Xnp.shape[1] // 2))
    ores = O.rbrp(Xnp, tau=tau, b=cfg.b, seed=0)
    replay_near_tie(Xnp, ores, np.float64, cfg.b)


@cuda
def test_near_tie_fp32_c4_like():
    cfg = small_config("c4", n=20000, d=192, b=64)
    Xnp = make(cfg).numpy()
    ores = O.rbrp(Xnp, tau=1e-3, b=64, seed=0)
    replay_near_tie(Xnp, ores, np.float32, 64)


# ---------------------------------------------------------------------------------
# Alg. 3 on its own, Remark 5.2 fallback
# ---------------------------------------------------------------------------------
def _form_w_case(k, n, sig, seed, triangular):
    rng = np.random.default_rng(seed)
    if triangular:
        L1 = np.eye(k) + np.tril(rng.standard_normal((k, k)), -1) * (0.3 / np.sqrt(k))
        for j, s in sig.items():
            L1[j, j] = s
    else:
        U = np.linalg.qr(rng.standard_normal((k, k)))[0]
        V = np.linalg.qr(rng.standard_normal((k, k)))[0]
        L1 = (U * sig) @ V.T
    L = rng.standard_normal((n, k))
    S = sorted(rng.choice(n, k, replace=False).tolist())
    rng.shuffle(S)
    L[S] = L1
    return L, S


@cuda
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_form_w_trsm_matches_oracle(dtype):
    L, S = _form_w_case(96, 5000, {}, 0, True)
    L = L.astype(dtype)
    W, flags, ncl = _rb().rbrp.form_w(torch.from_numpy(L).cuda(), S, method="auto")
    assert flags == 0 and ncl == 0
    Wo, kappa, _ = O.form_W(L, S, method="trsm")
    u = 1.1e-16 if dtype == np.float64 else 6e-8
    assert np.max(np.abs(W.double().cpu().numpy() - Wo)) <= max(TOL[dtype], 10 * kappa * u) * np.max(np.abs(Wo))
    assert np.array_equal(W.double().cpu().numpy()[S], np.eye(len(S)))


@cuda
@pytest.mark.parametrize("k", [37, 160, 300])
def test_form_w_clipped_svd_matches_oracle(k):
    """method "pinv" on a general L_1 whose smallest singular values lie below 1e-12
    sigma_max: the same number of them is discarded and W equals the oracle's clipped-SVD
    W (Remark 5.2) element-wise; the kept spectrum has kappa <= 1e6."""
    sig = np.logspace(0, -6, k)
    sig[-3:] = [3e-14, 1e-15, 0.0]
    L, S = _form_w_case(k, 4000, sig, 1, False)
    W, flags, ncl = _rb().rbrp.form_w(torch.from_numpy(L).cuda(), S, method="pinv")
    Wo, kappa, clipped = O.form_W(L, S, method="pinv")
    assert clipped and (flags & _rb().rbrp.F_W_CLIPPED) and ncl == 3
    Wg = W.cpu().numpy()
    assert np.max(np.abs(Wg - Wo)) <= 1e-8 * np.max(np.abs(Wo))
    assert np.array_equal(Wg[S], np.eye(k))


@cuda
def test_form_w_auto_triggers_on_tiny_diagonal():
    """method "auto": a lower-triangular L_1 with one diagonal entry 1e-14 x the others
    fires the Remark 5.2 trigger (reading R17) and W is the clipped-SVD W, not the
    unbounded triangular solve."""
    L, S = _form_w_case(64, 3000, {20: 1e-14}, 2, True)
    W, flags, ncl = _rb().rbrp.form_w(torch.from_numpy(L).cuda(), S, method="auto")
    Wo, kappa, clipped = O.form_W(L, S, method="pinv")
    assert clipped and kappa > 1e12
    assert (flags & _rb().rbrp.F_W_CLIPPED) and ncl >= 1
    Wg = W.cpu().numpy()
    assert np.max(np.abs(Wg - Wo)) <= 1e-8 * np.max(np.abs(Wo))
    Wt, _, _ = O.form_W(L, S, method="trsm")
    assert np.max(np.abs(Wt)) > 1e6 * np.max(np.abs(Wg))     # what the plain solve would give


@cuda
@pytest.mark.parametrize("name,kw,dtype", [
    ("c3", dict(n=5 * 4096 + 300, d=128, n_heavy_dirs=30, n_heavy_rows=9000, b=32), np.float64),
    ("c5", dict(n=6 * 4096 + 77, d=160, n_centres=64, b=64), np.float64),
    ("c4", dict(n=5 * 4096 + 11, d=192, b=32), np.float32),
])
def test_same_seed_end_to_end_multichunk(name, kw, dtype):
    """SURVEY T3 on the other constructions (several 4096-row chunks, the tcgen05 kernel
    for fp32): same seed -> the same skeletons on >= 8 of 10 seeds, |S| within b on all, both
    meet the stop rule (Alg. 2 l.3, l.5).  "The same" compares what is unique: per block, the
    SET of kept rows up to exact duplicates (each index mapped to the first row with the
    same bytes).  On c3 the heavy directions all have norm exactly 100 and every one has
    many bitwise-identical copies, so the pivot order inside a block and the copy that
    wins an exact tie are decided by rounding (the oracle's multithreaded BLAS does not
    update identical columns bit-identically); the kept row vectors, b' and rho_t are
    unique."""
    cfg = small_config(name, **kw)
    Xnp = make(cfg).numpy()
    if cfg.tau is not None:
        tau = cfg.tau
    else:
        tau = (1 + cfg.eps) * R.eta(np.asarray(Xnp, np.float64), min(cfg.r, Xnp.shape[1] // 4))
    Xd = torch.from_numpy(Xnp).cuda()
    rb = _rb()
    first = {}
    canon = [first.setdefault(Xnp[i].tobytes(), i) for i in range(Xnp.shape[0])]
    same = 0
    for seed in range(10):
        ores = O.rbrp(Xnp, tau=tau, b=cfg.b, seed=seed)
        res = rb.id(Xd, tol=tau, b=cfg.b, seed=seed)
        assert res.blocks[0] == ores.blocks[0].S_t, seed
        assert abs(res.k - ores.k) <= cfg.b
        assert res.resid_rel <= tau and ores.rho <= tau
        gs = [canon[i] for i in res.S.tolist()]
        os_ = [canon[i] for i in ores.S]
        if _block_sets(gs, res.b_prime) == _block_sets(os_, [blk.b_prime for blk in ores.blocks]):
            same += 1
            for a, blk in zip(res.rho, ores.blocks):
                assert abs(a - blk.rho) <= TOL[dtype]
    assert same >= 8, same


def _block_sets(S, bps):
    out, o = [], 0
    for bp in bps:
        out.append(sorted(S[o:o + bp]))
        o += bp
    return out
