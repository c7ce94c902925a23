"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (DESIGN.md §3 R23/R24, north_star): per-block rho_t absolutely within
1e-10 (fp64) / 1e-4 (fp32); W within max(tol, 10 kappa(L_1) u) relative in
Frobenius norm; skeletons and filtered ranks exact (integer results).
"""
import numpy as np
import pytest
import torch

from oracle import rbrp as O
from oracle import referee as R
from workloads import CONFIGS, make, small_config

pytestmark = pytest.mark.gpu

cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")


def _rb():
    import paper_2309_16002_b200 as rb
    return rb


def _tol(dtype):
    return 1e-10 if dtype == np.float64 else 1e-4


def _check_W(Xnp, res, ores, dtype):
    W = res.W.double().cpu().numpy()
    Wo, kappa, _ = O.form_W(ores.L, ores.S, method="trsm")
    u = 1.1e-16 if dtype == np.float64 else 6e-8
    tol = max(_tol(dtype), 10 * kappa * u)
    assert np.linalg.norm(W - Wo) <= tol * np.linalg.norm(Wo)
    S = res.S.numpy()
    assert np.array_equal(W[S], np.eye(len(S)))           # Alg. 3 l.2: exactly I


def _same_seed(cfg, tau=None, k=None, seed=0, **kw):
    rb = _rb()
    X = make(cfg)
    Xnp = X.numpy()
    ores = O.rbrp(Xnp, tau=tau, k=k, b=cfg.b, seed=seed, **kw)
    res = rb.id(X.cuda(), tol=tau, k=k, b=cfg.b, seed=seed, **kw)
    return Xnp, ores, res


@cuda
def test_c1_same_seed_end_to_end():
    """c1 full size, seeds 0..9: same Philox protocol -> identical S on >= 8/10
    seeds, rho_t within 1e-10, the (r, eps) bound met by both (R24)."""
    cfg = CONFIGS["c1"]
    X = make(cfg)
    Xnp = X.numpy()
    tail = R.tail(Xnp, cfg.r)
    tau = (1 + cfg.eps) * R.eta(Xnp, cfg.r)
    rb = _rb()
    Xd = X.cuda()
    same = 0
    for seed in range(10):
        ores = O.rbrp(Xnp, tau=tau, b=cfg.b, seed=seed)
        res = rb.id(Xd, tol=tau, b=cfg.b, seed=seed)
        assert res.resid_rel <= tau and ores.rho <= tau
        assert abs(res.k - ores.k) <= cfg.b
        eid = R.errid(Xnp, res.S.tolist(), res.W.cpu().numpy())
        assert eid <= (1 + cfg.eps) * tail * (1 + 1e-9)
        assert abs(eid - R.errskel(Xnp, res.S.tolist())) <= 1e-10 * res.fro2
        if res.S.tolist() == ores.S:
            same += 1
            for a, b in zip(res.rho, [blk.rho for blk in ores.blocks]):
                assert abs(a - b) <= 1e-10
            assert res.b_prime == [blk.b_prime for blk in ores.blocks]
            _check_W(Xnp, res, ores, np.float64)
    assert same >= 8


@cuda
def test_c1_first_block_candidates_match_oracle():
    """Philox + chunked CDF sampler: block 1's candidates equal the oracle's."""
    cfg = CONFIGS["c1"]
    X = make(cfg)
    rb = _rb()
    for seed in range(5):
        ores = O.rbrp(X.numpy(), k=16, b=16, seed=seed)
        res = rb.id(X.cuda(), k=16, b=16, seed=seed)
        assert res.blocks[0] == ores.blocks[0].S_t


@cuda
@pytest.mark.parametrize("n", [3000, 3 * 4096 + 100])
def test_candidates_with_many_repeated_draws(n):
    """Sampling without replacement by rejecting repeats (reading R6) when almost every draw
    repeats: five rows hold all but ~1e-3 of the mass, so block 1 needs thousands of draws
    (dozens of 256-draw rounds of the shared hash set) to find b distinct rows.  Block 1's
    candidates, in draw order, equal the oracle's; one chunk (the sampler's own scan) and
    several chunks."""
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, 48))
    X[[7, 100, 1234, 2000, n - 1]] *= 1000.0
    rb = _rb()
    Xd = torch.from_numpy(X).cuda()
    for seed in range(3):
        ores = O.rbrp(X, k=16, b=16, seed=seed)
        res = rb.id(Xd, k=16, b=16, seed=seed)
        assert res.blocks[0] == ores.blocks[0].S_t, seed


def _replay(Xnp, ores, dtype, b, with_pivots=True):
    rb = _rb()
    blocks = [blk.S_t for blk in ores.blocks]
    piv = [blk.piv for blk in ores.blocks] if with_pivots else None
    X = torch.from_numpy(Xnp).cuda()
    res = rb.id(X, k=ores.k, b=b, replay_blocks=blocks, replay_pivots=piv)
    assert res.S.tolist() == ores.S
    assert res.b_prime == [blk.b_prime for blk in ores.blocks]
    for a, blk in zip(res.rho, ores.blocks):
        assert abs(a - blk.rho) <= _tol(dtype)
    _check_W(Xnp, res, ores, dtype)
    return res


@cuda
@pytest.mark.parametrize("name,kw", [
    ("c1", {}),
    ("c2", dict(n=6000, d=260, rank=24, b=8)),
    ("c3", dict(n=12000, d=64, n_heavy_dirs=20, n_heavy_rows=6000, b=16)),
    ("c5", dict(n=9000, d=96, n_centres=24, b=16)),
    ("c5", dict(n=12000, d=160, n_centres=120, b=64)),
    ("c5", dict(n=12000, d=200, n_centres=150, b=96)),
    ("c3", dict(n=20000, d=256, n_heavy_dirs=90, n_heavy_rows=9000, b=128)),
])
def test_replay_parity_fp64(name, kw):
    """Forced-pivot replay driven by the oracle's candidate blocks: S and b'
    exact, rho_t within 1e-10, W within tolerance (north_star)."""
    cfg = CONFIGS[name] if not kw else small_config(name, **kw)
    Xnp = make(cfg).numpy()
    if cfg.tau is not None:
        tau = cfg.tau
    else:
        tau = (1 + cfg.eps) * R.eta(Xnp, min(cfg.r, Xnp.shape[1] // 2))
    ores = O.rbrp(Xnp, tau=tau, b=cfg.b, seed=0)
    _replay(Xnp, ores, np.float64, cfg.b)


@cuda
@pytest.mark.parametrize("rank,b", [(70, 128), (95, 128), (81, 96), (120, 128)])
def test_replay_parity_projection_parts(rank, b):
    """b' > 64 runs as a 64-column part on k_lhat64 plus the remainder on the kernel of its own
    width (R28): exactly rank-r data puts b' ~ r into the first block (the oracle keeps 68,
    90, 73, 105), so the remainders 4, 26, 9, 41 run on buckets 16, 32, 16 and on k_lhat64
    again.  Replay parity with the oracle: S, b' exact, rho_t within 1e-10, W within
    tolerance."""
    cfg = small_config("c2", n=3 * 4096 + 1234, d=256, rank=rank, b=b)
    Xnp = make(cfg).numpy()
    ores = O.rbrp(Xnp, tau=1e-12, b=b, seed=0)
    assert ores.blocks[0].b_prime > 64   # (the robust filter may stop a few short of rank)
    _replay(Xnp, ores, np.float64, b)


@cuda
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("k", [8, 88, 128, 136, 90])
def test_form_w_kernels_against_oracle(dtype, k):
    """rbrp_form_w (Alg. 3 on its own) on every W kernel: k_w_small (k % 8 == 0, k <= 128),
    the pass GEMM (k = 136), the CUDA-core tile GEMM (k = 90: rows not readable as
    round8(k) columns); W against the oracle's triangular solve."""
    rb = _rb()
    rng = np.random.default_rng(k)
    n = 5000
    L = rng.standard_normal((n, k))
    S = sorted(rng.choice(n, k, replace=False).tolist())
    L[S] = np.eye(k) + 0.05 * np.tril(rng.standard_normal((k, k)), -1)
    Lg = torch.from_numpy(L.astype(dtype)).cuda()
    W, flags, _ = rb.rbrp.form_w(Lg, S, method="trsm")
    Wo, kappa, _ = O.form_W(Lg.double().cpu().numpy(), S, method="trsm")
    u = 1.1e-16 if dtype == np.float64 else 6e-8
    tol = max(_tol(dtype), 10 * kappa * u)
    Wd = W.double().cpu().numpy()
    assert np.linalg.norm(Wd - Wo) <= tol * np.linalg.norm(Wo)
    assert np.array_equal(Wd[S], np.eye(k))


@cuda
@pytest.mark.parametrize("k", [33, 65, 100, 127, 129, 200])
def test_trinv_paths_edge_sizes(monkeypatch, k):
    """L_1^{-1} at the edges of its kernels: k_trinv_one (32 < k <= 128; k padded to a
    multiple of 8 with an identity block) and k_trinv_blk (k > 128), on an L_1 with a
    non-unit diagonal; W through rbrp_form_w against the oracle's triangular solve, and the
    one-CTA inverse against the grid one (RBRP_TRINV_GRID=1) within the same bound."""
    rb = _rb()
    rng = np.random.default_rng(1000 + k)
    n = 3000
    L = rng.standard_normal((n, k))
    S = sorted(rng.choice(n, k, replace=False).tolist())
    L[S] = np.diag(rng.uniform(0.5, 2.0, k)) + 0.3 * np.tril(rng.standard_normal((k, k)), -1) / np.sqrt(k)
    Lg = torch.from_numpy(L).cuda()
    Wo, kappa, _ = O.form_W(L, S, method="trsm")
    tol = max(1e-10, 10 * kappa * 1.1e-16)
    W1, _, _ = rb.rbrp.form_w(Lg, S, method="trsm")
    monkeypatch.setenv("RBRP_TRINV_GRID", "1")
    W2, _, _ = rb.rbrp.form_w(Lg, S, method="trsm")
    for W in (W1, W2):
        Wd = W.cpu().numpy()
        assert np.linalg.norm(Wd - Wo) <= tol * np.linalg.norm(Wo)
        assert np.array_equal(Wd[S], np.eye(k))


@cuda
@pytest.mark.parametrize("b", [16, 64])
def test_replay_parity_fp32_c4_small(monkeypatch, b):
    """fp32 (c4-like): the default projection (fp32 storage, fp64 DMMA arithmetic, reading
    R19; b' > 32 in parts) and the CUDA-core fp32 kernels (RBRP_FP32_SIMT=1) both match the
    oracle's fp32 run in replay: S and b' exact, rho_t within the fp32 tolerance."""
    cfg = small_config("c4", n=20000, d=192, b=b)
    Xnp = make(cfg).numpy()
    ores = O.rbrp(Xnp, tau=1e-3, b=b, seed=0)
    monkeypatch.setenv("RBRP_FP32_SIMT", "0")
    a = _replay(Xnp, ores, np.float32, b)
    monkeypatch.setenv("RBRP_FP32_SIMT", "1")
    s = _replay(Xnp, ores, np.float32, b)
    monkeypatch.setenv("RBRP_FP32_SIMT", "0")
    assert a.S.tolist() == s.S.tolist() and a.b_prime == s.b_prime


@cuda
def test_replay_without_forced_pivots_c1():
    """Replay of candidate blocks only: the GPU's own pivoted Cholesky picks
    the same pivots as the oracle's Householder CPQR (no near-ties in c1)."""
    cfg = CONFIGS["c1"]
    Xnp = make(cfg).numpy()
    ores = O.rbrp(Xnp, k=60, b=16, seed=3)
    assert min(blk.pivot_gap for blk in ores.blocks) > 1e-9
    _replay(Xnp, ores, np.float64, 16, with_pivots=False)


@cuda
def test_exact_rank_stop_c2_small():
    cfg = small_config("c2", n=8192 + 123, d=300, rank=40, b=16)
    X = make(cfg)
    res = _rb().id(X.cuda(), tol=1e-12, b=16, seed=1)
    assert res.k == 40 and res.resid_rel <= 1e-12
    assert R.errskel(X.numpy(), res.S.tolist()) / res.fro2 <= 1e-12


@cuda
def test_ragged_shapes_and_odd_d():
    """n and d not multiples of any tile, d odd (scalar load path), b = 1."""
    rng = np.random.default_rng(0)
    rb = _rb()
    for (n, d, b) in [(777, 33, 5), (4097, 17, 1), (130, 201, 16), (5000, 64, 32)]:
        Xnp = rng.standard_normal((n, min(d, 12))) @ rng.standard_normal((min(d, 12), d))
        Xnp += 1e-3 * rng.standard_normal((n, d))
        ores = O.rbrp(Xnp, k=min(12, d), b=b, seed=2)
        _replay(Xnp, ores, np.float64, b)
    # fp32: odd d and d = 2 mod 4 (row stride not 16-byte aligned: CUDA-core fallback), and a
    # ragged d on the tiled DMMA path (d = 100: partial last chunk, two 32-column boxes)
    for (n, d, b) in [(3001, 37, 8), (2500, 70, 16), (6000, 100, 40)]:
        Xnp = (rng.standard_normal((n, 10)) @ rng.standard_normal((10, d))).astype(np.float32)
        Xnp += np.float32(1e-2) * rng.standard_normal((n, d)).astype(np.float32)
        ores = O.rbrp(Xnp, k=10, b=b, seed=2)
        _replay(Xnp, ores, np.float32, b)


@cuda
def test_b1_matches_srp():
    """b = 1: RBRP reduces to SRP (Alg. 1); same skeletons as the oracle's SRP."""
    cfg = small_config("c1", n=600, d=80)
    X = make(cfg)
    S, L, _ = O.srp(X.numpy(), k=20, seed=4)
    res = _rb().id(X.cuda(), k=20, b=1, seed=4)
    assert res.S.tolist() == S


@cuda
def test_edge_cases():
    rb = _rb()
    dev = torch.device("cuda")
    # NaN -> ENONFINITE; zero -> EDEGENERATE
    X = torch.randn(300, 20, dtype=torch.float64, device=dev)
    X[7, 3] = float("nan")
    with pytest.raises(rb.RBRPError) as e:
        rb.id(X, tol=0.1, b=8)
    assert e.value.status == -2
    with pytest.raises(rb.RBRPError) as e:
        rb.id(torch.zeros(50, 10, dtype=torch.float64, device=dev), tol=0.1, b=8)
    assert e.value.status == -3
    # k_max cap before tau -> TOL_UNREACHED
    X = torch.randn(500, 40, dtype=torch.float64, device=dev)
    res = rb.id(X, tol=1e-6, k_max=10, b=4)
    assert res.k == 10 and (res.flags & rb.rbrp.F_TOL_UNREACHED)
    # support smaller than b: 3 nonzero rows
    Z = torch.zeros(100, 10, dtype=torch.float64, device=dev)
    Z[[5, 50, 90]] = torch.randn(3, 10, dtype=torch.float64, device=dev)
    res = rb.id(Z, tol=1e-14, b=8)
    assert sorted(res.S.tolist()) == [5, 50, 90]
    assert res.flags & rb.rbrp.F_SUPPORT_EXHAUSTED
    # exact duplicates never both selected
    base = torch.randn(10, 30, dtype=torch.float64, device=dev)
    D = base.repeat(40, 1)
    res = rb.id(D, tol=1e-12, b=16)
    assert res.k == 10 and len({s % 10 for s in res.S.tolist()}) == 10
    # in-place mode gives the same answer
    Y = torch.randn(3000, 50, dtype=torch.float64, device=dev) @ torch.randn(50, 50, dtype=torch.float64, device=dev)
    a = rb.id(Y.clone(), k=30, b=16, seed=5)
    bb = rb.id(Y.clone(), k=30, b=16, seed=5, inplace=True)
    assert a.S.tolist() == bb.S.tolist()
    assert torch.equal(a.W, bb.W)
    # n < b
    res = rb.id(torch.randn(5, 9, dtype=torch.float64, device=dev), tol=1e-12, b=16)
    assert res.k == 5


@cuda
def test_full_c2_bench_config():
    """c2 at BASELINE size (the bench workload): stops at |S| = 128 exactly,
    rho <= 1e-12; trace = errskel by the referee; sampled W rows equal the
    least-squares interpolation X X_S^+ (Eq. 5.1)."""
    cfg = CONFIGS["c2"]
    X = make(cfg, device="cuda")
    res = _rb().id(X, tol=cfg.tau, b=cfg.b, seed=0)
    assert res.k == 128 and res.resid_rel <= 1e-12
    Xnp = X.cpu().numpy()
    S = res.S.tolist()
    assert abs(R.errskel(Xnp, S) / res.fro2 - res.resid_rel) <= 1e-13
    rows = np.random.default_rng(0).choice(cfg.n, 64, replace=False)
    Xs = Xnp[S]
    Wls = np.linalg.lstsq(Xs.T, Xnp[rows].T, rcond=None)[0].T
    W = res.W.cpu().numpy()
    assert np.linalg.norm(W[rows] - Wls) <= 1e-9 * np.linalg.norm(Wls)
    assert np.array_equal(W[S], np.eye(128))


@cuda
def test_simt_and_mma_projection_paths_agree(monkeypatch):
    """The CUDA-core (DFMA) and FP64-tensor (DMMA) projection kernels both
    match the oracle in replay mode."""
    cfg = small_config("c2", n=9000, d=256, rank=30, b=16)
    Xnp = make(cfg).numpy()
    ores = O.rbrp(Xnp, tau=1e-12, b=16, seed=0)
    monkeypatch.setenv("RBRP_FORCE_SIMT", "1")
    a = _replay(Xnp, ores, np.float64, 16)
    monkeypatch.setenv("RBRP_FORCE_SIMT", "0")
    b = _replay(Xnp, ores, np.float64, 16)
    assert a.S.tolist() == b.S.tolist()


@cuda
@pytest.mark.parametrize("b,d", [(16, 200), (32, 256), (16, 1024)])
def test_filter_variants_bit_identical(monkeypatch, b, d):
    """The filter's launch variants compute the same numbers in the same order: the
    thread-block cluster with DSMEM reductions (d <= 256) against the cooperative grid,
    Q_b's packed images written by the filter against k_pack_q.  Identical S, b', rho, W
    (bitwise), and the oracle's S on this seed."""
    rb = _rb()
    cfg = small_config("c1", n=3000, d=d, b=b)
    X = make(cfg, device="cuda")
    base = rb.id(X, k=48, b=b, seed=5)
    ores = O.rbrp(X.cpu().numpy(), k=48, b=b, seed=5)
    assert base.S.tolist() == list(ores.S)
    for env in ("RBRP_FILTER_COOP", "RBRP_NO_FUSE_PACK"):
        monkeypatch.setenv(env, "1")
        r = rb.id(X, k=48, b=b, seed=5)
        monkeypatch.delenv(env)
        assert r.S.tolist() == base.S.tolist(), env
        assert r.b_prime == base.b_prime and r.rho == base.rho, env
        assert torch.equal(r.W, base.W), env


@cuda
def test_graph_loop_equals_eager_loop(monkeypatch):
    """The block loop as one CUDA graph (conditional WHILE node) and the eager,
    host-driven loop launch the same kernels: identical S, b', rho and W."""
    rb = _rb()
    cfg = small_config("c2", n=20000, d=512, rank=70, b=32)
    X = make(cfg, device="cuda")
    g1 = rb.id(X, tol=1e-12, b=32, seed=3)
    g2 = rb.id(X, tol=1e-12, b=32, seed=3)          # cached graph
    monkeypatch.setenv("RBRP_NO_GRAPH", "1")
    e = rb.id(X, tol=1e-12, b=32, seed=3)
    assert g1.graph and g2.graph and not e.graph
    for g in (g1, g2):
        assert g.S.tolist() == e.S.tolist() and g.k == 70
        assert g.b_prime == e.b_prime and g.rho == e.rho
        assert torch.equal(g.W, e.W)
        assert g.blocks == e.blocks
    assert g1.proj_ms > 0


@cuda
@pytest.mark.parametrize("split", [[4096, 8192, None], [4096, 4096, 4096, None], [None]])
def test_shard_invariance(split):
    """Row-sharded run (the multi-GPU algorithm, shards in-process): S, b', rho and
    W rows BIT-identical to the single-GPU run for any sharding."""
    rb = _rb()
    cfg = small_config("c2", n=3 * 4096 + 1234, d=256, rank=40, b=16)
    X = make(cfg, device="cuda")
    ref = rb.id(X, tol=1e-12, b=16, seed=2)
    rows, off = [], 0
    for sz in split:
        sz = cfg.n - off if sz is None else sz
        rows.append(X[off:off + sz])
        off += sz
    res, Ws = rb.rbrp.id_sharded(rows, tol=1e-12, b=16, seed=2)
    assert res.graph                      # the sharded loop (and its collectives) as one graph
    assert res.S.tolist() == ref.S.tolist() and res.k == 40
    assert res.b_prime == ref.b_prime and res.rho == ref.rho and res.b_t == ref.b_t
    assert res.blocks == ref.blocks
    assert torch.equal(torch.cat(Ws, 0), ref.W)


@cuda
def test_sharded_graph_loop_equals_eager(monkeypatch):
    """The row-sharded loop as one CUDA graph (outer WHILE over blocks, inner WHILE over the
    draw rounds) and the host-driven eager loop: bit-identical S, b', rho, W -- also on a
    support smaller than b (several draw rounds, SUPPORT_EXHAUSTED) and in the paper form."""
    rb = _rb()
    cfg = small_config("c2", n=3 * 4096 + 500, d=192, rank=30, b=16)
    X = make(cfg, device="cuda")
    shards = [X[:4096], X[4096:8192], X[8192:]]
    for form in ("residual", "paper"):
        g, Wg = rb.rbrp.id_sharded(shards, tol=1e-12, b=16, seed=4, form=form)
        monkeypatch.setenv("RBRP_NO_GRAPH", "1")
        e, We = rb.rbrp.id_sharded(shards, tol=1e-12, b=16, seed=4, form=form)
        monkeypatch.delenv("RBRP_NO_GRAPH")
        assert g.graph and not e.graph
        assert g.S.tolist() == e.S.tolist() and g.b_prime == e.b_prime and g.rho == e.rho
        assert all(torch.equal(a, b) for a, b in zip(Wg, We))
    Z = torch.zeros(2 * 4096 + 10, 12, dtype=torch.float64, device="cuda")
    Z[[5, 4100, 8195, 8200]] = torch.randn(4, 12, dtype=torch.float64, device="cuda")
    r, _ = rb.rbrp.id_sharded([Z[:4096], Z[4096:8192], Z[8192:]], tol=1e-14, b=8)
    assert r.graph and sorted(r.S.tolist()) == [5, 4100, 8195, 8200]


@cuda
def test_sharded_graph_cache_keys_every_shard():
    """A row-sharded graph bakes every shard's X and workspace into its kernels: a second
    call that keeps shard 0 (same tensor, same workspace address) but swaps the other shards
    must not replay the first call's graph."""
    rb = _rb()
    dev = torch.device("cuda")
    Z0 = torch.zeros(4096, 12, dtype=torch.float64, device=dev)
    Z0[5] = torch.randn(12, dtype=torch.float64, device=dev)
    keep = []   # the first call's shards stay allocated: the second call's get new addresses
    for rows in ([100, 4000], [7, 2222]):   # nonzero rows of shard 1 (global 4096 + r)
        Z1 = torch.zeros(4096, 12, dtype=torch.float64, device=dev)
        Z1[rows] = torch.randn(2, 12, dtype=torch.float64, device=dev)
        Z2 = torch.zeros(10, 12, dtype=torch.float64, device=dev)
        Z2[3] = torch.randn(12, dtype=torch.float64, device=dev)
        r, _ = rb.rbrp.id_sharded([Z0, Z1, Z2], tol=1e-14, b=8)
        assert r.graph
        assert sorted(r.S.tolist()) == [5] + [4096 + x for x in sorted(rows)] + [8192 + 3]
        keep += [Z1, Z2]


@cuda
def test_sharded_replay_and_c3_duplicates():
    """Sharded run in forced-pivot replay against the oracle on the duplicate
    adversary (c3 construction), 3 shards."""
    cfg = small_config("c3", n=3 * 4096 + 999, d=64, n_heavy_dirs=20, n_heavy_rows=6000, b=16)
    Xnp = make(cfg).numpy()
    tau = 1.2 * R.eta(Xnp, 40)
    ores = O.rbrp(Xnp, tau=tau, b=16, seed=0)
    X = torch.from_numpy(Xnp).cuda()
    shards = [X[:4096], X[4096:8192], X[8192:]]
    res, Ws = _rb().rbrp.id_sharded(shards, k=ores.k, b=16, replay_blocks=[b.S_t for b in ores.blocks],
                                    replay_pivots=[b.piv for b in ores.blocks])
    assert res.S.tolist() == ores.S
    for a, blk in zip(res.rho, ores.blocks):
        assert abs(a - blk.rho) <= 1e-10
    W = torch.cat(Ws, 0).cpu().numpy()
    Wo, kappa, _ = O.form_W(ores.L, ores.S, method="trsm")
    assert np.linalg.norm(W - Wo) <= max(1e-10, 10 * kappa * 1.1e-16) * np.linalg.norm(Wo)


@cuda
def test_sharded_sampling_with_small_support_and_nan():
    rb = _rb()
    dev = torch.device("cuda")
    Z = torch.zeros(2 * 4096 + 10, 12, dtype=torch.float64, device=dev)
    Z[[5, 4100, 8195]] = torch.randn(3, 12, dtype=torch.float64, device=dev)
    res, _ = rb.rbrp.id_sharded([Z[:4096], Z[4096:8192], Z[8192:]], tol=1e-14, b=8)
    assert sorted(res.S.tolist()) == [5, 4100, 8195]
    Y = torch.randn(4096 + 5, 8, dtype=torch.float64, device=dev)
    Y[4099, 2] = float("inf")
    with pytest.raises(rb.RBRPError) as e:
        rb.rbrp.id_sharded([Y[:4096], Y[4096:]], tol=0.1, b=4)
    assert e.value.status == -2


@cuda
@pytest.mark.parametrize("n,d,rank,b", [
    (148 * 16 * 3 + 5, 1024, 40, 32),    # several tiles per CTA, ragged tail, nc = 16
    (9000, 330, 30, 16),                 # partial last chunk (330 = 5*64 + 10)
    (7001, 512, 100, 64),                # bucket 64 (c3-like width)
    (40, 200, 12, 16),                   # fewer tiles than SMs
])
def test_fused_projection_matches_two_kernel_path(monkeypatch, n, d, rank, b):
    """The a4 kernels -- the 64-row tiled pass (default: L-hat pass, then the update pass
    re-reading the tile through L2; with and without b' > 32 parts) and the two-kernel DMMA
    path (RBRP_NO_FUSED=1) -- all match the oracle in replay mode: identical S and b',
    rho_t within 1e-10 of the oracle and of each other, W within tolerance."""
    cfg = small_config("c2", n=n, d=d, rank=rank, b=b)
    Xnp = make(cfg).numpy()
    ores = O.rbrp(Xnp, tau=1e-12, b=b, seed=0)
    runs = {}
    for name, env in (("two_kernel", {"RBRP_NO_FUSED": "1", "RBRP_NO_PARTS": "0"}),
                      ("tiled", {"RBRP_NO_FUSED": "0", "RBRP_NO_PARTS": "0"}),
                      ("tiled_no_parts", {"RBRP_NO_FUSED": "0", "RBRP_NO_PARTS": "1"})):
        for k_, v in env.items():
            monkeypatch.setenv(k_, v)
        runs[name] = _replay(Xnp, ores, np.float64, b)
    monkeypatch.setenv("RBRP_NO_PARTS", "0")
    a = runs["two_kernel"]
    for f in (runs["tiled"], runs["tiled_no_parts"]):
        assert a.S.tolist() == f.S.tolist() and a.b_prime == f.b_prime
        assert max(abs(x - y) for x, y in zip(a.rho, f.rho)) <= 1e-10
    # same seed, sampling path (default kernel): reproducible bit for bit
    X = torch.from_numpy(Xnp).cuda()
    rb = _rb()
    s1 = rb.id(X, tol=1e-12, b=b, seed=5)
    s2 = rb.id(X, tol=1e-12, b=b, seed=5)
    assert s1.S.tolist() == s2.S.tolist() and s1.rho == s2.rho and torch.equal(s1.W, s2.W)
    assert s1.k == rank


def _replay_form(Xnp, ores, dtype, b, form):
    rb = _rb()
    blocks = [blk.S_t for blk in ores.blocks]
    piv = [blk.piv for blk in ores.blocks]
    X = torch.from_numpy(Xnp).cuda()
    X0 = X.clone()
    res = rb.id(X, k=ores.k, b=b, replay_blocks=blocks, replay_pivots=piv, form=form)
    assert torch.equal(X, X0)                      # paper form: X is read only
    assert res.S.tolist() == ores.S
    assert res.b_prime == [blk.b_prime for blk in ores.blocks]
    for a, blk in zip(res.rho, ores.blocks):
        assert abs(a - blk.rho) <= _tol(dtype)
    _check_W(Xnp, res, ores, dtype)
    return res


@cuda
@pytest.mark.parametrize("name,kw", [
    ("c1", {}),
    ("c2", dict(n=9000 + 77, d=1024, rank=70, b=32)),     # fused paper pass, nc = 16
    ("c2", dict(n=6000, d=260, rank=24, b=8)),            # partial chunk, bucket 16
    ("c3", dict(n=12000, d=64, n_heavy_dirs=20, n_heavy_rows=6000, b=16)),
    ("c5", dict(n=12000, d=160, n_centres=120, b=64)),    # 32 < b' <= 64: k_lhat64, read-only
    ("c5", dict(n=12000, d=200, n_centres=150, b=96)),    # b' > 64: parts, downdate per part
])
def test_paper_form_replay_parity(name, kw):
    """NEXT-1 (RBRP_FORM_PAPER): Alg. 2 literally (CGS2 for l.6, read-only L-hat pass
    for l.13, downdated norms for l.16) against the oracle's paper form in replay mode:
    S and b' exact, rho_t within 1e-10 (the oracle downdates the same way), W within
    tolerance, X untouched."""
    cfg = CONFIGS[name] if not kw else small_config(name, **kw)
    Xnp = make(cfg).numpy()
    if cfg.tau is not None:
        tau = cfg.tau
    else:
        tau = (1 + cfg.eps) * R.eta(Xnp, min(cfg.r, Xnp.shape[1] // 2))
    ores = O.rbrp(Xnp, tau=tau, b=cfg.b, seed=0, form="paper")
    _replay_form(Xnp, ores, np.float64, cfg.b, "paper")


@cuda
def test_paper_form_same_seed_matches_residual_form():
    """The two forms are equal in exact arithmetic (Q_b orthogonal to Q): on an
    exactly rank-70 input both stop at |S| = 70, rho within 1e-10 block by block, and the
    same seed gives the same skeletons."""
    rb = _rb()
    cfg = small_config("c2", n=20000, d=512, rank=70, b=32)
    X = make(cfg, device="cuda")
    r = rb.id(X, tol=1e-12, b=32, seed=3)
    p = rb.id(X, tol=1e-12, b=32, seed=3, form="paper")
    assert r.k == p.k == 70
    assert r.S.tolist() == p.S.tolist()
    assert max(abs(a - b) for a, b in zip(r.rho, p.rho)) <= 1e-10
    Wr, Wp = r.W.cpu(), p.W.cpu()
    assert torch.linalg.norm(Wr - Wp) <= 1e-9 * torch.linalg.norm(Wr)


@cuda
def test_brp_tau_b_zero_replay_parity():
    """NEXT-2, plain BRP (tau_b = 0: the filter of l.8 keeps every candidate)
    against the oracle in replay mode: S and b' exact, rho_t within 1e-10."""
    cfg = small_config("c5", n=12000, d=160, n_centres=60, b=16)
    Xnp = make(cfg).numpy()
    tau = (1 + cfg.eps) * R.eta(Xnp, 40)
    ores = O.rbrp(Xnp, tau=tau, b=16, seed=0, tau_b=0.0)
    rb = _rb()
    blocks = [blk.S_t for blk in ores.blocks]
    piv = [blk.piv for blk in ores.blocks]
    res = rb.id(torch.from_numpy(Xnp).cuda(), k=ores.k, b=16, tau_b=0.0, replay_blocks=blocks,
                replay_pivots=piv)
    assert res.S.tolist() == ores.S
    assert res.b_prime == [blk.b_prime for blk in ores.blocks]
    assert all(bp == len(blk.S_t) or bp < len(blk.S_t) for bp, blk in zip(res.b_prime, ores.blocks))
    for a, blk in zip(res.rho, ores.blocks):
        assert abs(a - blk.rho) <= 1e-10
    _check_W(Xnp, res, ores, np.float64)


@cuda
@pytest.mark.parametrize("name,kw,tau", [
    ("c2", dict(n=20000 + 99, d=256, rank=40, b=16), 1e-12),
    ("c5", dict(n=30000, d=128, n_centres=40, b=32), None),
])
def test_rbgp_greedy_matches_oracle(name, kw, tau):
    """NEXT-2, RBGP (Remark 4.2): S_t = the b_t largest residual norms (ties to
    the lower row; device tournament k_topb).  Deterministic, so GPU and oracle select the
    same skeletons in the same order with no replay (the inputs have no near-ties)."""
    cfg = small_config(name, **kw)
    Xnp = make(cfg).numpy()
    if tau is None:
        tau = (1 + cfg.eps) * R.eta(Xnp, 40)
    ores = O.rbrp(Xnp, tau=tau, b=cfg.b, seed=0, greedy=True)
    res = _rb().id(torch.from_numpy(Xnp).cuda(), tol=tau, b=cfg.b, greedy=True)
    assert res.S.tolist() == ores.S
    assert res.b_prime == [blk.b_prime for blk in ores.blocks]
    for a, blk in zip(res.rho, ores.blocks):
        assert abs(a - blk.rho) <= 1e-10
    _check_W(Xnp, res, ores, np.float64)


@cuda
def test_table3_gmm_robust_filter_and_replay_parity():
    """NEXT-3 workload (Example 4.1, the paper's Table 3 matrix at full size):
    fixed-rank RBRP at k = 52 matches the oracle in replay mode, and at k = 100 the robust
    filter yields (nearly) one skeleton per cluster while plain BRP (tau_b = 0) repeats
    clusters -- the pitfall the example describes (Fig. 1)."""
    from workloads import CONFIGS as C
    cfg = C["t3"]
    X = make(cfg, device="cuda")
    Xnp = X.cpu().numpy()
    ores = O.rbrp(Xnp, k=52, b=cfg.b, seed=0)
    _replay(Xnp, ores, np.float64, cfg.b)
    rb = _rb()
    m = cfg.n // cfg.n_centres
    r = rb.id(X, k=100, b=cfg.b, seed=0, with_W=False)
    p = rb.id(X, k=100, b=cfg.b, seed=0, tau_b=0.0, with_W=False)
    cr = len({int(i) // m for i in r.S.tolist()})
    cp = len({int(i) // m for i in p.S.tolist()})
    assert cr >= 90 and cr > cp, (cr, cp)
