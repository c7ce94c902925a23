"""Seeded input generators for BASELINE.json's five configs (c1..c5).

Every matrix is drawn in row panels of PANEL rows; panel p of component c
uses its own torch.Generator seeded from (seed, c, p).  Hence a row shard that
is a union of whole panels is generated bit-identically whatever the number
of ranks, and a scaled-down config keeps the structure of
the full one.  Global orthonormalisations (c1's U and V, c4's U and V) are
harness code: they use torch.linalg and are never timed.

The constructions follow BASELINE.json `configs` with the readings of SURVEY
§8(c) A22:
  c1  X = U diag(0.8^i) V^T + 1e-3 G  (Gaussian-exp-like decay)
  c2  X = A B + 1e-8 G, A n x 128, B 128 x d   (exactly rank-128 + noise)
  c3  rows i < 50000: 100 * h_(i mod 100), h_j unit-norm Gaussian directions;
      rows >= 50000: N(0,1) * 0.95^j over columns j  (duplicate adversary,
      Example 2.3 / 4.1 spirit)
  c4  X = U diag(i^-1.5) V^T rounded to fp32, U CholQR2-orthonormalised
      Gaussian, V Haar
  t3  Example 4.1's adversarial GMM (the paper's Table 3 workload, NEXT-3): row
      m (j-1) + i = 10 j e_j + xi_i, j = 1..100 clusters of m = 1000 rows, xi ~ N(0, I)
  c5  row i = mu_(c(i)) + 0.05 xi_i, 256 centres mu ~ N(0, I)  (GMM, Example
      4.1 spirit)
No item of any public dataset is reproduced: all inputs are synthetic.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import torch

PANEL = 4096


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    kind: str            # c1..c5 construction
    dtype: str           # "f64" | "f32"
    n: int
    d: int
    b: int
    tau: Optional[float] = None      # relative squared-Frobenius tolerance
    r: Optional[int] = None          # (r, eps) form: tau = (1+eps) * eta_r
    eps: Optional[float] = None
    rank: int = 128                  # c2 exact rank
    n_heavy_dirs: int = 100          # c3
    n_heavy_rows: int = 50000        # c3
    n_centres: int = 256             # c5
    seed: int = 0                    # generator seed
    rbrp_seed: int = 0               # sampler seed

    @property
    def torch_dtype(self):
        return torch.float64 if self.dtype == "f64" else torch.float32


CONFIGS = {
    "c1": Config("c1", "c1", "f64", 2000, 200, 16, r=20, eps=0.1),
    "c2": Config("c2", "c2", "f64", 65536, 1024, 32, tau=1e-12, rank=128),
    "c3": Config("c3", "c3", "f64", 131072, 512, 64, r=200, eps=0.2),
    "c4": Config("c4", "c4", "f32", 1048576, 2048, 64, tau=1e-3),
    "c5": Config("c5", "c5", "f64", 4194304, 1024, 128, r=256, eps=0.1),
    # the paper's own GPU workload (Table 3): the adversarial GMM
    # of Example 4.1, n = 10^5, d = 10^3, k = 100 clusters of m = 1000 rows,
    # row m(j-1)+i = 10 j e_j + xi_i, run in fixed-rank mode with b = 40
    "t3": Config("t3", "t3", "f64", 100000, 1000, 40, n_centres=100),
}

# Table 3 fixed ranks
T3_RANKS = (32, 52, 73, 100, 157, 220, 283, 346, 409, 472)


def small_config(name: str, **kw) -> Config:
    """A scaled-down version of config `name` (same construction)."""
    return dataclasses.replace(CONFIGS[name], name=name + "s", **kw)


def _gen(seed: int, comp: int, panel: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    # fixed integer mix of (seed, component, panel); no method arithmetic
    g.manual_seed((seed * 1000003 + comp * 7919 + panel * 104729 + 12345) % (2**63 - 1))
    return g


def _randn_rows(seed, comp, r0, r1, cols, device, dtype=torch.float64):
    """Rows [r0, r1) of an infinite N(0,1) matrix with `cols` columns, drawn
    panel by panel so any row range is reproducible."""
    out = torch.empty((r1 - r0, cols), dtype=dtype, device=device)
    p0, p1 = r0 // PANEL, (r1 - 1) // PANEL if r1 > r0 else r0 // PANEL - 1
    for p in range(p0, p1 + 1):
        g = _gen(seed, comp, p, device)
        blk = torch.randn((PANEL, cols), generator=g, dtype=dtype, device=device)
        a, bnd = max(r0, p * PANEL), min(r1, (p + 1) * PANEL)
        out[a - r0:bnd - r0] = blk[a - p * PANEL:bnd - p * PANEL]
    return out


def _haar(m, seed, comp, device):
    """Haar-distributed m x m orthogonal matrix: QR of a Gaussian with the
    sign of diag(R) folded into Q."""
    g = _gen(seed, comp, 0, device)
    G = torch.randn((m, m), generator=g, dtype=torch.float64, device=device)
    Q, R = torch.linalg.qr(G)
    s = torch.sign(torch.diagonal(R))
    s[s == 0] = 1
    return Q * s


def make(cfg: Config, device="cpu", row_offset: int = 0, n_local: Optional[int] = None) -> torch.Tensor:
    """Rows [row_offset, row_offset + n_local) of config `cfg`'s X, as a
    contiguous row-major tensor of cfg's dtype on `device`."""
    n, d = cfg.n, cfg.d
    if n_local is None:
        n_local = n - row_offset
    r0, r1 = row_offset, row_offset + n_local
    s = cfg.seed
    dt = cfg.torch_dtype
    if cfg.kind == "c1":
        # global QR of the whole n x min(n,d) Gaussian: only for small n
        m = min(n, d)
        G1 = _randn_rows(s, 1, 0, n, m, device)
        U, _ = torch.linalg.qr(G1)
        V = _haar(d, s, 2, device)[:, :m]
        sig = 0.8 ** torch.arange(m, dtype=torch.float64, device=device)
        X = (U * sig) @ V.T + 1e-3 * _randn_rows(s, 3, 0, n, d, device)
        return X[r0:r1].to(dt).contiguous()
    if cfg.kind == "c2":
        k = cfg.rank
        A = _randn_rows(s, 1, r0, r1, k, device)
        B = _randn_rows(s, 2, 0, k, d, device)
        X = A @ B + 1e-8 * _randn_rows(s, 3, r0, r1, d, device)
        return X.to(dt).contiguous()
    if cfg.kind == "c3":
        nh, nrow = cfg.n_heavy_dirs, min(cfg.n_heavy_rows, n)
        H = _randn_rows(s, 1, 0, nh, d, device)
        H = 100.0 * H / torch.linalg.norm(H, dim=1, keepdim=True)
        X = torch.empty((r1 - r0, d), dtype=torch.float64, device=device)
        idx = torch.arange(r0, r1, device=device)
        heavy = idx < nrow
        if heavy.any():
            X[heavy] = H[idx[heavy] % nh]
        light = ~heavy
        if light.any():
            l0 = int(idx[light][0])
            scale = 0.95 ** torch.arange(d, dtype=torch.float64, device=device)
            X[light] = _randn_rows(s, 2, l0, r1, d, device) * scale
        return X.to(dt).contiguous()
    if cfg.kind == "c4":
        return _make_c4(cfg, device, r0, r1)
    if cfg.kind == "t3":
        # Example 4.1: clusters are contiguous row ranges of m = n / k rows
        m = n // cfg.n_centres
        j = torch.arange(r0, r1, device=device) // m                     # 0-based cluster
        X = _randn_rows(s, 1, r0, r1, d, device)
        X[torch.arange(r1 - r0, device=device), j] += 10.0 * (j + 1).to(torch.float64)
        return X.to(dt).contiguous()
    if cfg.kind == "c5":
        C = _randn_rows(s, 1, 0, cfg.n_centres, d, device)
        # label c(i): uniform over centres, drawn per panel
        lab = torch.empty(r1 - r0, dtype=torch.long, device=device)
        for p in range(r0 // PANEL, (r1 - 1) // PANEL + 1):
            g = _gen(s, 2, p, device)
            lp = torch.randint(0, cfg.n_centres, (PANEL,), generator=g, device=device)
            a, bnd = max(r0, p * PANEL), min(r1, (p + 1) * PANEL)
            lab[a - r0:bnd - r0] = lp[a - p * PANEL:bnd - p * PANEL]
        X = C[lab] + 0.05 * _randn_rows(s, 3, r0, r1, d, device)
        return X.to(dt).contiguous()
    raise ValueError(cfg.kind)


def _make_c4(cfg, device, r0, r1):
    """c4: U diag(sigma) V^T with U = CholQR2 of an n x m Gaussian (panel
    generated, three passes so U is never materialised in full)."""
    n, d, s = cfg.n, cfg.d, cfg.seed
    m = min(n, d)
    sig = torch.arange(1, m + 1, dtype=torch.float64, device=device) ** -1.5
    V = _haar(d, s, 2, device)[:, :m]
    chunk = 16 * PANEL

    def panels():
        for a in range(0, n, chunk):
            yield a, min(n, a + chunk)

    G = torch.zeros((m, m), dtype=torch.float64, device=device)
    for a, bnd in panels():
        P = _randn_rows(s, 1, a, bnd, m, device)
        G += P.T @ P
    R1 = torch.linalg.cholesky(G, upper=True)
    G2 = torch.zeros_like(G)
    for a, bnd in panels():
        P = torch.linalg.solve_triangular(R1, _randn_rows(s, 1, a, bnd, m, device), upper=True, left=False)
        G2 += P.T @ P
    R2 = torch.linalg.cholesky(G2, upper=True)
    R = R2 @ R1
    T = torch.linalg.solve_triangular(R, torch.eye(m, dtype=torch.float64, device=device), upper=True)
    M = (T * sig) @ V.T            # m x d: R^{-1} diag(sig) V^T
    out = torch.empty((r1 - r0, d), dtype=torch.float32, device=device)
    for a in range(r0, r1, chunk):
        bnd = min(r1, a + chunk)
        out[a - r0:bnd - r0] = (_randn_rows(s, 1, a, bnd, m, device) @ M).to(torch.float32)
    return out

