"""RBRP (Alg. 2), SRP (Alg. 1), the local Householder CPQR with the robust
filter (Remark 4.1) and the interpolation matrix (Alg. 3), written out step by
step from PAPER.md.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Never imported by the
product path; imports nothing from it.

Notation follows the paper: X (n x d) rows x_i, d^(t) residual squared row
norms, S skeletons in selection order, S_t the sampled block, V (d x b_t) its
residual columns, (Q_V, R_V, pi_V) the pivoted QR, b' the filtered rank,
Q'_V = Q_b the kept basis, L-hat the new columns of L.  Indices are 0-based
in code; the paper's 1-based i maps to i-1.

Readings of silent / ambiguous passages (DESIGN.md section "Readings") used
here: R1 loop sign '>' (Alg. 2 l.3; Alg. 1 l.3 P:289 garbled),
R4 tau_b = 1/b_t, R5 filter rule = l.8 literally, R6 without-replacement =
reject repeats of a fixed CDF, R7 small support, R8 Philox/CDF conventions,
R9 tie-break = lowest draw position, R10 diag(R_V) > 0, R13 L-hat on
skeleton rows, R14 clamp, R15 b_t = min(b, k-|S|), R19 precision policy.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence

import numpy as np
import scipy.linalg

from . import philox

# flags (same meaning as the report flags in include/rbrp.h; values restated)
F_TOL_UNREACHED = 1
F_ZERO_BLOCK = 2
F_W_CLIPPED = 4
F_SUPPORT_EXHAUSTED = 8
F_NEAR_TIE = 16

J_MAX = 1 << 20      # cap on draws per block (reading R6); never reached in practice


# --------------------------------------------------------------------------
# Alg. 2 l.2: d^(0)(i) = ||x_i||_2^2
# --------------------------------------------------------------------------
def row_sq_norms(X) -> np.ndarray:
    """d(i) = sum_j X(i,j)^2, accumulated in fp64 (reading R19)."""
    Xd = np.asarray(X, dtype=np.float64)
    return (Xd * Xd).sum(axis=1)


# --------------------------------------------------------------------------
# Alg. 2 l.5: S_t ~ d^(t-1) / ||d^(t-1)||_1 without replacement
# --------------------------------------------------------------------------
def sample_block(dvec: np.ndarray, b_t: int, seed: int, t: int):
    """Draw b_t distinct rows with the successive-sampling law of Eq. 2.2
     applied to d, 'without replacement' (footnote P:805).

    Reading R6: draws j = 0, 1, ... from the FIXED distribution d/||d||_1,
    rejecting indices already drawn in this block, until b_t are distinct --
    the same law as draw-and-zero (P(j | i drawn) = d_j / (D - d_i)).
    Reading R8: u_j = U53(Philox(ctr=(j, t, 0, 0), key=seed)); the row is the
    smallest i with C(i) > u_j * C(n-1), C the inclusive prefix sum of d in
    row order; a target past the end (rounding) maps to the last positive row.
    Reading R7: if at most b_t rows have d > 0, all of them are returned in
    row order and F_SUPPORT_EXHAUSTED is set.
    Returns (S_t in draw order, flags).
    """
    pos = np.flatnonzero(dvec > 0)
    if len(pos) <= b_t:
        return [int(i) for i in pos], F_SUPPORT_EXHAUSTED
    C = np.cumsum(dvec)
    total = C[-1]
    last_pos = int(pos[-1])
    chosen: List[int] = []
    seen = set()
    j = 0
    while len(chosen) < b_t and j < J_MAX:
        batch = philox.uniforms(seed, t, j, 4 * b_t)
        for u in batch:
            j += 1
            i = int(np.searchsorted(C, u * total, side="right"))
            if i >= len(C):
                i = last_pos
            if i not in seen:
                seen.add(i)
                chosen.append(i)
                if len(chosen) == b_t:
                    break
    return chosen, 0


def top_block(dvec: np.ndarray, b_t: int):
    """Remark 4.2 greedy variant: indices of the top-b_t entries
    of d (ties -> lower index), positive entries only."""
    order = sorted(range(len(dvec)), key=lambda i: (-dvec[i], i))
    return [int(i) for i in order[:b_t] if dvec[i] > 0]


# --------------------------------------------------------------------------
# Alg. 2 l.7: Q_V, R_V, pi_V = qr(V, "econ", "vector")
# --------------------------------------------------------------------------
@dataclasses.dataclass
class PivotedQR:
    Q: np.ndarray          # d x s, orthonormal columns (s = min(d, b))
    R: np.ndarray          # s x b, upper triangular, diag >= 0
    piv: np.ndarray        # permutation of range(b): V[:, piv] = Q R
    mass: np.ndarray       # mass[i] = ||R(i:, i:)||_F^2, i = 0..b-1
    gaps: np.ndarray       # per step: (best - second-best distinct residual) / avg


def cpqr(V, forced: Optional[Sequence[int]] = None) -> PivotedQR:
    """Householder QR with column pivoting (footnote P:182-184; Eq. 2.1
    P:181-188: pick the column of maximal residual norm, then reflect it).

    Residual column norms are recomputed exactly at every step (no
    downdating), so mass[i] = sum_{j>=i} (residual norm of column j)^2 before
    step i equals ||R_V(i:b, i:b)||_F^2 (the quantity of l.8, P:407 and of
    Remark 4.1).  Ties: lowest original position in V, i.e. draw order
    (reading R9).  Signs: diag(R) >= 0 (reading R10).  `forced` replays a
    given pivot order (forced-pivot replay mode)."""
    A = np.array(V, dtype=np.float64, copy=True)
    dd, b = A.shape
    s = min(dd, b)
    piv = np.arange(b)
    mass = np.zeros(b)
    gaps = np.full(b, np.inf)
    vs = []
    for i in range(b):
        res = (A[i:, i:] ** 2).sum(axis=0) if i < dd else np.zeros(b - i)
        mass[i] = res.sum()
        if i >= s:
            continue
        best = res.max()
        if forced is not None:
            p = i + int(np.flatnonzero(piv[i:] == forced[i])[0])
        else:
            ties = np.flatnonzero(res == best)
            p = i + int(ties[np.argmin(piv[i + ties])])
        lower = res[res < best]
        avg = mass[i] / (b - i)
        gaps[i] = (best - lower.max()) / avg if (len(lower) and avg > 0) else np.inf
        A[:, [i, p]] = A[:, [p, i]]
        piv[[i, p]] = piv[[p, i]]
        # Householder reflector H = I - 2 v v^T / (v^T v) on rows i.., zeroing A[i+1:, i]
        x = A[i:, i].copy()
        alpha = np.linalg.norm(x)
        v = x.copy()
        v[0] += alpha if x[0] >= 0 else -alpha
        vn = v @ v
        if vn > 0:
            A[i:, i:] -= np.outer(v, (2.0 / vn) * (v @ A[i:, i:]))
        vs.append((i, v, vn))
    R = np.triu(A[:s, :])
    # Q = H_0 H_1 ... H_{s-1} applied to the first s columns of the identity
    Q = np.eye(dd, s)
    for (i, v, vn) in reversed(vs):
        if vn > 0:
            Q[i:, :] -= np.outer(v, (2.0 / vn) * (v @ Q[i:, :]))
    sgn = np.where(np.diagonal(R)[:s] < 0, -1.0, 1.0)
    R = R * sgn[:, None]
    Q = Q * sgn[None, :]
    return PivotedQR(Q=Q, R=R, piv=piv, mass=mass, gaps=gaps)


def filter_rank(mass: np.ndarray, tau_b: float) -> int:
    """Alg. 2 l.8: b' = max{ i in [b] : ||R_V(i:b,i:b)||_F^2 >=
    tau_b ||R_V||_F^2 } (1-based i), with ||R_V||_F^2 = mass[0]; 0 if V = 0."""
    if len(mass) == 0 or mass[0] <= 0:
        return 0
    thr = tau_b * mass[0]
    keep = [i + 1 for i in range(len(mass)) if mass[i] >= thr]
    return max(keep) if keep else 0


# --------------------------------------------------------------------------
# Alg. 2
# --------------------------------------------------------------------------
@dataclasses.dataclass
class BlockLog:
    t: int
    S_t: List[int]
    b_t: int
    b_prime: int
    piv: List[int]
    mass: np.ndarray
    rho: float             # ||d^(t)||_1 / ||d^(0)||_1 after the block
    pivot_gap: float       # min relative pivot gap over the kept steps
    filter_margin: float   # |mass at the b' boundary - tau_b m_1| / m_1
    R_kept: np.ndarray     # R_V(1:b', 1:b')


@dataclasses.dataclass
class RBRPResult:
    S: List[int]
    L: np.ndarray          # n x k (config precision)
    Q: np.ndarray          # d x k
    d: np.ndarray          # final residual squared row norms
    D0: float
    blocks: List[BlockLog]
    flags: int

    @property
    def k(self):
        return len(self.S)

    @property
    def rho(self):
        return float(self.d.sum() / self.D0)


def rbrp(X, tau: Optional[float] = None, k: Optional[int] = None, b: int = 16,
         tau_b: float = -1.0, seed: int = 0, k_max: Optional[int] = None,
         greedy: bool = False, form: str = "residual",
         replay_blocks: Optional[Sequence[Sequence[int]]] = None,
         replay_pivots: Optional[Sequence[Sequence[int]]] = None) -> RBRPResult:
    """Robust blockwise random pivoting, Alg. 2.

    tau: relative squared-Frobenius tolerance (l.3, Remark 1.1 P:76-80);
    k: fixed rank instead of tau (l.3 "(or |S| < k)"); k_max caps |S| in tau
    mode; b: block size; tau_b: filter tolerance (< 0 -> 1/b_t, reading R4;
    0 -> plain BRP); greedy: RBGP (Remark 4.2); form: "residual"
    keeps X_res = X - L Q^T and updates it per block (P:523 footnote,
    north_star step 4) / "paper" runs l.6 and l.13 literally on X (CGS2 for
    l.6, reading R11); replay_*: forced candidate blocks / pivot orders."""
    X = np.asarray(X)
    wdt = np.float32 if X.dtype == np.float32 else np.float64
    X = X.astype(wdt, copy=False)
    n, dd = X.shape
    if tau is None and k is None:
        raise ValueError("need tau or k")
    cap = k if k is not None else (k_max if k_max else min(n, dd))
    # l.1
    S: List[int] = []
    Lcols: List[np.ndarray] = []
    Q = np.zeros((dd, 0), dtype=np.float64)
    t = 0
    # l.2
    d0 = row_sq_norms(X)
    D0 = float(d0.sum())
    dvec = d0.copy()
    Xres = X.copy() if form == "residual" else None
    blocks: List[BlockLog] = []
    flags = 0
    if D0 == 0:
        raise ValueError("X = 0 (degenerate)")

    def more():
        if len(S) >= cap:
            return False
        if k is not None:
            return True
        return dvec.sum() > tau * D0           # l.3 with reading R1 ('>')

    while more():
        # l.4
        t += 1
        b_t = min(b, cap - len(S))
        # l.5
        if replay_blocks is not None:
            if t - 1 >= len(replay_blocks):
                break
            S_t = [int(i) for i in replay_blocks[t - 1]]
        elif greedy:
            S_t = top_block(dvec, b_t)
            if len(S_t) < b_t:
                flags |= F_SUPPORT_EXHAUSTED
        else:
            S_t, f = sample_block(dvec, b_t, seed, t)
            flags |= f
        b_t = len(S_t)
        if b_t == 0:
            break
        # l.6: V = X(S_t,:)^T - Q (Q^T X(S_t,:)^T)
        if form == "residual":
            V = Xres[S_t].astype(np.float64).T
        else:
            Xs = X[S_t].astype(np.float64).T
            V = Xs - Q @ (Q.T @ Xs)
            V = V - Q @ (Q.T @ V)
        # l.7
        forced = replay_pivots[t - 1] if replay_pivots is not None else None
        qr = cpqr(V, forced=forced)
        # l.8
        tb = (1.0 / b_t) if tau_b < 0 else tau_b
        bp = filter_rank(qr.mass, tb)
        if bp == 0:
            flags |= F_ZERO_BLOCK
            break
        # l.9
        Sp = [S_t[int(qr.piv[i])] for i in range(bp)]
        Qb = qr.Q[:, :bp]
        # l.10
        Q = np.concatenate([Q, Qb], axis=1)
        # l.11-13: L-hat(pi_a,:) = X(pi_a,:) Q'_V; pi_a excludes earlier skeletons
        Qw = Qb.astype(wdt)
        Lhat = (Xres @ Qw) if form == "residual" else (X @ Qw)
        if S:
            Lhat[S] = 0
        Lhat[Sp] = qr.R[:bp, :bp].T.astype(wdt)        # reading R13
        # l.14-15
        S_prev = list(S)
        S.extend(Sp)
        Lcols.append(Lhat)
        # l.16
        if form == "residual":
            Xres -= Lhat @ Qw.T
            Xres[S] = 0
            dvec = row_sq_norms(Xres)
        else:
            dvec = np.maximum(dvec - row_sq_norms(Lhat), 0.0)   # reading R14
        dvec[S] = 0.0
        del S_prev
        gap = float(np.min(qr.gaps[:bp])) if bp > 0 else np.inf
        thr = tb * qr.mass[0]
        fm = abs(qr.mass[bp - 1] - thr)
        if bp < len(qr.mass):
            fm = min(fm, abs(qr.mass[bp] - thr))
        blocks.append(BlockLog(t=t, S_t=S_t, b_t=b_t, b_prime=bp, piv=[int(p) for p in qr.piv],
                               mass=qr.mass, rho=float(dvec.sum() / D0), pivot_gap=gap,
                               filter_margin=float(fm / qr.mass[0]), R_kept=qr.R[:bp, :bp].copy()))
    if k is None and dvec.sum() > tau * D0:
        flags |= F_TOL_UNREACHED
    L = np.concatenate(Lcols, axis=1) if Lcols else np.zeros((n, 0), dtype=wdt)
    return RBRPResult(S=S, L=L, Q=Q, d=dvec, D0=D0, blocks=blocks, flags=flags)


# --------------------------------------------------------------------------
# Alg. 1: sequential random pivoting, verbatim
# --------------------------------------------------------------------------
def srp(X, tau: Optional[float] = None, k: Optional[int] = None, seed: int = 0,
        k_max: Optional[int] = None):
    """Alg. 1 with the loop sign of reading R1.  Line 5's draw uses
    the block sampler with b_t = 1 and block counter t (reading R8), so SRP
    and RBRP(b=1) consume the same random numbers.  Returns (S, L, d)."""
    X = np.asarray(X, dtype=np.float64)
    n, dd = X.shape
    cap = k if k is not None else (k_max if k_max else min(n, dd))
    # l.1
    S: List[int] = []
    Lcols = []
    Q = np.zeros((dd, 0))
    t = 0
    # l.2
    d0 = row_sq_norms(X)
    dvec = d0.copy()
    while len(S) < cap and (k is not None or dvec.sum() > tau * d0.sum()):
        # l.4
        t += 1
        # l.5
        drawn, _ = sample_block(dvec, 1, seed, t)
        if not drawn:
            break
        s = drawn[0]
        # l.6-7: pi_a = pi(t:n) = everything but the previous skeletons
        S_prev = list(S)
        S.append(s)
        # l.8
        v = X[s] - Q @ (Q.T @ X[s])
        # l.10
        Q = np.concatenate([Q, (v / np.linalg.norm(v))[:, None]], axis=1)
        # l.12
        a = X @ v
        a[S_prev] = 0.0
        # l.14
        Lcols.append(a / np.sqrt(a[s]))
        # l.16
        dvec = dvec - a * a / a[s]
        dvec[S] = 0.0
        dvec = np.maximum(dvec, 0.0)
    L = np.stack(Lcols, axis=1) if Lcols else np.zeros((n, 0))
    return S, L, dvec


# --------------------------------------------------------------------------
# Alg. 3 and Remark 5.2
# --------------------------------------------------------------------------
def form_W(L, S: Sequence[int], method: str = "pinv", clip: float = 1e-12):
    """W(S,:) = I_k, W(rest,:) = L_2 L_1^{-1} (Alg. 3), computed in
    fp64.  method "pinv": L_1^{-1} by SVD with singular values below
    clip * sigma_max discarded (Remark 5.2; reading R17).
    method "trsm": substitution on the lower-triangular L_1.
    Returns (W, kappa(L_1), clipped?)."""
    L = np.asarray(L, dtype=np.float64)
    n, k = L.shape
    S = list(S)
    rest = np.setdiff1d(np.arange(n), np.asarray(S, dtype=np.int64))
    L1 = L[S]
    W = np.zeros((n, k))
    W[S] = np.eye(k)
    sv = np.linalg.svd(L1, compute_uv=False)
    kappa = float(sv[0] / sv[-1]) if sv[-1] > 0 else np.inf
    clipped = bool(sv[-1] < clip * sv[0])
    if method == "pinv":
        U, s, Vt = np.linalg.svd(L1)
        keep = s >= clip * s[0]
        L1p = (Vt[keep].T / s[keep]) @ U[:, keep].T
        W[rest] = L[rest] @ L1p
    elif method == "trsm":
        # W L_1 = L_2  <=>  L_1^T W^T = L_2^T, L_1^T upper triangular
        W[rest] = scipy.linalg.solve_triangular(L1, L[rest].T, lower=True, trans="T").T
    else:
        raise ValueError(method)
    return W, kappa, clipped
