"""Sketchy pivoting with LUPP (SkLUPP, section 3.2) and the oversampled
sketchy interpolation matrix (OSID, Alg. 4 and Eq. 5.3): SURVEY section 8(f)
NEXT-4, the paper's fastest GPU competitor (Table 3).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain NumPy, fp64, no blocking.

  gaussian_embedding(d, l, seed)  Omega (d x l), iid N(0, 1/l) (Prop. 5.3, P:643;
                                  Remark 3.2), drawn with Philox4x32-10 and the
                                  Box-Muller transform (reading R25).
  sketch(X, Omega)                Y = X Omega ("the sketched sample matrix";
                                  Alg. 4 l.1).
  lupp(Y, k)                      the first k pivot rows of LU with partial pivoting on Y
                                  ("LUPP [GVL 3.4] ... on Y"); reading R26.
  osid_w(Y, S)                    W(S,:) = I_k, W(rest,:) = (Y(rest,:) Q) R^{-T} with
                                  Y_S^T = Q R (Alg. 4 l.2-4; Eq. 5.3).
  sketchy_id(X, k, Omega)         S = lupp(X Omega, k), W = osid_w(X Omega, S).

Reading R25 (the paper names no generator): entry (j, i) of Omega^T (row j < l, column
i < d; e = j d + i) is normal number e % 2 of Philox block q = e // 2 with counter
(q_lo, q_hi, 0, 0x4F4D4547) and key (seed_lo, seed_hi); with u1 = U53(w0, w1),
u2 = U53(w2, w3): r = sqrt(-2 ln(1 - u1)), z0 = r cos(2 pi u2), z1 = r sin(2 pi u2),
entry = z / sqrt(l).  The fourth counter word keeps these blocks apart from the
sampler's (j, t, 0, 0).

Reading R26 (LUPP conventions the paper leaves to [GVL 3.4]): rows are not swapped;
step m takes the active column c (starting at 0) and pivots on the active row of
largest |A(i, c)|, ties to the lowest row index; an exactly zero active column is
skipped (c advances, no pivot); the Schur update of every other active row is
A(i, c+1:) -= l_i A(p, c+1:) with l_i = A(i, c) / A(p, c), the product rounded before
the subtraction (NumPy's outer product, no fused multiply-add).  Stop after k pivots
or when the columns run out (short output).
"""
from __future__ import annotations

import dataclasses
from typing import List, Sequence

import numpy as np
import scipy.linalg

from . import philox

OMEGA_TAG = 0x4F4D4547   # counter word 3 of the embedding's Philox blocks (reading R25)


def gaussian_embedding(d: int, l: int, seed: int) -> np.ndarray:
    """Omega (d x l) with iid N(0, 1/l) entries, by reading R25.  Pure Python
    per Philox block: for small d * l only."""
    key = philox.seed_key(seed)
    total = d * l
    vals = np.empty(total + (total & 1))
    for q in range((total + 1) // 2):
        w = philox.philox4x32_10((q & 0xFFFFFFFF, q >> 32, 0, OMEGA_TAG), key)
        u1 = philox.u53(w[0:2])
        u2 = philox.u53(w[2:4])
        r = np.sqrt(-2.0 * np.log(1.0 - u1))
        vals[2 * q] = r * np.cos(2.0 * np.pi * u2)
        vals[2 * q + 1] = r * np.sin(2.0 * np.pi * u2)
    OmT = vals[:total].reshape(l, d) / np.sqrt(l)   # row j of Omega^T
    return OmT.T.copy()


def sketch(X, Omega) -> np.ndarray:
    """Y = X Omega (Alg. 4 l.1), fp64."""
    return np.asarray(X, dtype=np.float64) @ np.asarray(Omega, dtype=np.float64)


@dataclasses.dataclass
class LUPP:
    piv: List[int]        # pivot rows in selection order (S = piv[:k])
    pcol: List[int]       # active column of each pivot (differs from m after a skip)
    L: np.ndarray         # n x k multipliers: L[i, m] = l_i of step m for rows active then
    U: np.ndarray         # k x l: U[m, c] = A(piv[m], c) at step m for c >= pcol[m], else 0
    short: bool           # fewer than k pivots (columns exhausted)


def lupp(Y, k: int) -> LUPP:
    """Partial-pivoting LU on Y (n x l), first k steps, reading R26."""
    A = np.array(Y, dtype=np.float64, copy=True)
    n, l = A.shape
    active = np.ones(n, dtype=bool)
    L = np.zeros((n, k))
    U = np.zeros((k, l))
    piv: List[int] = []
    pcol: List[int] = []
    c = 0
    while len(piv) < k and c < l and active.any():
        mag = np.abs(A[:, c])
        mag[~active] = -1.0
        p = int(np.argmax(mag))          # first maximum: ties to the lowest row
        if not mag[p] > 0.0:             # exactly zero active column: skip it
            c += 1
            continue
        m = len(piv)
        U[m, c:] = A[p, c:]
        active[p] = False
        rows = np.nonzero(active)[0]
        lv = A[rows, c] / A[p, c]
        L[rows, m] = lv
        A[np.ix_(rows, np.arange(c + 1, l))] -= np.outer(lv, A[p, c + 1:])
        piv.append(p)
        pcol.append(c)
        c += 1
    return LUPP(piv, pcol, L, U, len(piv) < k)


def osid_w(Y, S: Sequence[int]) -> np.ndarray:
    """Alg. 4: Q, R = qr(Y(S,:)^T, "econ"); W = 0; W(S,:) = I_k;
    W(rest,:) = (Y(rest,:) Q) R^{-T}  (Eq. 5.3: W = Y Y_S^+)."""
    Y = np.asarray(Y, dtype=np.float64)
    S = list(S)
    n, k = Y.shape[0], len(S)
    Q, R = np.linalg.qr(Y[S].T, mode="reduced")               # l.2
    W = np.zeros((n, k))                                        # l.3
    W[S] = np.eye(k)
    rest = np.setdiff1d(np.arange(n), np.asarray(S, dtype=np.int64))
    YQ = Y[rest] @ Q                                            # l.4: (Y(rest) Q) R^{-T}
    W[rest] = scipy.linalg.solve_triangular(R, YQ.T, lower=False).T   # R W^T = (Y Q)^T
    return W


def sketchy_id(X, k: int, Omega):
    """SkLUPP-OSID: Y = X Omega, S = first k LUPP pivots of Y, W = osid_w(Y, S)."""
    Y = sketch(X, Omega)
    f = lupp(Y, k)
    W = osid_w(Y, f.piv)
    return f, W, Y
