"""Referee quantities, independent of the RBRP loop.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  errskel(X, S)   = ||X - X X_S^+ X_S||_F^2                 Eq. 1.2
  errid(X, S, W)  = ||X - W X_S||_F^2
  eta(X, r)       = ||X - [X]_r||_F^2 / ||X||_F^2            Eq. 1.3
  best_subset     = min over |S| = k of errskel (brute force, tiny inputs)
All in fp64.
"""
from __future__ import annotations

import itertools
from typing import Sequence

import numpy as np


def _row_space_basis(Xs: np.ndarray) -> np.ndarray:
    """Orthonormal basis (d x rank) of the row space of X_S, by SVD with the
    usual numerical-rank cut (max(shape) * eps * sigma_max)."""
    if Xs.shape[0] == 0:
        return np.zeros((Xs.shape[1], 0))
    _, s, Vt = np.linalg.svd(Xs, full_matrices=False)
    tol = max(Xs.shape) * np.finfo(np.float64).eps * (s[0] if len(s) else 0.0)
    return Vt[s > tol].T


def errskel(X, S: Sequence[int]) -> float:
    """Eq. 1.2: X X_S^+ X_S is the projection of each row onto the
    row space of X_S; computed directly as X - (X B) B^T (no norm downdating)."""
    X = np.asarray(X, dtype=np.float64)
    B = _row_space_basis(X[list(S)])
    E = X - (X @ B) @ B.T
    return float((E * E).sum())


def errid(X, S: Sequence[int], W) -> float:
    """Interpolation error ||X - W X_S||_F^2."""
    X = np.asarray(X, dtype=np.float64)
    E = X - np.asarray(W, dtype=np.float64) @ X[list(S)]
    return float((E * E).sum())


def eta(X, r: int) -> float:
    """Relative tail eta_r (Eq. 1.3) from the singular values."""
    X = np.asarray(X, dtype=np.float64)
    if X.shape[0] > 4 * X.shape[1]:
        # tall: eigenvalues of the d x d Gram are sigma_i^2
        ev = np.linalg.eigvalsh(X.T @ X)[::-1]
        s2 = np.maximum(ev, 0.0)
    else:
        s2 = np.linalg.svd(X, compute_uv=False) ** 2
    return float(s2[r:].sum() / s2.sum())


def tail(X, r: int) -> float:
    """||X - [X]_r||_F^2 (absolute)."""
    X = np.asarray(X, dtype=np.float64)
    return eta(X, r) * float((X * X).sum())


def best_subset(X, k: int):
    """Brute-force min over all |S| = k of errskel(X, S) (tiny inputs only)."""
    X = np.asarray(X, dtype=np.float64)
    best, arg = np.inf, None
    for S in itertools.combinations(range(X.shape[0]), k):
        e = errskel(X, S)
        if e < best:
            best, arg = e, S
    return best, arg
