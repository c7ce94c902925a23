"""Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as
easy as 1, 2, 3", SC'11) and the uniform map the sampler uses.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper does not say how the squared-norm distribution (Eq. 2.2)
is sampled ("Sample ... without replacement"); reading R8
fixes: draw j of block t uses counter (j, t, 0, 0) and key (seed_lo, seed_hi);
u_j = top 53 bits of (w1 << 32 | w0) times 2^-53, in [0, 1).

Written with Python integers, one 32-bit word at a time, so a reader can
check each round against the SC'11 definition: per round
    (hi0, lo0) = mulhilo(M0, c0);  (hi1, lo1) = mulhilo(M1, c2)
    c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
and the key is bumped by the Weyl constants (W0, W1) between rounds.
"""
from __future__ import annotations

import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """One Philox4x32-10 block: ctr = 4 x uint32, key = 2 x uint32 -> 4 x uint32."""
    c0, c1, c2, c3 = (int(x) & MASK for x in ctr)
    k0, k1 = (int(x) & MASK for x in key)
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + W0) & MASK
            k1 = (k1 + W1) & MASK
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK
        hi1, lo1 = p1 >> 32, p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & MASK, lo1, (hi0 ^ c3 ^ k1) & MASK, lo0
    return (c0, c1, c2, c3)


def u53(words) -> float:
    """U53 of the first two output words: ((w1 << 32 | w0) >> 11) * 2^-53."""
    x = ((int(words[1]) << 32) | int(words[0])) >> 11
    return x * (2.0 ** -53)


def seed_key(seed: int):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return (seed & MASK, seed >> 32)


def uniforms(seed: int, t: int, j0: int, count: int) -> np.ndarray:
    """u_j for draws j = j0 .. j0+count-1 of block t (counter (j, t, 0, 0))."""
    key = seed_key(seed)
    return np.array([u53(philox4x32_10((j, t, 0, 0), key)) for j in range(j0, j0 + count)],
                    dtype=np.float64)
