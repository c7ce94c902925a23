"""Seeded synthetic workload generators shared by the oracle tests, the GPU
parity tests and bench.py.

This package holds NO arithmetic of the RBRP method (no norms, sampling,
pivoting, projection or interpolation): it only draws the input matrices of
BASELINE.json's configs (and scaled-down versions of them) from a seeded
generator.  Both the CPU oracle (`oracle/`) and the CUDA path consume its
output; neither imports the other.
"""
from .generators import CONFIGS, T3_RANKS, Config, make, small_config  # noqa: F401
