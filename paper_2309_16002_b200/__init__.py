"""B200-native robust blockwise random pivoting (RBRP), arXiv 2309.16002.

`librbrp.so` (C ABI, include/rbrp.h) runs the per-block adaptive-sampling loop
of Alg. 2 and the interpolation matrix of Alg. 3 as hand-written sm_100a
kernels; `paper_2309_16002_b200.rbrp` is the ctypes binding.
"""
from .rbrp import RBRPError, Result, id, id_host, lib, workspace_size  # noqa: F401

__all__ = ["id", "id_host", "lib", "workspace_size", "Result", "RBRPError"]
