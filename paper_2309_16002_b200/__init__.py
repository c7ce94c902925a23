"""B200-native robust blockwise random pivoting (RBRP), arXiv 2309.16002.

`librbrp.so` (C ABI, include/rbrp.h) runs the per-block adaptive-sampling loop
of Alg. 2 and the interpolation matrix of Alg. 3 as hand-written sm_100a
kernels; `paper_2309_16002_b200.rbrp` is the ctypes binding.  The sketchy-pivoting
competitor SkLUPP-OSID (include/rbrp_sketch.h) is bound in `.sketch`.
"""
from .rbrp import RBRPError, Result, id, id_host, lib, workspace_size  # noqa: F401
from .sketch import gaussian_embedding, lupp, sketch_id  # noqa: F401

__all__ = ["id", "id_host", "lib", "workspace_size", "Result", "RBRPError", "gaussian_embedding", "lupp",
           "sketch_id"]
