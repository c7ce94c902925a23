"""Thin ctypes binding of the SkLUPP-OSID entry points (include/rbrp_sketch.h,
SURVEY NEXT-4): the Gaussian embedding, LUPP on a sketch and the full sketchy ID.

Argument marshalling only, as rbrp.py: torch supplies device memory and the current
stream; every step runs in librbrp.so's kernels, with no fallback.
"""
from __future__ import annotations

import ctypes
import dataclasses
from typing import List, Optional

import torch

from .rbrp import RBRPError, lib as _base_lib

SK_MAX_K = 512
SK_SHORT = 1
PHASES = ["embedding", "sketch", "lupp", "osid"]
EXPORTED = ["rbrp_gaussian_embedding", "rbrp_lupp_workspace_size", "rbrp_lupp",
            "rbrp_sketch_workspace_size", "rbrp_sketch_id"]


class SketchReport(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int64), ("flags", ctypes.c_uint32), ("ms_total", ctypes.c_float),
                ("profile", ctypes.c_int32), ("ms_phase", ctypes.c_float * 4), ("launches", ctypes.c_int32)]


_ready = False


def lib() -> ctypes.CDLL:
    global _ready
    L = _base_lib()
    if not _ready:
        P, I64, SZ, VP = ctypes.POINTER, ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p
        L.rbrp_gaussian_embedding.argtypes = [I64, I64, ctypes.c_uint64, VP, I64, VP]
        L.rbrp_lupp_workspace_size.argtypes = [I64, I64, I64, P(SZ)]
        L.rbrp_lupp.argtypes = [VP, I64, I64, I64, I64, VP, SZ, VP, P(I64), P(I64), P(I64), VP]
        L.rbrp_sketch_workspace_size.argtypes = [I64, I64, I64, I64, P(SZ)]
        L.rbrp_sketch_id.argtypes = [VP, I64, I64, I64, I64, I64, ctypes.c_uint64, VP, VP, SZ, VP,
                                     P(I64), VP, P(SketchReport)]
        for f in EXPORTED:
            getattr(L, f).restype = ctypes.c_int
        _ready = True
    return L


def _check(rc, what):
    if rc:
        raise RBRPError(rc, what)


def _stream(dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def gaussian_embedding(d: int, l: int, seed: int = 0, device="cuda") -> torch.Tensor:
    """Omega^T (l x d, fp64, on `device`), iid N(0, 1/l) by reading R25."""
    OmT = torch.empty((l, d), dtype=torch.float64, device=device)
    _check(lib().rbrp_gaussian_embedding(d, l, seed, ctypes.c_void_p(OmT.data_ptr()), d, _stream(OmT.device)),
           "gaussian_embedding")
    return OmT


@dataclasses.dataclass
class LUPPResult:
    piv: List[int]                  # pivot rows in order
    pcol: List[int]                 # column of each pivot
    L: Optional[torch.Tensor]       # n x k multipliers (device) if requested


def lupp(Y: torch.Tensor, k: int, with_L: bool = False) -> LUPPResult:
    """First k pivots of partial-pivoting LU on the CUDA fp64 matrix Y (n x l)
    (reading R26)."""
    if not Y.is_cuda or Y.dtype != torch.float64 or Y.dim() != 2 or Y.stride(1) != 1:
        raise ValueError("Y must be a row-major CUDA float64 matrix")
    L = lib()
    n, l = Y.shape
    sz = ctypes.c_size_t()
    _check(L.rbrp_lupp_workspace_size(n, l, k, ctypes.byref(sz)), "lupp_workspace_size")
    ws = torch.empty(sz.value, dtype=torch.uint8, device=Y.device)
    piv = (ctypes.c_int64 * k)()
    pcol = (ctypes.c_int64 * k)()
    npiv = ctypes.c_int64()
    Lm = torch.empty((n, k), dtype=torch.float64, device=Y.device) if with_L else None
    _check(L.rbrp_lupp(ctypes.c_void_p(Y.data_ptr()), n, l, Y.stride(0), k, ctypes.c_void_p(ws.data_ptr()),
                       sz.value, _stream(Y.device), piv, pcol, ctypes.byref(npiv),
                       ctypes.c_void_p(Lm.data_ptr()) if Lm is not None else None), "lupp")
    m = npiv.value
    return LUPPResult([int(piv[i]) for i in range(m)], [int(pcol[i]) for i in range(m)], Lm)


@dataclasses.dataclass
class SketchResult:
    S: torch.Tensor                 # int64 [k] on CPU, pivot order
    W: Optional[torch.Tensor]       # n x k on the device, W[S] = I
    k: int
    flags: int
    ms: float                       # device time of the call, ms
    ms_phase: dict                  # per-phase device ms (profile=True)
    launches: int


def sketch_workspace_size(n: int, d: int, k: int, l: int) -> int:
    sz = ctypes.c_size_t()
    _check(lib().rbrp_sketch_workspace_size(n, d, k, l, ctypes.byref(sz)), "sketch_workspace_size")
    return sz.value


def sketch_id(X: torch.Tensor, k: int, l: Optional[int] = None, seed: int = 0,
              omega_T: Optional[torch.Tensor] = None, with_W: bool = True, profile: bool = False,
              workspace: Optional[torch.Tensor] = None, W_out: Optional[torch.Tensor] = None) -> SketchResult:
    """SkLUPP-OSID of the CUDA fp64 matrix X (n x d): Y = X Omega, S = LUPP pivots of Y,
    W = Y Y_S^+ (Alg. 4).  l defaults to 3k; omega_T (l x d) overrides the
    seeded embedding."""
    if not X.is_cuda or X.dtype != torch.float64 or X.dim() != 2 or X.stride(1) != 1:
        raise ValueError("X must be a row-major CUDA float64 matrix")
    L = lib()
    n, d = X.shape
    l = 3 * k if l is None else l
    sz = sketch_workspace_size(n, d, k, l)
    if workspace is None or workspace.numel() < sz:
        workspace = torch.empty(sz, dtype=torch.uint8, device=X.device)
    if omega_T is not None:
        if omega_T.shape != (l, d) or omega_T.dtype != torch.float64 or not omega_T.is_contiguous():
            raise ValueError(f"omega_T must be a contiguous ({l}, {d}) float64 tensor")
    W = None
    if with_W:
        W = W_out if W_out is not None else torch.empty((n, k), dtype=torch.float64, device=X.device)
    S = torch.empty(k, dtype=torch.int64)
    rep = SketchReport()
    rep.profile = 1 if profile else 0
    _check(L.rbrp_sketch_id(ctypes.c_void_p(X.data_ptr()), n, d, X.stride(0), k, l, seed,
                            ctypes.c_void_p(omega_T.data_ptr()) if omega_T is not None else None,
                            ctypes.c_void_p(workspace.data_ptr()), sz, _stream(X.device),
                            ctypes.cast(S.data_ptr(), ctypes.POINTER(ctypes.c_int64)),
                            ctypes.c_void_p(W.data_ptr()) if W is not None else None, ctypes.byref(rep)),
           "sketch_id")
    return SketchResult(S[:rep.k], W, rep.k, rep.flags, rep.ms_total,
                        dict(zip(PHASES, list(rep.ms_phase))) if profile else {}, rep.launches)
