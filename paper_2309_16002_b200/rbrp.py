"""Thin ctypes binding of librbrp.so (include/rbrp.h).

Argument marshalling only: torch supplies device memory (workspace, W) and the
current CUDA stream; every step of RBRP runs in the library's sm_100a kernels.
There is no CPU or PyTorch fallback: if the library cannot be loaded, every
call raises.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import threading
from typing import List, Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RBRP_LIB_PATH") or os.path.join(_HERE, "lib", "librbrp.so")

RBRP_F32, RBRP_F64 = 0, 1
RBRP_INPLACE, RBRP_NO_W, RBRP_FORM_PAPER = 1, 2, 4
F_TOL_UNREACHED, F_ZERO_BLOCK, F_W_CLIPPED, F_SUPPORT_EXHAUSTED, F_NEAR_TIE = 1, 2, 4, 8, 16
CHUNK = 4096
MAX_B = 128

STATUS = {0: "RBRP_OK", -1: "RBRP_EINVAL", -2: "RBRP_ENONFINITE", -3: "RBRP_EDEGENERATE",
          -4: "RBRP_ENOMEM", -5: "RBRP_ECUDA", -6: "RBRP_ENCCL", -7: "RBRP_EREPLAY",
          -8: "RBRP_ENOTSUP"}

EXPORTED = ["rbrp_version", "rbrp_strerror", "rbrp_workspace_size", "rbrp_id", "rbrp_id_sharded",
            "rbrp_comm_unique_id", "rbrp_comm_init", "rbrp_comm_destroy", "rbrp_form_w",
            "rbrp_form_w_workspace_size", "rbrp_id_host", "rbrp_workspace_size_host"]


class Problem(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int), ("n_global", ctypes.c_int64), ("n_local", ctypes.c_int64),
                ("row_offset", ctypes.c_int64), ("d", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("tol", ctypes.c_double), ("k_max", ctypes.c_int64), ("b", ctypes.c_int32),
                ("tau_b", ctypes.c_double), ("greedy", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("flags", ctypes.c_uint32), ("replay_blocks", ctypes.POINTER(ctypes.c_int64)),
                ("replay_lens", ctypes.POINTER(ctypes.c_int32)),
                ("replay_pivots", ctypes.POINTER(ctypes.c_int32)),
                ("replay_nblocks", ctypes.c_int32)]


class Report(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int64), ("resid_rel", ctypes.c_double), ("fro2", ctypes.c_double),
                ("nblocks", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("max_blocks", ctypes.c_int32), ("b_t", ctypes.POINTER(ctypes.c_int32)),
                ("b_prime", ctypes.POINTER(ctypes.c_int32)), ("rho", ctypes.POINTER(ctypes.c_double)),
                ("block_idx", ctypes.POINTER(ctypes.c_int64)),
                ("block_piv", ctypes.POINTER(ctypes.c_int32)), ("ms_total", ctypes.c_float),
                ("profile", ctypes.c_int32), ("ms_phase", ctypes.c_float * 8),
                ("launches", ctypes.c_int32), ("proj_calls", ctypes.c_int32),
                ("proj_ms", ctypes.c_float), ("graph", ctypes.c_int32),
                ("proj_ms_blk", ctypes.POINTER(ctypes.c_float)), ("d_out", ctypes.c_void_p)]

PHASES = ["init", "sample", "filter", "projection", "unused", "fixup_scan", "W", "comm"]


class RBRPError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}{': ' + what if what else ''}")


_lib = None
_tls = threading.local()


def lib() -> ctypes.CDLL:
    """Load librbrp.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"librbrp.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        L.rbrp_version.restype = ctypes.c_int
        L.rbrp_strerror.restype = ctypes.c_char_p
        L.rbrp_strerror.argtypes = [ctypes.c_int]
        L.rbrp_workspace_size.argtypes = [ctypes.POINTER(Problem), ctypes.POINTER(ctypes.c_size_t)]
        L.rbrp_workspace_size.restype = ctypes.c_int
        L.rbrp_id.argtypes = [ctypes.POINTER(Problem), ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.POINTER(Report)]
        L.rbrp_id.restype = ctypes.c_int
        L.rbrp_id_sharded.argtypes = [ctypes.POINTER(Problem), ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_void_p),
                                      ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_void_p,
                                      ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_void_p),
                                      ctypes.POINTER(Report)]
        L.rbrp_id_sharded.restype = ctypes.c_int
        L.rbrp_comm_unique_id.argtypes = [ctypes.c_void_p]
        L.rbrp_comm_init.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int]
        L.rbrp_comm_destroy.argtypes = [ctypes.c_void_p]
        L.rbrp_form_w_workspace_size.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_size_t)]
        L.rbrp_form_w_workspace_size.restype = ctypes.c_int
        L.rbrp_form_w.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                  ctypes.POINTER(ctypes.c_int64), ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                  ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                  ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int32)]
        L.rbrp_form_w.restype = ctypes.c_int
        L.rbrp_workspace_size_host.argtypes = [ctypes.POINTER(Problem), ctypes.POINTER(ctypes.c_size_t)]
        L.rbrp_workspace_size_host.restype = ctypes.c_int
        L.rbrp_id_host.argtypes = [ctypes.POINTER(Problem), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                   ctypes.c_void_p, ctypes.POINTER(Report)]
        L.rbrp_id_host.restype = ctypes.c_int
        _lib = L
    return _lib


@dataclasses.dataclass
class Result:
    S: torch.Tensor                 # int64 [k] on CPU, selection order
    W: Optional[torch.Tensor]       # [n_local, k] on the device (None with with_W=False)
    k: int
    resid_rel: float                # ||d||_1 / ||d0||_1 = errskel / ||X||_F^2
    fro2: float
    flags: int
    nblocks: int
    b_t: List[int]
    b_prime: List[int]
    rho: List[float]
    blocks: List[List[int]]         # candidate blocks S_t (global ids, draw order)
    pivots: List[List[int]]         # local pivot orders
    ms: float                       # device time of the call (CUDA events), ms
    ms_phase: dict                  # per-phase device ms (profile=True)
    launches: int                   # kernels launched by the call
    proj_calls: int
    proj_ms: float                  # device time of the projection passes (in-kernel stamps)
    graph: bool                     # block loop ran as one CUDA graph launch
    proj_ms_blk: List[float] = dataclasses.field(default_factory=list)   # per block
    d: Optional[torch.Tensor] = None  # final residual squared row norms (return_d=True), device


def _problem(X: torch.Tensor, tol, k, b, seed, k_max, tau_b, flags, n_global, row_offset, greedy):
    if X.dim() != 2 or X.stride(1) != 1:
        raise ValueError("X must be a 2-D row-major tensor (stride(1) == 1)")
    if X.dtype not in (torch.float32, torch.float64):
        raise ValueError("X must be float32 or float64")
    p = Problem()
    p.dtype = RBRP_F64 if X.dtype == torch.float64 else RBRP_F32
    p.n_local = X.shape[0]
    p.n_global = n_global if n_global is not None else X.shape[0]
    p.row_offset = row_offset
    p.d = X.shape[1]
    p.ld = X.stride(0) if X.shape[0] > 1 else X.shape[1]
    if k is not None:
        p.tol = 0.0
        p.k_max = int(k)
    else:
        p.tol = float(tol)
        p.k_max = int(k_max or 0)
    p.b = int(b)
    p.tau_b = float(tau_b)
    p.greedy = int(bool(greedy))
    p.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    p.flags = flags
    p.replay_nblocks = 0
    return p


def workspace_size(X: torch.Tensor, tol=None, k=None, b=16, k_max=0, tau_b=-1.0, with_W=True,
                   inplace=False, n_global=None, row_offset=0) -> int:
    flags = (0 if with_W else RBRP_NO_W) | (RBRP_INPLACE if inplace else 0)
    p = _problem(X, tol, k, b, 0, k_max, tau_b, flags, n_global, row_offset, False)
    sz = ctypes.c_size_t()
    rc = lib().rbrp_workspace_size(ctypes.byref(p), ctypes.byref(sz))
    if rc:
        raise RBRPError(rc)
    return sz.value


def id(X: torch.Tensor, tol: Optional[float] = None, k: Optional[int] = None, b: int = 16,
       seed: int = 0, k_max: int = 0, tau_b: float = -1.0, with_W: bool = True,
       inplace: bool = False, greedy: bool = False,
       replay_blocks: Optional[Sequence[Sequence[int]]] = None,
       replay_pivots: Optional[Sequence[Sequence[int]]] = None,
       max_blocks: int = 1024, log_blocks: bool = True, workspace: Optional[torch.Tensor] = None,
       comm=None, n_global: Optional[int] = None, row_offset: int = 0,
       profile: bool = False, W_out: Optional[torch.Tensor] = None, form: str = "residual",
       return_d: bool = False) -> Result:
    """RBRP interpolative decomposition X ~ W X_S of a CUDA tensor X (n x d).

    tol: tau, relative to ||X||_F^2 (for an (r, eps)-ID pass tol = (1+eps) eta_r,
    PAPER.md l.86); or k: fixed rank.  b: block size; seed: Philox key;
    tau_b < 0 -> 1/b_t.  Returns S (CPU int64, selection order), W (device,
    n x k, W[S] = I) and the per-block log.  workspace / W_out: optional
    preallocated buffers (W_out: n x k_cap, k_cap = k or k_max or min(n, d)).
    form: "residual" (north_star: X_res updated per block, exact residual norms) or
    "paper" (Alg. 2 literally: X read only, CGS2 for l.6, downdated norms l.16).
    return_d: also return the final residual squared row norms d (Result.d, device fp64).
    replay_pivots: a block whose list starts with -1 is not forced (NEAR_TIE rule)."""
    if not X.is_cuda:
        raise ValueError("X must be a CUDA tensor (use id_host for host buffers)")
    if tol is None and k is None:
        raise ValueError("need tol or k")
    L = lib()
    if form not in ("residual", "paper"):
        raise ValueError("form must be 'residual' or 'paper'")
    flags = ((0 if with_W else RBRP_NO_W) | (RBRP_INPLACE if inplace else 0)
             | (RBRP_FORM_PAPER if form == "paper" else 0))
    p = _problem(X, tol, k, b, seed, k_max, tau_b, flags, n_global, row_offset, greedy)
    keep = []
    if replay_blocks is not None:
        flat = [int(i) for blk in replay_blocks for i in blk]
        lens = [len(blk) for blk in replay_blocks]
        arr = (ctypes.c_int64 * max(1, len(flat)))(*flat)
        la = (ctypes.c_int32 * max(1, len(lens)))(*lens)
        p.replay_blocks = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int64))
        p.replay_lens = ctypes.cast(la, ctypes.POINTER(ctypes.c_int32))
        p.replay_nblocks = len(lens)
        keep += [arr, la]
        if replay_pivots is not None:
            fp = [int(i) for blk in replay_pivots for i in blk]
            pa = (ctypes.c_int32 * max(1, len(fp)))(*fp)
            p.replay_pivots = ctypes.cast(pa, ctypes.POINTER(ctypes.c_int32))
            keep.append(pa)
    sz = ctypes.c_size_t()
    rc = L.rbrp_workspace_size(ctypes.byref(p), ctypes.byref(sz))
    if rc:
        raise RBRPError(rc, "workspace_size")
    if workspace is None or workspace.numel() < sz.value:
        workspace = torch.empty(sz.value, dtype=torch.uint8, device=X.device)
    ws_bytes = sz.value
    k_cap = p.k_max if p.k_max > 0 else min(p.n_global, p.d)
    W = None
    if with_W:
        if W_out is not None:
            if (W_out.shape != (X.shape[0], k_cap) or W_out.dtype != X.dtype or not W_out.is_contiguous()
                    or W_out.device != X.device):
                raise ValueError(f"W_out must be a contiguous {(X.shape[0], k_cap)} {X.dtype} tensor on {X.device}")
            W = W_out
        else:
            W = torch.empty((X.shape[0], k_cap), dtype=X.dtype, device=X.device)
    mb = max_blocks
    # host buffers of the report, reused across calls of the same shape (per thread)
    key = (mb, b if log_blocks else 0, k_cap)
    cache = _tls.__dict__.setdefault("bufs", {})
    if key not in cache:
        if len(cache) > 16:
            cache.clear()
        rep = _with_proj_blk(Report(), mb)
        b_t = (ctypes.c_int32 * mb)()
        b_pr = (ctypes.c_int32 * mb)()
        rho = (ctypes.c_double * mb)()
        rep.max_blocks = mb
        rep.b_t = ctypes.cast(b_t, ctypes.POINTER(ctypes.c_int32))
        rep.b_prime = ctypes.cast(b_pr, ctypes.POINTER(ctypes.c_int32))
        rep.rho = ctypes.cast(rho, ctypes.POINTER(ctypes.c_double))
        bidx = bpiv = None
        if log_blocks:
            bidx = (ctypes.c_int64 * (mb * b))()
            bpiv = (ctypes.c_int32 * (mb * b))()
            rep.block_idx = ctypes.cast(bidx, ctypes.POINTER(ctypes.c_int64))
            rep.block_piv = ctypes.cast(bpiv, ctypes.POINTER(ctypes.c_int32))
        S = torch.empty(k_cap, dtype=torch.int64)
        cache[key] = (rep, b_t, b_pr, rho, bidx, bpiv, S)
    rep, b_t, b_pr, rho, bidx, bpiv, S = cache[key]
    rep.profile = 1 if profile else 0
    dv = torch.empty(X.shape[0], dtype=torch.float64, device=X.device) if return_d else None
    rep.d_out = dv.data_ptr() if dv is not None else None
    stream = torch.cuda.current_stream(X.device).cuda_stream
    rc = L.rbrp_id(ctypes.byref(p), ctypes.c_void_p(X.data_ptr()),
                   ctypes.c_void_p(workspace.data_ptr()), ws_bytes,
                   ctypes.c_void_p(comm) if comm else None, ctypes.c_void_p(stream),
                   ctypes.cast(S.data_ptr(), ctypes.POINTER(ctypes.c_int64)),
                   ctypes.c_void_p(W.data_ptr()) if W is not None else None, ctypes.byref(rep))
    if rc:
        raise RBRPError(rc, L.rbrp_strerror(rc).decode())
    res = _result(rep, S, W, b_t, b_pr, rho, bidx if log_blocks else None, bpiv if log_blocks else None,
                  mb, b, log_blocks)
    res.d = dv
    return res


def _result(rep, S, W, b_t, b_pr, rho, bidx, bpiv, mb, b, log_blocks):
    kk = rep.k
    nb = min(rep.nblocks, mb)
    blocks, pivots = [], []
    if log_blocks:
        for t in range(nb):
            bt = b_t[t]
            blocks.append([bidx[t * b + i] for i in range(bt)])
            pivots.append([bpiv[t * b + i] for i in range(bt)])
    return Result(S=S[:kk].clone(), W=W[:, :kk] if W is not None else None, k=kk,
                  resid_rel=rep.resid_rel, fro2=rep.fro2, flags=rep.flags, nblocks=rep.nblocks,
                  b_t=list(b_t[:nb]), b_prime=list(b_pr[:nb]), rho=list(rho[:nb]),
                  blocks=blocks, pivots=pivots, ms=rep.ms_total,
                  ms_phase={nm: rep.ms_phase[i] for i, nm in enumerate(PHASES)},
                  launches=rep.launches, proj_calls=rep.proj_calls, proj_ms=rep.proj_ms,
                  graph=bool(rep.graph), proj_ms_blk=list(rep._pms[:nb]) if hasattr(rep, "_pms") else [])


def _with_proj_blk(rep, mb):
    """attach the optional per-block projection-time array (kept alive on the report)"""
    rep._pms = (ctypes.c_float * mb)()
    rep.proj_ms_blk = ctypes.cast(rep._pms, ctypes.POINTER(ctypes.c_float))
    return rep


def _report(mb, b, log_blocks):
    rep = _with_proj_blk(Report(), mb)
    b_t = (ctypes.c_int32 * mb)()
    b_pr = (ctypes.c_int32 * mb)()
    rho = (ctypes.c_double * mb)()
    rep.max_blocks = mb
    rep.b_t = ctypes.cast(b_t, ctypes.POINTER(ctypes.c_int32))
    rep.b_prime = ctypes.cast(b_pr, ctypes.POINTER(ctypes.c_int32))
    rep.rho = ctypes.cast(rho, ctypes.POINTER(ctypes.c_double))
    bidx = bpiv = None
    if log_blocks:
        bidx = (ctypes.c_int64 * (mb * b))()
        bpiv = (ctypes.c_int32 * (mb * b))()
        rep.block_idx = ctypes.cast(bidx, ctypes.POINTER(ctypes.c_int64))
        rep.block_piv = ctypes.cast(bpiv, ctypes.POINTER(ctypes.c_int32))
    return rep, b_t, b_pr, rho, bidx, bpiv


def id_sharded(shards: Sequence[torch.Tensor], tol: Optional[float] = None, k: Optional[int] = None,
               b: int = 16, seed: int = 0, k_max: int = 0, tau_b: float = -1.0, with_W: bool = True,
               replay_blocks=None, replay_pivots=None, max_blocks: int = 1024, form: str = "residual"):
    """The row-sharded (multi-GPU) algorithm over in-process shards on one device:
    `shards` are consecutive row blocks of X (every one but the last a multiple of
    4096 rows).  Returns (Result of shard 0 with W = None, [W_h per shard])."""
    L = lib()
    X0 = shards[0]
    n_global = sum(int(x.shape[0]) for x in shards)
    flags = (0 if with_W else RBRP_NO_W) | (RBRP_FORM_PAPER if form == "paper" else 0)
    p = _problem(X0, tol, k, b, seed, k_max, tau_b, flags, n_global, 0, False)
    keep = []
    if replay_blocks is not None:
        flat = [int(i) for blk in replay_blocks for i in blk]
        lens = [len(blk) for blk in replay_blocks]
        arr = (ctypes.c_int64 * max(1, len(flat)))(*flat)
        la = (ctypes.c_int32 * max(1, len(lens)))(*lens)
        p.replay_blocks = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int64))
        p.replay_lens = ctypes.cast(la, ctypes.POINTER(ctypes.c_int32))
        p.replay_nblocks = len(lens)
        keep += [arr, la]
        if replay_pivots is not None:
            fp = [int(i) for blk in replay_pivots for i in blk]
            pa = (ctypes.c_int32 * max(1, len(fp)))(*fp)
            p.replay_pivots = ctypes.cast(pa, ctypes.POINTER(ctypes.c_int32))
            keep.append(pa)
    ws_bytes = 0
    for x in shards:
        q = _problem(x, tol, k, b, seed, k_max, tau_b, flags, n_global, 0, False)
        sz = ctypes.c_size_t()
        rc = L.rbrp_workspace_size(ctypes.byref(q), ctypes.byref(sz))
        if rc:
            raise RBRPError(rc, "workspace_size")
        ws_bytes = max(ws_bytes, sz.value)
    wss = [torch.empty(ws_bytes, dtype=torch.uint8, device=x.device) for x in shards]
    k_cap = p.k_max if p.k_max > 0 else min(p.n_global, p.d)
    Ws = [torch.empty((x.shape[0], k_cap), dtype=x.dtype, device=x.device) for x in shards] if with_W else None
    S = torch.empty(k_cap, dtype=torch.int64)
    rows = (ctypes.c_int64 * len(shards))(*[int(x.shape[0]) for x in shards])
    Xp = (ctypes.c_void_p * len(shards))(*[x.data_ptr() for x in shards])
    Wp = (ctypes.c_void_p * len(shards))(*[w.data_ptr() for w in Ws]) if Ws else None
    Sp = (ctypes.c_void_p * len(shards))(*[w.data_ptr() for w in wss])
    rep, b_t, b_pr, rho, bidx, bpiv = _report(max_blocks, b, True)
    stream = torch.cuda.current_stream(X0.device).cuda_stream
    rc = L.rbrp_id_sharded(ctypes.byref(p), len(shards), rows, Xp, Sp, ws_bytes, ctypes.c_void_p(stream),
                           ctypes.cast(S.data_ptr(), ctypes.POINTER(ctypes.c_int64)), Wp, ctypes.byref(rep))
    if rc:
        raise RBRPError(rc, L.rbrp_strerror(rc).decode())
    res = _result(rep, S, None, b_t, b_pr, rho, bidx, bpiv, max_blocks, b, True)
    Wk = [w[:, :res.k] for w in Ws] if Ws else None
    return res, Wk


def form_w(L: torch.Tensor, S: Sequence[int], method: str = "auto", W_out: Optional[torch.Tensor] = None):
    """Alg. 3 on its own: W(S,:) = I, W(rest,:) = L_2 L_1^{-1} from a device L
    (n x k, row-major) and the skeleton rows S.  method: "auto" (triangular solve unless
    min |diag L_1| < 1e-12 max |diag L_1|, then the clipped SVD of Remark 5.2), "trsm", or
    "pinv" (clipped SVD, singular values < 1e-12 sigma_max discarded).
    Returns (W (n x k device), flags, number of discarded singular values)."""
    if not L.is_cuda or L.dim() != 2 or L.stride(1) != 1 or L.dtype not in (torch.float32, torch.float64):
        raise ValueError("L must be a row-major float32/float64 CUDA matrix")
    Lb = lib()
    n, k = L.shape
    dt = RBRP_F64 if L.dtype == torch.float64 else RBRP_F32
    meth = {"auto": 0, "trsm": 1, "pinv": 2}[method]
    sz = ctypes.c_size_t()
    rc = Lb.rbrp_form_w_workspace_size(dt, k, ctypes.byref(sz))
    if rc:
        raise RBRPError(rc, "form_w_workspace_size")
    ws = torch.empty(sz.value, dtype=torch.uint8, device=L.device)
    W = W_out if W_out is not None else torch.empty((n, k), dtype=L.dtype, device=L.device)
    Sa = (ctypes.c_int64 * len(S))(*[int(i) for i in S])
    fl = ctypes.c_uint32()
    nc = ctypes.c_int32()
    stream = torch.cuda.current_stream(L.device).cuda_stream
    rc = Lb.rbrp_form_w(dt, ctypes.c_void_p(L.data_ptr()), L.stride(0), n, Sa, len(S), meth,
                        ctypes.c_void_p(W.data_ptr()), W.stride(0), ctypes.c_void_p(ws.data_ptr()), sz.value,
                        ctypes.c_void_p(stream), ctypes.byref(fl), ctypes.byref(nc))
    if rc:
        raise RBRPError(rc, Lb.rbrp_strerror(rc).decode())
    return W, fl.value, nc.value


def id_host(X_host: torch.Tensor, tol: Optional[float] = None, k: Optional[int] = None, b: int = 16,
            seed: int = 0, k_max: int = 0, tau_b: float = -1.0, with_W: bool = True, greedy: bool = False,
            form: str = "residual", device="cuda", workspace: Optional[torch.Tensor] = None,
            W_host: Optional[torch.Tensor] = None, comm=None, n_global: Optional[int] = None,
            row_offset: int = 0, max_blocks: int = 1024):
    """End-to-end entry with HOST buffers through the C ABI (rbrp_id_host): the library
    copies X_host (n x d, row-major; pinned memory for full PCIe bandwidth) into a private
    device copy inside `workspace`, runs the ID on it in place, and copies W (first k
    columns) back into W_host (n x k_cap, pinned, allocated if None).
    Returns (Result with W = the n x k host view, W_host)."""
    if X_host.is_cuda:
        raise ValueError("X_host must be a host tensor (use id for device tensors)")
    if tol is None and k is None:
        raise ValueError("need tol or k")
    L = lib()
    dev = torch.device(device)
    flags = (0 if with_W else RBRP_NO_W) | (RBRP_FORM_PAPER if form == "paper" else 0)
    p = _problem(X_host, tol, k, b, seed, k_max, tau_b, flags, n_global, row_offset, greedy)
    sz = ctypes.c_size_t()
    rc = L.rbrp_workspace_size_host(ctypes.byref(p), ctypes.byref(sz))
    if rc:
        raise RBRPError(rc, "workspace_size_host")
    if workspace is None or workspace.numel() < sz.value:
        workspace = torch.empty(sz.value, dtype=torch.uint8, device=dev)
    k_cap = p.k_max if p.k_max > 0 else min(p.n_global, p.d)
    if with_W and W_host is None:
        W_host = torch.empty((X_host.shape[0], k_cap), dtype=X_host.dtype, pin_memory=True)
    rep, b_t, b_pr, rho, bidx, bpiv = _report(max_blocks, b, False)
    S = torch.empty(k_cap, dtype=torch.int64)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = L.rbrp_id_host(ctypes.byref(p), ctypes.c_void_p(X_host.data_ptr()), ctypes.c_void_p(workspace.data_ptr()),
                        sz.value, ctypes.c_void_p(comm) if comm else None, ctypes.c_void_p(stream),
                        ctypes.cast(S.data_ptr(), ctypes.POINTER(ctypes.c_int64)),
                        ctypes.c_void_p(W_host.data_ptr()) if with_W else None, ctypes.byref(rep))
    if rc:
        raise RBRPError(rc, L.rbrp_strerror(rc).decode())
    res = _result(rep, S, None, b_t, b_pr, rho, None, None, max_blocks, b, False)
    if with_W:
        res.W = W_host[:, :res.k]
    return res, W_host
