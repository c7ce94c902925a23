"""Probe k_proj_tc32 in isolation (rbrp_debug_tc32) against numpy fp64.  Development tool."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_16002_b200 as rb  # noqa: E402

L_ = rb.lib()
f = L_.rbrp_debug_tc32
f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
              ctypes.c_void_p]
for (n, d, b) in [(128, 32, 16), (256, 64, 16), (300, 96, 32), (1000, 256, 64), (5000, 2048, 64)]:
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, d)).astype(np.float32)
    Q = np.ascontiguousarray(np.linalg.qr(rng.standard_normal((d, b)))[0].T.astype(np.float32))
    Xd = torch.from_numpy(X).cuda()
    Qd = torch.from_numpy(Q).cuda()
    Ld = torch.full((n, b), float("nan"), dtype=torch.float32, device="cuda")
    dv = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    rc = f(Xd.data_ptr(), n, d, Qd.data_ptr(), b, Ld.data_ptr(), dv.data_ptr())
    X64, Q64 = X.astype(np.float64), Q.astype(np.float64)
    Lr = X64 @ Q64.T
    Xr = X64 - Lr @ Q64
    Lg = Ld.cpu().numpy().astype(np.float64)
    Xg = Xd.cpu().numpy().astype(np.float64)
    print((n, d, b), "rc", rc, "L err", np.nanmax(np.abs(Lg - Lr)) / np.abs(Lr).max(), "nan L", np.isnan(Lg).sum(),
          "X err", np.max(np.abs(Xg - Xr)) / np.abs(X64).max(),
          "d err", np.nanmax(np.abs(dv.cpu().numpy() - (Xg ** 2).sum(1)) / (X64 ** 2).sum(1)), flush=True)
    if n <= 300:
        print(" L row0", np.round(Lg[0, :8], 4), "ref", np.round(Lr[0, :8], 4))
        print(" L row1", np.round(Lg[1, :8], 4), "ref", np.round(Lr[1, :8], 4))
        print(" X row0", np.round(Xg[0, :8], 4), "ref", np.round(Xr[0, :8], 4))
