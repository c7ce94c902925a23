"""Structured probe of k_proj_tc32: X[i,k] = i + k/256, Q = unit rows -> L-hat[i,j] should be
X[i, c_j].  Prints the decoded (row, col) each L-hat entry came from.  Development tool."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_16002_b200 as rb  # noqa: E402

f = rb.lib().rbrp_debug_tc32
f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
              ctypes.c_void_p]
n, d, b = 128, 32, 16
X = (np.arange(n)[:, None] + np.arange(d)[None, :] / 256.0).astype(np.float32)
for cols in ([0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15], [16, 17, 18, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31]):
    Q = np.zeros((b, d), np.float32)
    for j, c in enumerate(cols):
        Q[j, c] = 1.0
    Xd = torch.from_numpy(X.copy()).cuda()
    Ld = torch.zeros((n, b), dtype=torch.float32, device="cuda")
    dv = torch.zeros((n,), dtype=torch.float64, device="cuda")
    f(Xd.data_ptr(), n, d, torch.from_numpy(Q).cuda().data_ptr(), b, Ld.data_ptr(), dv.data_ptr())
    Lg = Ld.cpu().numpy()
    print("cols", cols[0], "..")
    for i in [0, 1, 2, 7, 8, 9, 31, 32, 64, 127]:
        dec = [(int(np.floor(v)), int(round((v - np.floor(v)) * 256))) if abs(v) > 0 else None for v in Lg[i]]
        print(" row", i, dec)
    Xg = Xd.cpu().numpy()
    print(" X out row 5", np.round(Xg[5, :20], 4))
