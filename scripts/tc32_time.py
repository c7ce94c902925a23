"""Time one k_proj_tc32 projection (rbrp_debug_tc32) at c4's shape for several b' (the kernel in
isolation, CUDA events, 3 repeats).  Development tool."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_16002_b200 as rb  # noqa: E402

f = rb.lib().rbrp_debug_tc32
f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
              ctypes.c_void_p]
n, d = 1 << 20, 2048
X = torch.randn(n, d, device="cuda")
for b in [int(x) for x in os.environ.get("BS", "4,27,57,64").split(",")]:
    Q = torch.linalg.qr(torch.randn(d, b, device="cuda", dtype=torch.float64))[0].T.contiguous().float()
    L = torch.empty(n, b, device="cuda")
    dv = torch.empty(n, dtype=torch.float64, device="cuda")
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f(X.data_ptr(), n, d, Q.data_ptr(), b, L.data_ptr(), dv.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"b'={b}: {min(ts):.3f} ms  ({2 * n * d * 4 / min(ts) / 1e9:.0f} GB/s algorithmic)", flush=True)
