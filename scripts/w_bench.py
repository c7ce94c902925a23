"""Time Alg. 3 alone (rbrp_form_w, trsm): W = L_2 L_1^{-1} at the c5 / c3 / c2 shapes.
Reports ms and the triangular-GEMM rate n k^2 / t (the W GEMM skips L_1^{-T}'s zero chunks)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_16002_b200 as rb  # noqa: E402

shapes = [(4194304, 512), (131072, 240), (65536, 128)]
if os.environ.get("SHAPES"):
    shapes = [tuple(int(v) for v in s.split("x")) for s in os.environ["SHAPES"].split(",")]
for n, k in shapes:
    g = torch.Generator(device="cuda").manual_seed(0)
    L = torch.randn(n, k, dtype=torch.float64, device="cuda", generator=g)
    S = torch.randperm(n, device="cuda", generator=g)[:k].sort().values
    L1 = torch.eye(k, dtype=torch.float64, device="cuda") + 0.1 * torch.tril(
        torch.randn(k, k, dtype=torch.float64, device="cuda", generator=g), -1)
    L[S] = L1
    Sl = S.tolist()
    W = torch.empty_like(L)
    for _ in range(2):
        rb.rbrp.form_w(L, Sl, method="trsm", W_out=W)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        rb.rbrp.form_w(L, Sl, method="trsm", W_out=W)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"n={n} k={k}: {ms:.3f} ms  {n * k * k / ms / 1e9:.1f} TF (n k^2)", flush=True)
    del L, W
    torch.cuda.empty_cache()
