"""Repeat tests/test_gpu_parity.py::test_sharded_sampling_with_small_support_and_nan's first
half many times (it failed once with a duplicate skeleton row)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import make, small_config  # noqa: E402

dev = torch.device("cuda")
bad = 0
for it in range(int(os.environ.get("ITERS", "200"))):
    torch.manual_seed(it)
    if it % 3 == 0:   # something else in between (other kernels, other graph keys)
        cfg = small_config("c2", n=7001, d=512, rank=100, b=64)
        X = make(cfg, device="cuda")
        rb.id(X, tol=1e-12, b=64, seed=it)
    Z = torch.zeros(2 * 4096 + 10, 12, dtype=torch.float64, device=dev)
    Z[[5, 4100, 8195]] = torch.randn(3, 12, dtype=torch.float64, device=dev)
    res, _ = rb.rbrp.id_sharded([Z[:4096], Z[4096:8192], Z[8192:]], tol=1e-14, b=8, seed=it)
    S = sorted(res.S.tolist())
    if S != [5, 4100, 8195]:
        bad += 1
        print("iter", it, "S", res.S.tolist(), "b'", res.b_prime, "rho", res.rho, "flags", getattr(res, "flags", None),
              flush=True)
print("bad", bad)
