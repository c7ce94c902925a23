"""fp32 projection efficiency vs the row-tile working set: the same bytes of X with d = 1024
(512 KB per 128-row tile, 76 MB over 148 SMs: fits the 126 MB L2 between the two passes)
and d = 2048 (1 MB tiles, 148 MB: does not).  Prints per-block projection time and the
achieved X_res read+write rate (2 n d 4 bytes per block)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_16002_b200 as rb  # noqa: E402

for n, d in ((1 << 20, 2048), (1 << 21, 1024), (1 << 22, 512)):
    g = torch.Generator(device="cuda").manual_seed(0)
    r = 96
    A = torch.randn(n, r, device="cuda", generator=g) * (torch.arange(1, r + 1, device="cuda") ** -1.0)
    B = torch.randn(r, d, device="cuda", generator=g)
    X = (A @ B).contiguous()
    X += 1e-4 * torch.randn(n, d, device="cuda", generator=g)
    for rep in range(2):
        res = rb.id(X, k=96, b=64, seed=0)
        torch.cuda.synchronize()
    gbs = [2 * n * d * 4 / (t * 1e-3) / 1e9 for t in res.proj_ms_blk]
    print(f"n={n} d={d}: b'={res.b_prime} ms={[round(t, 3) for t in res.proj_ms_blk]} GB/s={[round(x) for x in gbs]}",
          flush=True)
    del X, A, B
    torch.cuda.empty_cache()
