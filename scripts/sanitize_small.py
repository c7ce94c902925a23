"""Small end-to-end workload for compute-sanitizer (one tool per run): every kernel family
of the library on c1-size inputs -- graph and eager block loops (residual and paper forms,
fp64 and fp32 incl. the tcgen05 projection), RBGP, the sharded emulation, the Remark 5.2
W fallback, SkLUPP-OSID."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import make, small_config  # noqa: E402


def main():
    dev = torch.device("cuda")
    cfg = small_config("c2", n=9000, d=256, rank=40, b=16)
    X = make(cfg, device=dev)
    r = rb.id(X, tol=1e-12, b=16, seed=1)                       # graph loop, residual form
    p = rb.id(X, tol=1e-12, b=16, seed=1, form="paper")         # paper form
    os.environ["RBRP_NO_GRAPH"] = "1"
    e = rb.id(X, tol=1e-12, b=32, seed=2)                       # eager loop, tiled DMMA
    os.environ.pop("RBRP_NO_GRAPH")
    g = rb.id(X, tol=1e-12, b=16, greedy=True)                  # RBGP (k_topb)
    c5 = small_config("c5", n=12000, d=160, n_centres=120, b=64)
    Y = make(c5, device=dev)
    q = rb.id(Y, k=100, b=64, seed=0)                           # b' > 32 parts, 64 < b filter
    f32 = small_config("c4", n=9000, d=192, b=64)
    Z = make(f32, device=dev)
    z = rb.id(Z, tol=1e-3, b=64, seed=0)                        # fp32: tcgen05 projection
    sh, _ = rb.rbrp.id_sharded([X[:4096], X[4096:]], tol=1e-12, b=16, seed=1)
    rng = np.random.default_rng(2)
    L = rng.standard_normal((3000, 64))
    S = list(range(0, 3000, 47))[:64]
    L1 = np.eye(64) + np.tril(rng.standard_normal((64, 64)), -1) * 0.03
    L1[20, 20] = 1e-14
    L[S] = L1
    W, fl, nc = rb.rbrp.form_w(torch.from_numpy(L).to(dev), S, method="auto")   # clipped-SVD W
    sk = rb.sketch_id(X, 24, 72, seed=0)                        # SkLUPP-OSID
    torch.cuda.synchronize()
    print("ok", r.k, p.k, e.k, g.k, q.k, z.k, sh.k, fl, nc, sk.k)


if __name__ == "__main__":
    main()
