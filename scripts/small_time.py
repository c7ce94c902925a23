"""Device time per ID (graph loop, CUDA events inside the call: r.ms) of the small configs
c1 / c2 after warm-up, median of REPS calls; the verdict's latency targets (c1 <= 0.2 ms,
c2 <= 1.9 ms) are on this number.  CFGS=c1,c2 REPS=20."""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import CONFIGS, make  # noqa: E402

for name in os.environ.get("CFGS", "c1,c2").split(","):
    cfg = CONFIGS[name]
    X0 = make(cfg, device="cuda")
    tau = bench._tau(cfg, X0)
    km = bench.K_MAX.get(cfg.name, 0)
    ms = []
    for i in range(3 + int(os.environ.get("REPS", "20"))):
        X = X0.clone()
        r = rb.id(X, tol=tau, b=cfg.b, seed=0, k_max=km or 0)
        torch.cuda.synchronize()
        if i >= 3:
            ms.append(r.ms)
    print(f"{name}: k={r.k} b'={r.b_prime} graph={r.graph} device ms per ID: median {statistics.median(ms):.4f} "
          f"min {min(ms):.4f} max {max(ms):.4f}", flush=True)
