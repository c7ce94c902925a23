"""One or more IDs of a BASELINE config for profiling (eager block loop so ncu sees every
kernel).  CFG=c5|c4|c3|c2, REPS=n.  tau as bench.py (Gram spectrum for (r, eps) configs)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RBRP_NO_GRAPH", "1")
import bench  # noqa: E402
import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import CONFIGS, make  # noqa: E402

cfg = CONFIGS[os.environ.get("CFG", "c5")]
X = make(cfg, device="cuda")
tau = bench._tau(cfg, X)
km = bench.K_MAX.get(cfg.name, 0)
for i in range(int(os.environ.get("REPS", "1"))):
    r = rb.id(X, tol=tau, b=cfg.b, seed=0, k_max=km or 0)
    torch.cuda.synchronize()
    print(cfg.name, i, r.k, r.b_prime, f"{r.ms:.3f} ms", [round(x, 3) for x in r.proj_ms_blk], flush=True)
