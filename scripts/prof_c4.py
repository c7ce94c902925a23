"""c4 IDs for profiling (eager block loop so ncu sees every kernel): 2 IDs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RBRP_NO_GRAPH", "1")
import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import CONFIGS, make  # noqa: E402

cfg = CONFIGS[os.environ.get("CFG", "c4")]
X = make(cfg, device="cuda")
for i in range(int(os.environ.get("REPS", "2"))):
    r = rb.id(X, tol=cfg.tau if cfg.tau else 1e-3, b=cfg.b, seed=0)
    torch.cuda.synchronize()
    print(i, r.k, r.b_prime, r.ms, [round(x, 3) for x in r.proj_ms_blk], flush=True)
