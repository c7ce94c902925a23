"""One (or a few) RBRP IDs of a config, for ncu / compute-sanitizer runs.

    python scripts/prof_one.py [--config c2] [--reps 1] [--warm 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import CONFIGS, make, small_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--warm", type=int, default=1)
ap.add_argument("--small", action="store_true")
a = ap.parse_args()
cfg = CONFIGS[a.config] if not a.small else small_config(a.config, n=20000)
X = make(cfg, device="cuda")
tau = cfg.tau if cfg.tau is not None else 1e-3
for i in range(a.warm + a.reps):
    res = rb.id(X, tol=tau, b=cfg.b, seed=0)
torch.cuda.synchronize()
print(f"k={res.k} blocks={res.nblocks} b'={res.b_prime} ms={res.ms:.3f}")
