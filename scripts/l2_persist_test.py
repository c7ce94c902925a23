"""Experiment: does an L2 set-aside for persisting accesses (cudaLimitPersistingL2CacheSize)
change the tcgen05 projection's pass-2 re-read misses (the pass-1 loads carry an evict_last
policy)?  Runs c4 with the set-aside given in MB by PERSIST_MB (0 = default)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RBRP_NO_GRAPH", "1")
from cuda import cudart  # noqa: E402

import bench  # noqa: E402
import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import CONFIGS, make  # noqa: E402

torch.cuda.init()
mb = int(os.environ.get("PERSIST_MB", "-1"))
err, prop = cudart.cudaGetDeviceProperties(0)
print("persistingL2CacheMaxSize MB", prop.persistingL2CacheMaxSize / 2**20, "l2 MB", prop.l2CacheSize / 2**20)
if mb >= 0:
    print(cudart.cudaDeviceSetLimit(cudart.cudaLimit.cudaLimitPersistingL2CacheSize, mb << 20))
err, v = cudart.cudaDeviceGetLimit(cudart.cudaLimit.cudaLimitPersistingL2CacheSize)
print("limit MB", v / 2**20)
cfg = CONFIGS["c4"]
X = make(cfg, device="cuda")
tau = bench._tau(cfg, X)
for i in range(3):
    r = rb.id(X, tol=tau, b=cfg.b, seed=0)
    torch.cuda.synchronize()
    print(i, r.k, r.b_prime, f"{r.ms:.3f} ms", [round(x, 3) for x in r.proj_ms_blk], flush=True)
