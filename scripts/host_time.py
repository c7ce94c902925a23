"""Host-side cost of one rb.id call at a config (RBRP_HOST_TIMING marks of the C ABI, plus the
Python wall time per call against the device time r.ms), graph loop, after warm-up.
CFG=c2 REPS=10."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import CONFIGS, make  # noqa: E402

cfg = CONFIGS[os.environ.get("CFG", "c2")]
X = make(cfg, device="cuda")
tau = bench._tau(cfg, X)
km = bench.K_MAX.get(cfg.name, 0)
ws = torch.empty(rb.workspace_size(X, tol=tau, b=cfg.b, k_max=km or 0), dtype=torch.uint8, device="cuda")
k_cap = km or min(cfg.n, cfg.d)
Wb = torch.empty((cfg.n, k_cap), dtype=cfg.torch_dtype, device="cuda")
kw = dict(tol=tau, b=cfg.b, seed=0, k_max=km or 0, workspace=ws, log_blocks=False, W_out=Wb)
for _ in range(3):
    rb.id(X, **kw)
torch.cuda.synchronize()
n = int(os.environ.get("REPS", "10"))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
dev = []
for _ in range(n):
    r = rb.id(X, **kw)
    dev.append(r.ms)
e1.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / n * 1e3
print(f"{cfg.name}: stream time per ID {e0.elapsed_time(e1) / n:.4f} ms, wall {wall:.4f} ms, "
      f"device time inside the call {sum(dev) / n:.4f} ms", flush=True)
