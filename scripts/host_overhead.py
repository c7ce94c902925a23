"""Host-side overhead of one rbrp_id call on c2: device time inside the call (its own
events) vs the device time per call of back-to-back calls (bench.py's timing), plus a
cProfile of the Python side.   python scripts/host_overhead.py"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import CONFIGS, make  # noqa: E402

X = make(CONFIGS["c2"], device="cuda")
ws = torch.empty(rb.workspace_size(X, tol=1e-12, b=32), dtype=torch.uint8, device="cuda")
W = torch.empty((X.shape[0], 1024), dtype=torch.float64, device="cuda")
kw = dict(tol=1e-12, b=32, seed=0, workspace=ws, log_blocks=False, W_out=W)
for _ in range(5):
    rb.id(X, **kw)
torch.cuda.synchronize()
K = 50
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
inner = 0.0
t0 = time.perf_counter()
e0.record()
for _ in range(K):
    r = rb.id(X, **kw)
    inner += r.ms
e1.record()
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"per call: device {e0.elapsed_time(e1) / K:.4f} ms, inside the call {inner / K:.4f} ms, "
      f"wall {(t1 - t0) / K * 1e3:.4f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    rb.id(X, **kw)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
