"""SkLUPP-OSID on c2 (65536 x 1024 fp64, k = 128, l = 3k = 384): time per
call and per phase, with the FP64 rate of the two GEMMs (Y = X Omega: 2 n d l flops;
W = Y M: 2 n l k flops).   python scripts/sketch_c2.py [--reps 10]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import CONFIGS, make  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--k", type=int, default=128)
a = ap.parse_args()
cfg = CONFIGS["c2"]
X = make(cfg, device="cuda")
k, l = a.k, 3 * a.k
for _ in range(2):
    rb.sketch_id(X, k, l, seed=1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    res = rb.sketch_id(X, k, l, seed=1)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
ph = rb.sketch_id(X, k, l, seed=1, profile=True).ms_phase
lp = (l + 7) // 8 * 8
print(json.dumps({"workload": "c2 65536 x 1024 f64", "method": "sklupp_osid", "k": k, "l": l, "ms": ms,
                  "ms_phase": ph, "sketch_tflops": 2 * cfg.n * cfg.d * lp / (ph["sketch"] * 1e9),
                  "lupp_ms": ph["lupp"], "launches": res.launches}))
