"""Cycle trace of k_proj_tc32 (CTA 0, tiles 0-1) on c4's first block.  Profiling tool:
RBRP_TC_TRACE=1 records the first launch of the process."""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ.setdefault("RBRP_TC_TRACE", "1")
os.environ["RBRP_NO_GRAPH"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import CONFIGS, make  # noqa: E402

cfg = CONFIGS["c4"]
X = make(cfg, device="cuda")
r = rb.id(X, tol=cfg.tau, b=cfg.b, seed=0)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (9 * 2 * 128))()
n = rb.lib().rbrp_debug_tc_trace(buf, 9 * 2 * 128)
t = np.array(buf[:], dtype=np.int64).reshape(9, 2, 128)
t0 = t[t > 0].min()
nc = 64
names = ["mma_ready", "mma_issued", "rw_xfull", "rw_aempty", "rw_afull", "rw_a2full", "rw_xfull2", "rw_stored", "xprod"]
for p in range(2):
    print("tile", p)
    for s in list(range(0, 8)) + list(range(56, 72)) + list(range(120, 128)):
        row = []
        for e in range(9):
            idx = s if e in (0, 1, 8) else (s if s < nc else s - nc)
            if e in (2, 3, 4) and s >= nc:
                row.append("      -")
                continue
            if e in (5, 6, 7) and s < nc:
                row.append("      -")
                continue
            v = t[e, p, idx]
            row.append(f"{(v - t0) if v else -1:7d}")
        print(f" s{s:3d} " + " ".join(row))
print("cols:", names)
# per-step intervals over tile 1 (steady state): median cycles between consecutive steps
for e, nm in enumerate(names):
    rng = range(0, 2 * nc) if e in (0, 1, 8) else range(0, nc)
    v = np.array([t[e, 1, i] for i in rng if i < 128])
    v = v[v > 0]
    if len(v) > 2:
        dv = np.diff(v)
        print(f"{nm:12s} median step {int(np.median(dv)):6d} cyc  mean {int(dv.mean()):6d}  (n={len(dv)})")
# tile 1 length and phases
p1 = t[2, 1, 0], t[4, 1, nc - 1], t[5, 1, 0], t[7, 1, nc - 1]
print("tile1 pass1 start->end", p1[1] - p1[0], " pass1 end->pass2 first a2full", p1[2] - p1[1],
      " pass2", p1[3] - p1[2], " total", p1[3] - p1[0])
print("k", r.k, r.b_prime, r.proj_ms_blk)
