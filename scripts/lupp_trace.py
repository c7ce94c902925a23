"""LUPP phase cycles of CTA 0 (debug library built with -DLU_TRACE) on the Table 3 sketch
Y = X Omega (1e5 x 3k):  RBRP_LIB_PATH=build/lutrace/librbrp.so python scripts/lupp_trace.py
Phases: subst (U rows of earlier pivots), rows (own rows, panel columns), scan (local
argmax), gsync (grid barrier per step), winner, update (multipliers + panel update),
panel (grid barrier per panel)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_16002_b200 as rb  # noqa: E402
from paper_2309_16002_b200 import sketch as sk  # noqa: E402
from workloads import CONFIGS, make  # noqa: E402

L = sk.lib()
tr = (ctypes.c_longlong * 8)()
names = ["subst", "rows", "scan", "gsync", "winner", "update", "panel"]
cfg = CONFIGS["t3"]
X = make(cfg, device="cuda")
for k in [int(v) for v in (sys.argv[1:] or ["157", "472"])]:
    l = 3 * k
    OmT = sk.gaussian_embedding(cfg.d, l, seed=0)
    Y = X @ OmT.T
    sk.lupp(Y, k)
    L.rbrp_debug_lu_trace(tr, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sk.lupp(Y, k)
    e1.record()
    torch.cuda.synchronize()
    L.rbrp_debug_lu_trace(tr, 1)
    tot = sum(tr[:7])
    print(f"k={k} ms={e0.elapsed_time(e1):.2f} cycles={tot} " +
          " ".join(f"{n}={tr[i]} ({100 * tr[i] / max(tot, 1):.0f}%)" for i, n in enumerate(names)))
