"""Cycle trace of the fused projection on CTA 0 (RBRP_FZ_TRACE=1 RBRP_NO_GRAPH=1).
Prints per-step producer issue times and consumer wait/finish times (in SM cycles)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RBRP_FZ_TRACE"] = "1"
os.environ["RBRP_NO_GRAPH"] = "1"
import numpy as np, torch
import paper_2309_16002_b200 as rb
from workloads import CONFIGS, make, small_config
D = int(os.environ.get("FZ_D", "1024"))
cfg = CONFIGS["c2"] if D == 1024 else small_config("c2", n=65536 * 1024 // D, d=D)
X = make(cfg, device="cuda")
res = rb.id(X, tol=1e-12, b=32, seed=0)   # trace: first bucket-32 launch (block 1)
L = rb.lib()
buf = (ctypes.c_longlong * (16 * 512))()
L.rbrp_debug_fz_trace(buf, 16 * 512)
a = np.frombuffer(buf, dtype=np.int64).reshape(16, 512).astype(np.float64)
t0 = a[a > 0].min()
a = np.where(a > 0, a - t0, np.nan)
names = ["x_issue", "q_issue", "p1_qfull", "p1_xfull", "p1_end", "p2_qfull", "p2_end", "p2_xfull", "p2_mmaiss", "p2_arrive", "p2_mmadone", "p1_mmaiss", "p1_mmadone"]
print("step " + " ".join(f"{n:>9s}" for n in names))
for s in range(0, 160):
    print(f"{s:4d} " + " ".join(f"{v:9.0f}" for v in a[:13, s]))
d = np.diff(a[4, 20:140]); print("p1 step period (cyc) median", np.nanmedian(d))
d = np.diff(a[6, 20:140]); print("p2 step period (cyc) median", np.nanmedian(d))
print("q latency issue->p1_qfull median", np.nanmedian(a[2, 20:140] - a[1, 20:140]))
print("x latency issue->p1_xfull median", np.nanmedian(a[3, 20:140] - a[0, 20:140]))

def med(i, j): return np.nanmedian(a[j, 20:140] - a[i, 20:140])
print("P2: qfull->xfull %.0f  xfull->mma_issued %.0f  ->arrive %.0f  ->mma_done %.0f  ->end %.0f" % (med(5,7), med(7,8), med(8,9), med(9,10), med(10,6)))
print("P1: qfull->xfull %.0f  xfull->mma_issued %.0f  ->mma_done %.0f  ->end %.0f" % (med(2,3), med(3,11), med(11,12), med(12,4)))
