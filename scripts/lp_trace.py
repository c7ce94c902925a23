"""Cycle trace of the 64-row-tile projection (k_lhat_paper, residual form) on CTA 0
(RBRP_LP_TRACE=1 RBRP_NO_GRAPH=1): per tile, where the consumer warps spend their cycles."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RBRP_LP_TRACE"] = "1"
os.environ["RBRP_NO_GRAPH"] = "1"
import numpy as np
import paper_2309_16002_b200 as rb
from workloads import CONFIGS, make
X = make(CONFIGS["c2"], device="cuda")
rb.id(X, tol=1e-12, b=32, seed=0)   # trace: first bucket-32 launch (block 1)
buf = (ctypes.c_longlong * 5120)()
rb.lib().rbrp_debug_lp_trace(buf, 5120)
a = np.frombuffer(buf, dtype=np.int64).astype(np.float64)
ev = a[:1024].reshape(16, 8, 8)
st = a[1024:].reshape(16, 256)
t0 = ev[ev > 0].min()
ev = np.where(ev > 0, ev - t0, np.nan)
st = np.where(st > 0, st - t0, np.nan)
names = ["start", "p1_end", "bar1", "bar2", "bcast", "p2_end", "nbar", "end"]
for p in range(8):
    if np.all(np.isnan(ev[:, p, 0])):
        break
    e = ev[:, p, :]
    print(f"tile {p}: " + "  ".join(f"{n}={np.nanmin(e[:, i]):.0f}..{np.nanmax(e[:, i]):.0f}" for i, n in enumerate(names)))
dur = np.nanmax(ev[:, :, 7], axis=0) - np.nanmin(ev[:, :, 0], axis=0)
print("tile durations", dur[~np.isnan(dur)])
seg = lambda i, j: np.nanmedian(ev[:, 1:6, j] - ev[:, 1:6, i])
print("median per warp: p1 %.0f  p1_end->bar1 %.0f  bar1->bar2 %.0f  bar2->bcast %.0f  bcast->p2_end %.0f  p2_end->nbar %.0f  nbar->end %.0f  end->next start"
      % (seg(0, 1), seg(1, 2), seg(2, 3), seg(3, 4), seg(4, 5), seg(5, 6), seg(6, 7)))
ds = np.diff(st[:, :224], axis=1)
print("step period median (all warps) %.0f, p10 %.0f p90 %.0f" % (np.nanmedian(ds), np.nanpercentile(ds, 10), np.nanpercentile(ds, 90)))
sk = np.nanmax(st[:, :224], axis=0) - np.nanmin(st[:, :224], axis=0)
print("warp skew per step median %.0f max %.0f" % (np.nanmedian(sk), np.nanmax(sk)))
for s in range(0, 64):
    print(s, " ".join(f"{v:7.0f}" for v in st[::3, s]))
