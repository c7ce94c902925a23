import sys, os; sys.path.insert(0, ".")
import torch, paper_2309_16002_b200 as rb
from workloads import CONFIGS, make
X = make(CONFIGS["c2"], device="cuda")
for _ in range(3): r = rb.id(X, tol=1e-12, b=32, seed=0, log_blocks=False)
import statistics
blk = [[] for _ in range(5)]; ms = []
for _ in range(10):
    r = rb.id(X, tol=1e-12, b=32, seed=0, log_blocks=False)
    ms.append(r.ms)
    for i, v in enumerate(r.proj_ms_blk[:5]): blk[i].append(v)
print(os.environ.get("RBRP_LP_NS", "default"), round(statistics.median(ms), 3), [round(statistics.median(b), 4) for b in blk], r.b_prime)
