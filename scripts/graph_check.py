import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_16002_b200 as rb
from workloads import CONFIGS, make
cfg = CONFIGS["c2"]
X = make(cfg, device="cuda")
ws = torch.empty(rb.workspace_size(X, tol=1e-12, b=32), dtype=torch.uint8, device="cuda")
for mode in ["graph", "eager", "graph"]:
    if mode == "eager": os.environ["RBRP_NO_GRAPH"] = "1"
    else: os.environ.pop("RBRP_NO_GRAPH", None)
    for i in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = rb.id(X, tol=1e-12, b=32, seed=0, workspace=ws, log_blocks=False)
        torch.cuda.synchronize()
        print(mode, i, f"wall {1e3*(time.perf_counter()-t):.2f} ms  lib {r.ms:.2f} ms  proj {r.proj_ms:.2f} graph={r.graph} k={r.k} blocks={r.nblocks}", flush=True)
