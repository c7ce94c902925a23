"""Quick timing of one config: graph-mode time per ID, projection time and the eager
per-phase profile.   python scripts/quick.py [c2|c1|c3|...] [tau]"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_16002_b200 as rb
from workloads import CONFIGS, make
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = CONFIGS[name]
X = make(cfg, device="cuda")
tau = cfg.tau if cfg.tau is not None else float(sys.argv[2])
ws = torch.empty(rb.workspace_size(X, tol=tau, b=cfg.b), dtype=torch.uint8, device="cuda")
W = torch.empty((cfg.n, min(cfg.n, cfg.d)), dtype=X.dtype, device="cuda")
for i in range(5):
    r = rb.id(X, tol=tau, b=cfg.b, seed=0, workspace=ws, W_out=W, log_blocks=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); n = 10; pj = 0
for i in range(n):
    r = rb.id(X, tol=tau, b=cfg.b, seed=0, workspace=ws, W_out=W, log_blocks=False); pj += r.proj_ms
e1.record(); torch.cuda.synchronize()
print(f"{name}: {e0.elapsed_time(e1)/n:.3f} ms/ID  proj {pj/n:.3f} ms  k={r.k} blocks={r.nblocks} b'={r.b_prime} graph={r.graph}")
p = rb.id(X, tol=tau, b=cfg.b, seed=0, workspace=ws, W_out=W, log_blocks=False, profile=True)
print("eager phases:", {k: round(v, 3) for k, v in p.ms_phase.items()}, "sum", round(sum(p.ms_phase.values()), 3), "total", round(p.ms, 3))
