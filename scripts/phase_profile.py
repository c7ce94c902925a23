import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2309_16002_b200 as rb
from workloads import CONFIGS, make
cfg = CONFIGS["c2"]; X = make(cfg, device="cuda")
for form in ("residual", "paper"):
    for _ in range(2): rb.id(X, tol=1e-12, b=32, seed=0, form=form)
    r = rb.id(X, tol=1e-12, b=32, seed=0, form=form, profile=True)
    print(form, r.ms, {k: round(v, 3) for k, v in r.ms_phase.items()})
