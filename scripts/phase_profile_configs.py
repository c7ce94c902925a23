import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, paper_2309_16002_b200 as rb
from workloads import CONFIGS, make
for name in sys.argv[1].split(","):
    cfg = CONFIGS[name]; X = make(cfg, device="cuda")
    tau = cfg.tau if cfg.tau is not None else {"c5": 0.0020709267553592823, "c3": 5.272668127303654e-08}[name]
    for form in ("residual", "paper"):
        kw = dict(tol=tau, b=cfg.b, seed=0, k_max=768 if name == "c5" else 0, form=form)
        rb.id(X, **kw)
        r = rb.id(X, profile=True, **kw)
        print(name, form, round(r.ms, 2), {k: round(v, 2) for k, v in r.ms_phase.items() if k != "unused"}, flush=True)
    del X; torch.cuda.empty_cache()
