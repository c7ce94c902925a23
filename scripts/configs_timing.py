"""Time-to-ID of every BASELINE.json config at full size on one GPU (both forms of Alg. 2),
with the projection's achieved FP64 TFLOP/s.  Writes one JSON line per (config, form).

    python scripts/configs_timing.py [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import CONFIGS, make  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
a = ap.parse_args()


def gram_tau(cfg, X, chunk=1 << 18):
    G = torch.zeros((X.shape[1],) * 2, dtype=torch.float64, device=X.device)
    for s in range(0, X.shape[0], chunk):
        Xc = X[s:s + chunk].double()
        G += Xc.T @ Xc
    ev = torch.linalg.eigvalsh(G).flip(0).clamp_min(0)
    return float((1 + cfg.eps) * ev[cfg.r:].sum() / ev.sum())


for name in a.configs.split(","):
    cfg = CONFIGS[name]
    X = make(cfg, device="cuda")
    tau = cfg.tau if cfg.tau is not None else gram_tau(cfg, X)
    kmax = 768 if name == "c5" else 0
    for form in ("residual", "paper"):
        kw = dict(tol=tau, b=cfg.b, seed=0, k_max=kmax, form=form, log_blocks=False,
                  inplace=False)
        if name == "c5" and form == "residual":
            kw["inplace"] = False   # X 34 GB + X_res 34 GB + L and W (k_max 768) 52 GB: fits
        try:
            rb.id(X, **kw)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rs = []
            for _ in range(a.reps):
                r = rb.id(X, **kw)
                r.W = None
                rs.append(r)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            w = 8 if cfg.dtype == "f64" else 4
            fl = 0.0
            for r in rs:
                for bp in r.b_prime:
                    fl += (4.0 if form == "residual" else 2.0) * cfg.n * cfg.d * bp
            pm = sum(r.proj_ms for r in rs)
            print(json.dumps({"config": name, "form": form, "n": cfg.n, "d": cfg.d, "dtype": cfg.dtype,
                              "b": cfg.b, "tau": tau, "k": rs[-1].k, "blocks": rs[-1].nblocks,
                              "b_prime": rs[-1].b_prime, "resid_rel": rs[-1].resid_rel,
                              "ms_per_id": ms, "proj_ms_per_id": pm / a.reps,
                              "proj_tflops": fl / (pm / 1e3) / 1e12 if pm > 0 else None}), flush=True)
        except Exception as ex:   # noqa: BLE001
            print(json.dumps({"config": name, "form": form, "error": str(ex)[:200]}), flush=True)
    del X
    torch.cuda.empty_cache()
