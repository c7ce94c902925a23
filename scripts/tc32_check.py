"""Quick check of the tcgen05 fp32 projection (k_proj_tc32) against the fp64-DMMA fp32 path
(RBRP_FP32_DMMA=1) and the oracle, then c4 timings of both.  Development tool."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_16002_b200 as rb  # noqa: E402
from oracle import rbrp as O  # noqa: E402
from workloads import CONFIGS, make, small_config  # noqa: E402


def run(X, env, **kw):
    os.environ["RBRP_FP32_DMMA"] = env
    r = rb.id(X, **kw)
    torch.cuda.synchronize()
    return r


def main():
    for (n, d, b) in ([] if os.environ.get("TC_TIME_ONLY") else [(20000, 192, 64), (3000, 64, 16), (9001, 100, 40), (12345, 2048, 64)]):
        cfg = small_config("c4", n=n, d=d, b=b)
        Xnp = make(cfg).numpy()
        ores = O.rbrp(Xnp, tau=1e-3, b=b, seed=0)
        X = torch.from_numpy(Xnp).cuda()
        blocks = [blk.S_t for blk in ores.blocks]
        piv = [blk.piv for blk in ores.blocks]
        out = {}
        for env in ("1", "0"):
            r = run(X, env, k=ores.k, b=b, replay_blocks=blocks, replay_pivots=piv, return_d=True)
            print(env, "k", r.k, ores.k, "bp", r.b_prime, [x.b_prime for x in ores.blocks], "flags", r.flags,
                  "rho", r.rho, [x.rho for x in ores.blocks], flush=True)
            if r.k != ores.k:
                continue
            Wo, kap, _ = O.form_W(ores.L, ores.S, method="trsm")
            W = r.W.double().cpu().numpy()
            out[env] = dict(S=r.S.tolist() == ores.S, bp=r.b_prime == [x.b_prime for x in ores.blocks],
                            drho=max(abs(a - x.rho) for a, x in zip(r.rho, ores.blocks)),
                            dW=float(np.max(np.abs(W - Wo)) / max(1.0, np.max(np.abs(Wo)))),
                            dd=float(np.max(np.abs(r.d.cpu().numpy() - ores.d) / (O.row_sq_norms(Xnp) + 1e-300))))
        print("replay", (n, d, b), out, flush=True)
    cfg = CONFIGS["c4"]
    X = make(cfg, device="cuda")
    for env in ("1", "0", "1", "0"):
        os.environ["RBRP_FP32_DMMA"] = env
        r = rb.id(X, tol=cfg.tau, b=cfg.b, seed=0)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            r = rb.id(X, tol=cfg.tau, b=cfg.b, seed=0, log_blocks=False)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 5
        print("c4", "dmma" if env == "1" else "tc32", f"{dt*1e3:.2f} ms", r.k, r.b_prime, f"{r.resid_rel:.6e}",
              "proj_ms_blk", [round(x, 3) for x in r.proj_ms_blk], flush=True)


if __name__ == "__main__":
    main()
