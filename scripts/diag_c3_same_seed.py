import os, sys
sys.path.insert(0, "/root/repo")
os.chdir(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_2309_16002_b200 as rb
from oracle import rbrp as O
from oracle import referee as R
from workloads import make, small_config
cfg = small_config("c3", n=5 * 4096 + 300, d=128, n_heavy_dirs=30, n_heavy_rows=9000, b=32)
Xnp = make(cfg).numpy()
tau = (1 + cfg.eps) * R.eta(np.asarray(Xnp, np.float64), min(cfg.r, Xnp.shape[1] // 4))
print("tau", tau)
Xd = torch.from_numpy(Xnp).cuda()
for seed in range(10):
    ores = O.rbrp(Xnp, tau=tau, b=cfg.b, seed=seed)
    res = rb.id(Xd, tol=tau, b=cfg.b, seed=seed)
    ob = [blk.b_prime for blk in ores.blocks]
    print("seed", seed, "k", res.k, ores.k, "bp gpu", res.b_prime, "orc", ob)
    o = 0
    for t, blk in enumerate(ores.blocks):
        if t >= len(res.blocks): print("  gpu has fewer blocks"); break
        if res.blocks[t] != blk.S_t:
            print("  block", t, "candidates differ"); break
        gs = sorted(res.S.tolist()[o:o + res.b_prime[t]]); os_ = sorted([blk.S_t[i] for i in blk.piv[:blk.b_prime]])
        if gs != os_:
            print("  block", t, "sets differ: gpu-only", sorted(set(gs) - set(os_))[:10], "orc-only", sorted(set(os_) - set(gs))[:10],
                  "gap", blk.pivot_gap, "margin", blk.filter_margin, "mass", blk.mass[:4] if len(blk.mass) else None)
            break
        o += res.b_prime[t]
