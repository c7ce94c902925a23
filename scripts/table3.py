"""the paper's own GPU workload (Table 3) on one B200.

Example 4.1's adversarial GMM, n = 10^5, d = 10^3, 100 clusters; fixed-rank RBRP-ID
(Alg. 2 + Alg. 3) at the table's ranks with b = 40 (the table does not state b,
reading R21).  Prints one JSON line per (form, rank) with the B200 time and the paper's
V100 RBRP-ID time (units unstated in the paper; seconds assumed, reading R21) -- context,
not a target: different hardware, and b and precision are assumptions.
Then SkLUPP-OSID (l = 3k) at the ranks rbrp_sketch_id supports
(k <= RBRP_SK_MAX_K), next to the paper's V100 SkLUPP-OSID row.

    python scripts/table3.py [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import CONFIGS, T3_RANKS, make  # noqa: E402

# Table 3, RBRP-ID row, V100
PAPER_V100_S = dict(zip(T3_RANKS, (3.105e-2, 4.448e-2, 5.838e-2, 7.231e-2, 9.512e-2, 1.073e-1, 1.217e-1,
                                   1.336e-1, 1.473e-1, 1.596e-1)))

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--sketch-only", action="store_true", help="SkLUPP-OSID rows only")
a = ap.parse_args()
# Table 3, SkLUPP-OSID row, V100
PAPER_V100_SK = dict(zip(T3_RANKS, (1.036e-2, 1.204e-2, 1.666e-2, 2.233e-2, 3.430e-2, 4.835e-2, 6.960e-2,
                                    8.254e-2, 1.017e-1, 1.189e-1)))
cfg = CONFIGS["t3"]
X = make(cfg, device="cuda")
m = cfg.n // cfg.n_centres
for form in (() if a.sketch_only else ("residual", "paper")):
    for r in T3_RANKS:
        kw = dict(k=r, b=cfg.b, seed=0, form=form, log_blocks=False)
        rb.id(X, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            res = rb.id(X, **kw)
        e1.record()
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / a.reps / 1e3
        clusters = len({int(i) // m for i in res.S.tolist()})
        print(json.dumps({"workload": "t3 (Example 4.1 GMM 1e5 x 1e3, k=100)", "form": form, "rank": r, "b": cfg.b,
                          "seconds_b200": s, "blocks": res.nblocks, "resid_rel": res.resid_rel,
                          "distinct_clusters": clusters, "paper_v100_rbrp_id_s": PAPER_V100_S[r],
                          "v100_over_b200": PAPER_V100_S[r] / s}), flush=True)
for r in T3_RANKS:
    if r > rb.sketch.SK_MAX_K:
        continue
    kw = dict(k=r, l=3 * r, seed=0)
    rb.sketch_id(X, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        res = rb.sketch_id(X, **kw)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / a.reps / 1e3
    ph = rb.sketch_id(X, profile=True, **kw).ms_phase
    clusters = len({int(i) // m for i in res.S.tolist()})
    print(json.dumps({"workload": "t3 (Example 4.1 GMM 1e5 x 1e3, k=100)", "method": "sklupp_osid", "rank": r,
                      "l": 3 * r, "seconds_b200": s, "ms_phase": ph, "distinct_clusters": clusters,
                      "paper_v100_sklupp_osid_s": PAPER_V100_SK[r], "v100_over_b200": PAPER_V100_SK[r] / s}),
          flush=True)
