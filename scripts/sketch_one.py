"""One SkLUPP-OSID call on the Table 3 matrix at rank k (l = 3k), for launch lists:
python scripts/sketch_one.py [k]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_16002_b200 as rb  # noqa: E402
from workloads import CONFIGS, make  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 472
cfg = CONFIGS["t3"]
X = make(cfg, device="cuda")
r = rb.sketch_id(X, k, 3 * k, seed=0, profile=True)
torch.cuda.synchronize()
print(k, r.k, {n: round(v, 3) for n, v in r.ms_phase.items()})
