import sys; sys.path.insert(0, ".")
import paper_2309_16002_b200 as rb
from workloads import CONFIGS, make
X = make(CONFIGS["c5"], device="cuda")
r = rb.id(X, tol=0.0020709267553592823, b=128, seed=0, k_max=768)
print(r.k)
