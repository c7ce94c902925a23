import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_16002_b200 as rb
torch.manual_seed(0)
for (n, d, r) in [(65536, 256, 128), (65536, 1024, 128), (65536, 1024, 1000), (8192, 1024, 1000)]:
    X = torch.randn(n, r, dtype=torch.float64, device="cuda") @ torch.randn(r, d, dtype=torch.float64, device="cuda")
    print(f"n={n} d={d} rank={r}", file=sys.stderr)
    res = rb.id(X, k=64, b=32, seed=0)
    torch.cuda.synchronize()
