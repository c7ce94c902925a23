"""The NCCL data path of the row-sharded RBRP on one GPU: a one-rank
communicator runs every exchange point of a multi-GPU call for real (NCCL loaded at run
time, chunk totals, draw-round candidates, V rows and L_1 through ncclAllReduce on the
device) and must give exactly the single-GPU result -- the same S, b' and rho_t bit for
bit, the same W -- and match the oracle in replay.  Runs in a subprocess so that its
torch.distributed process group (gloo, 127.0.0.1) cannot leak into other tests."""
import os
import subprocess
import sys
import textwrap

import pytest
import torch

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu
cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")

SCRIPT = textwrap.dedent(r"""
    import os, sys, socket
    sys.path.insert(0, os.environ["ROOT"])
    import numpy as np, torch, torch.distributed as dist
    import paper_2309_16002_b200 as rb
    from paper_2309_16002_b200 import dist as rdist
    from oracle import rbrp as O
    from workloads import make, small_config
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    dev = torch.device("cuda", 0)
    comm = rdist.Comm(dev)
    for form in ("residual", "paper"):
        cfg = small_config("c2", n=3 * 4096 + 1000, d=256, rank=40, b=16)
        X = make(cfg, device="cuda")
        a = rb.id(X, tol=1e-12, b=16, seed=3, form=form)
        c = rdist.id_distributed(X, cfg.n, 0, comm, tol=1e-12, b=16, seed=3, form=form)
        assert c.graph, form        # the loop with its NCCL collectives captured as one graph
        assert a.S.tolist() == c.S.tolist(), form
        assert a.b_prime == c.b_prime and a.rho == c.rho, form
        assert torch.allclose(a.W, c.W, rtol=0, atol=1e-12), form
        assert c.k == 40
        os.environ["RBRP_NO_GRAPH"] = "1"   # the eager, host-driven loop: same answer
        e = rdist.id_distributed(X, cfg.n, 0, comm, tol=1e-12, b=16, seed=3, form=form)
        del os.environ["RBRP_NO_GRAPH"]
        assert not e.graph and e.S.tolist() == c.S.tolist() and e.rho == c.rho, form
    # replay through the communicator against the oracle
    cfg = small_config("c3", n=12000, d=64, n_heavy_dirs=20, n_heavy_rows=6000, b=16)
    Xnp = make(cfg).numpy()
    tau = 0.05
    ores = O.rbrp(Xnp, tau=tau, b=16, seed=0)
    X = torch.from_numpy(Xnp).cuda()
    r = rdist.id_distributed(X, cfg.n, 0, comm, k=ores.k, b=16,
                             replay_blocks=[blk.S_t for blk in ores.blocks],
                             replay_pivots=[blk.piv for blk in ores.blocks])
    assert r.S.tolist() == ores.S
    assert r.b_prime == [blk.b_prime for blk in ores.blocks]
    assert max(abs(x - blk.rho) for x, blk in zip(r.rho, ores.blocks)) <= 1e-10
    comm.close()
    dist.destroy_process_group()
    print("OK")
""")


@cuda
def test_one_rank_nccl_communicator_equals_single_gpu():
    env = dict(os.environ, ROOT=ROOT, MASTER_ADDR="127.0.0.1")
    p = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "OK" in p.stdout, p.stdout[-2000:] + p.stderr[-4000:]
