"""Out-of-bounds and uninitialised-memory checks of our own (compute-sanitizer is closed on
this GPU pool: gpurun refuses it, see profiles/README.md).

* Guard bands: X, the workspace and W_out are carved from larger buffers whose margins hold
  a byte pattern; every kernel family runs; the margins must be intact afterwards (a write
  past any caller buffer would show), and X must be unchanged (read-only unless INPLACE).
* Poisoned workspace: the same call on a workspace pre-filled with NaN bytes and on a zeroed
  one must give bit-identical S, rho, d and W (no kernel may consume workspace memory it did
  not write first in this call).
"""
import pytest
import torch

from workloads import make, small_config

pytestmark = pytest.mark.gpu

cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")

G = 1 << 16   # guard bytes on each side (multiple of 256: keeps the 256-byte alignment)


def _rb():
    import paper_2309_16002_b200 as rb
    return rb


def _guarded(nbytes, fill):
    buf = torch.full((nbytes + 2 * G,), fill, dtype=torch.uint8, device="cuda")
    return buf, buf[G:G + nbytes]


def _intact(buf, nbytes, fill):
    return bool((buf[:G] == fill).all()) and bool((buf[G + nbytes:] == fill).all())


CASES = [
    ("c2", dict(n=9000, d=256, rank=40, b=16), dict(tol=1e-12), {}),
    ("c2", dict(n=9000, d=256, rank=40, b=16), dict(tol=1e-12, form="paper"), {}),
    ("c2", dict(n=9000, d=256, rank=40, b=32), dict(tol=1e-12), {"RBRP_NO_GRAPH": "1"}),
    ("c5", dict(n=12000, d=160, n_centres=120, b=64), dict(k=100), {}),
    ("c4", dict(n=9000, d=192, b=64), dict(tol=1e-3), {}),     # fp32: tcgen05 projection
    ("c4", dict(n=9000, d=100, b=40), dict(tol=1e-3), {}),     # fp32: ragged d (tcgen05, partial chunk)
]


@cuda
@pytest.mark.parametrize("name,kw,call,env", CASES)
def test_guard_bands_and_poisoned_workspace(monkeypatch, name, kw, call, env):
    rb = _rb()
    for k_, v in env.items():
        monkeypatch.setenv(k_, v)
    cfg = small_config(name, **kw)
    X0 = make(cfg, device="cuda")
    n, d = X0.shape
    es = X0.element_size()
    xbuf, xv = _guarded(n * d * es, 0x5A)
    X = xv.view(X0.dtype).view(n, d)
    X.copy_(X0)
    k_cap = call.get("k", min(n, d))
    wsz = rb.workspace_size(X, tol=call.get("tol"), k=call.get("k"), b=cfg.b)
    wbuf, wv = _guarded(n * k_cap * es, 0xA5)
    W = wv.view(X0.dtype).view(n, k_cap)
    results = []
    for fill in (0x00, 0xFF):   # zeroed workspace, then all-NaN bytes
        sbuf, sv = _guarded(wsz, 0x3C)
        sv.fill_(fill)
        r = rb.id(X, b=cfg.b, seed=3, workspace=sv, W_out=W, return_d=True, **call)
        torch.cuda.synchronize()
        assert _intact(sbuf, wsz, 0x3C), "write outside the workspace"
        assert _intact(wbuf, n * k_cap * es, 0xA5), "write outside W_out"
        assert _intact(xbuf, n * d * es, 0x5A), "write outside X"
        assert torch.equal(X, X0), "X modified"
        results.append((r.S.tolist(), r.rho, r.b_prime, r.d.clone(), r.W.clone()))
    (S0, rho0, bp0, d0, W0), (S1, rho1, bp1, d1, W1) = results
    assert S0 == S1 and rho0 == rho1 and bp0 == bp1
    assert torch.equal(d0, d1) and torch.equal(W0, W1)
    assert torch.isfinite(W0).all() and torch.isfinite(d0).all()


@cuda
def test_guard_bands_sharded_and_form_w():
    rb = _rb()
    cfg = small_config("c2", n=3 * 4096 + 77, d=128, rank=30, b=16)
    X = make(cfg, device="cuda")
    ref = rb.id(X, tol=1e-12, b=16, seed=2)
    res, Ws = rb.rbrp.id_sharded([X[:4096], X[4096:8192], X[8192:]], tol=1e-12, b=16, seed=2)
    assert res.S.tolist() == ref.S.tolist()
    assert torch.equal(torch.cat(Ws, 0), ref.W)
    # Alg. 3 on its own into a guarded W
    L = torch.randn(2000, 48, dtype=torch.float64, device="cuda")
    S = list(range(0, 2000, 41))[:48]
    L[S] = torch.eye(48, dtype=torch.float64, device="cuda") + 0.01 * torch.tril(
        torch.randn(48, 48, dtype=torch.float64, device="cuda"), -1)
    wbuf, wv = _guarded(2000 * 48 * 8, 0x77)
    Wg = wv.view(torch.float64).view(2000, 48)
    for method in ("trsm", "pinv"):
        rb.rbrp.form_w(L, S, method=method, W_out=Wg)
        torch.cuda.synchronize()
        assert _intact(wbuf, 2000 * 48 * 8, 0x77)
