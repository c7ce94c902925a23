"""The C-ABI library loads and exports every symbol include/rbrp.h declares;
host-side validation (no GPU needed: these calls fail before any CUDA work)."""
import ctypes
import os
import re

import pytest
import torch

from tests.conftest import ROOT

rb = pytest.importorskip("paper_2309_16002_b200.rbrp")


def _declared(header="rbrp.h"):
    txt = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(rbrp_\w+)\s*\(", txt, re.M)))


def test_library_exports_header_symbols():
    L = rb.lib()
    decl = _declared()
    assert "rbrp_id" in decl and "rbrp_workspace_size" in decl
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(rb.EXPORTED)


def test_library_exports_sketch_header_symbols():
    from paper_2309_16002_b200 import sketch as sk
    L = sk.lib()
    decl = _declared("rbrp_sketch.h")
    assert "rbrp_sketch_id" in decl and "rbrp_lupp" in decl
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(sk.EXPORTED)
    headers = sorted(f for f in os.listdir(os.path.join(ROOT, "include")) if f.endswith(".h"))
    assert headers == ["rbrp.h", "rbrp_sketch.h"]


def test_sketch_validation_before_cuda():
    from paper_2309_16002_b200 import sketch as sk
    L = sk.lib()
    sz = ctypes.c_size_t()
    assert L.rbrp_sketch_workspace_size(1000, 64, 10, 30, ctypes.byref(sz)) == 0
    assert sz.value > 1000 * 32 * 8
    for bad in [(1000, 64, 0, 30), (1000, 64, 10, 9), (1000, 64, 10, 41), (4000, 2048, 513, 1600),
                (5, 64, 10, 30)]:
        assert L.rbrp_sketch_workspace_size(*bad, ctypes.byref(sz)) == -1, bad
    assert L.rbrp_sketch_workspace_size(1000, 16, 10, 30, ctypes.byref(sz)) == 0   # l > d allowed
    assert L.rbrp_lupp_workspace_size(1000, 30, 10, ctypes.byref(sz)) == 0
    assert L.rbrp_lupp_workspace_size(1000, 30, 31, ctypes.byref(sz)) == -1
    assert L.rbrp_gaussian_embedding(0, 10, 0, None, 0, None) == -1


def test_version_and_strerror():
    L = rb.lib()
    assert L.rbrp_version() == (0 << 16) | 1
    for code, name in rb.STATUS.items():
        assert L.rbrp_strerror(code).decode().startswith(name)
    assert b"unknown" in L.rbrp_strerror(-99)


def _ws(**kw):
    X = torch.empty((1000, 64), dtype=torch.float64)
    return rb.workspace_size(X, **kw)


def test_workspace_size_and_validation():
    base = _ws(tol=0.1, b=16)
    assert base > 1000 * 64 * 8
    assert _ws(tol=0.1, b=16, inplace=True) < base
    assert _ws(tol=0.1, b=16, with_W=False) < base
    for bad in [dict(tol=1.0), dict(tol=float("nan")), dict(tol=0.1, b=0), dict(tol=0.1, b=129),
                dict(tol=0.0), dict(tol=0.1, tau_b=1.5)]:
        kw = dict(b=16)
        kw.update(bad)
        with pytest.raises(rb.RBRPError) as e:
            _ws(**kw)
        assert e.value.status == -1
    assert _ws(k=10, b=4) > 0          # fixed-rank mode


def test_rbrp_id_rejects_before_cuda():
    L = rb.lib()
    X = torch.empty((100, 8), dtype=torch.float64)
    p = rb._problem(X, 0.1, None, 8, 0, 0, -1.0, 0, None, 0, False)
    S = (ctypes.c_int64 * 8)()
    # workspace too small -> ENOMEM; NULL S_out -> EINVAL
    rc = L.rbrp_id(ctypes.byref(p), ctypes.c_void_p(1), ctypes.c_void_p(256), 16, None, None, S,
                   None, None)
    assert rc == -4
    rc = L.rbrp_id(ctypes.byref(p), ctypes.c_void_p(1), ctypes.c_void_p(256), 1 << 40, None, None,
                   None, None, None)
    assert rc == -1
    p.ld = 4   # ld < d
    rc = L.rbrp_id(ctypes.byref(p), ctypes.c_void_p(1), ctypes.c_void_p(256), 1 << 40, None, None,
                   S, None, None)
    assert rc == -1


def test_binding_refuses_cpu_tensor():
    with pytest.raises(ValueError):
        rb.id(torch.ones((10, 3), dtype=torch.float64), tol=0.1)
