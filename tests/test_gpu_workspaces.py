"""Workspace bounds: every native routine that takes caller-owned scratch is
run with EXACTLY the size its *_workspace_* query reports, followed by a
canary region that must come back untouched (an overflow into a neighbouring
tensor is invisible to results until it corrupts one -- the syevd T-factor
overflow for n < 32 was found that way)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CANARY = 1234.5678
GUARD = 4096


def _guarded(ndoubles):
    import torch

    buf = torch.full((int(ndoubles) + GUARD,), CANARY, dtype=torch.float64, device="cuda")
    return buf, buf[: int(ndoubles)]


def _intact(buf, ndoubles):
    import torch

    torch.cuda.synchronize()
    tail = buf[int(ndoubles):].cpu().numpy()
    return bool(np.all(tail == CANARY))


@pytest.mark.parametrize("n", [2, 3, 5, 8, 17, 31, 32, 33, 64, 96, 97, 130, 260])
@pytest.mark.parametrize("method", ["syevd", "syevj"])
def test_eigensolver_workspaces(n, method):
    from paper_1810_06860_b200 import _native, device

    lib = _native.load()
    X = np.random.default_rng(n).standard_normal((2 * n, n))
    A = device.to_device(X.T @ X)
    d = device.vector(n)
    V = device.empty(n, n)
    if method == "syevd":
        need = int(lib.lr_syevd_workspace_doubles(n))
        buf, work = _guarded(need)
        ncl = ctypes.c_int(0)
        _native.call("lr_syevd_f64", n, device.ptr(A), device.ld(A), device.ptr(d), device.ptr(V), device.ld(V),
                     device.ptr(work), ctypes.byref(ncl), device.stream())
    else:
        need = int(lib.lr_syevj_workspace_doubles(n))
        buf, work = _guarded(need)
        sweeps = ctypes.c_int(0)
        _native.call("lr_syevj_f64", n, device.ptr(A), device.ld(A), device.ptr(d), device.ptr(V), device.ld(V),
                     60, device.ptr(work), ctypes.byref(sweeps), device.stream())
    assert _intact(buf, need), (method, n)
    np.testing.assert_allclose(np.sort(device.to_host(d)), np.linalg.eigvalsh(X.T @ X), rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("n", [1, 5, 31, 32, 33, 100, 660])
def test_potrf_workspace(n):
    from paper_1810_06860_b200 import _native, device

    lib = _native.load()
    X = np.random.default_rng(n).standard_normal((3 * n + 2, n))
    G = device.to_device(X.T @ X)
    Rinv = device.empty(n, n)
    need = int(lib.lr_potrf_workspace_doubles(n))
    buf, work = _guarded(need)
    info = ctypes.c_int(0)
    _native.call("lr_potrf_inv_f64", n, device.ptr(G), device.ld(G), 0.0, device.ptr(Rinv), device.ld(Rinv),
                 device.ptr(work), ctypes.byref(info), device.stream())
    assert info.value == 0 and _intact(buf, need)


@pytest.mark.parametrize("m,n", [(7, 3), (40, 16), (1000, 16), (3000, 40), (20000, 110)])
def test_lu_workspace(m, n):
    from paper_1810_06860_b200 import _native, device

    lib = _native.load()
    X = device.to_device(np.random.default_rng(m).standard_normal((m, n)))
    need = int(lib.lr_lu_workspace_doubles(m, n))
    buf, work = _guarded(need)
    status = (ctypes.c_double * 4)()
    _native.call("lr_lu_pl_f64", m, n, device.ptr(X), device.ld(X), device.ptr(work), status, device.stream())
    assert status[0] == -1.0 and _intact(buf, need)


@pytest.mark.parametrize("M,N,K,transA,flags", [(660, 660, 100000, 1, 2), (110, 110, 5000, 1, 2), (50, 7, 90000, 1, 0),
                                                 (300, 40, 3000, 1, 0)])
def test_gemm_splitk_workspace(M, N, K, transA, flags):
    from paper_1810_06860_b200 import _native, device

    lib = _native.load()
    rng = np.random.default_rng(M + N)
    A = device.to_device(rng.standard_normal((K, M) if transA else (M, K)))
    B = A if flags == 2 else device.to_device(rng.standard_normal((K, N)))
    C = device.empty(M, N)
    need = int(lib.lr_gemm_workspace_doubles(transA, M, N, K, flags))
    buf, work = _guarded(max(need, 1))
    _native.call("lr_gemm_f64", transA, M, N, K, 1.0, device.ptr(A), device.ld(A), device.ptr(B), device.ld(B), 0.0,
                 device.ptr(C), device.ld(C), flags, device.ptr(work), need, device.stream())
    assert _intact(buf, max(need, 1))
    Ah, Bh = device.to_host(A), device.to_host(B)
    ref = Ah.T @ Bh if transA else Ah @ Bh
    assert np.abs(device.to_host(C) - ref).max() <= 1e-12 * np.abs(ref).max()
