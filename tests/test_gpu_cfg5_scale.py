"""BASELINE configs[4] at its full size (1e6 x 2e5, 2e8 uniform observations):
size-independent properties of the CUDA path where no CPU oracle finishes in
seconds -- the CSR and CSC copies describe the same matrix (adjoint identity,
checksums), the products are linear, sampled rows agree with scipy's SpMM
(the reference's own kernel, sparse.py:153-158), and the fused SVT step
(completion.py:373-386) updates sampled entries exactly as the host formula
does.  Inputs: workloads.cfg5_device (the configuration's distribution,
seeded, sampled on the GPU)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg5():
    import torch

    from paper_1810_06860_b200 import workloads
    from paper_1810_06860_b200.sparse import ObservationSet

    o = workloads.cfg5_device()
    torch.cuda.empty_cache()
    obs = ObservationSet(o.m, o.n, o.rows, o.cols, o.values)  # device duplicate search + CSR build
    A = obs.train_matrix()
    yield o, obs, A
    del A, obs, o
    torch.cuda.empty_cache()


def test_cfg5_pattern_and_products(cfg5):
    import scipy.sparse as sps
    import torch

    from paper_1810_06860_b200 import device
    from paper_1810_06860_b200.sparse import spmm_dev, spmm_t_dev

    o, obs, A = cfg5
    assert A.shape == (1_000_000, 200_000) and A.nnz == 200_000_000
    dp = A.pattern()
    # CSR offsets = the host row histogram; CSC offsets = the column histogram; perm is a permutation
    assert np.array_equal(A.indptr[1:], np.cumsum(np.bincount(o.rows, minlength=o.m)))
    assert np.array_equal(device.to_host(dp.csc.ptr)[1:].astype(np.int64),
                          np.cumsum(np.bincount(o.cols, minlength=o.n)))
    perm = dp.perm.long()
    assert int(torch.bincount(perm, minlength=A.nnz).max()) == 1 and int(perm.sum()) == A.nnz * (A.nnz - 1) // 2
    rng = np.random.default_rng(0)
    w = 12
    X = device.to_device(rng.standard_normal((o.n, w)))
    H = device.to_device(rng.standard_normal((o.m, w)))
    YX, YtH = spmm_dev(A, X), spmm_t_dev(A, H)
    # adjoint identity <H, Y X> = <Y^T H, X>: the CSR and CSC copies are the same matrix
    a, b = float((H * YX).sum()), float((YtH * X).sum())
    assert abs(a - b) <= 1e-11 * float(torch.linalg.norm(H) * torch.linalg.norm(YX))
    # checksums: Y 1 and Y^T 1 both sum to the sum of the stored values
    ones_n, ones_m = device.to_device(np.ones((o.n, 2))), device.to_device(np.ones((o.m, 2)))
    total = float(np.sum(o.values))
    scale = float(np.sum(np.abs(o.values)))
    assert abs(float(spmm_dev(A, ones_n)[:, 0].sum()) - total) <= 1e-12 * scale
    assert abs(float(spmm_t_dev(A, ones_m)[:, 0].sum()) - total) <= 1e-12 * scale
    # linearity
    X2 = device.to_device(rng.standard_normal((o.n, w)))
    lhs = spmm_dev(A, 0.3 * X - 1.7 * X2)
    rhs = 0.3 * YX - 1.7 * spmm_dev(A, X2)
    assert float(torch.linalg.norm(lhs - rhs)) <= 1e-13 * float(torch.linalg.norm(rhs)) * np.sqrt(w) * 10
    # sampled rows / columns against scipy's own SpMM
    rows = rng.choice(o.m, 1500, replace=False)
    lo, hi = A.indptr[rows], A.indptr[rows + 1]
    sel = np.concatenate([np.arange(a_, b_) for a_, b_ in zip(lo, hi)])
    sub = sps.csr_matrix((o.values[sel], o.cols[sel], np.concatenate([[0], np.cumsum(hi - lo)])), shape=(1500, o.n))
    ref = sub @ device.to_host(X)
    assert np.linalg.norm(device.to_host(YX[torch.from_numpy(rows).cuda()]) - ref) <= 1e-13 * np.linalg.norm(ref)
    cols = rng.choice(o.n, 300, replace=False)
    mask = np.isin(o.cols, cols)
    subT = sps.csr_matrix((o.values[mask], (o.cols[mask], o.rows[mask])), shape=(o.n, o.m))[cols]
    refT = subT @ device.to_host(H)
    assert np.linalg.norm(device.to_host(YtH[torch.from_numpy(cols).cuda()]) - refT) <= 1e-13 * np.linalg.norm(refT)


@pytest.mark.parametrize("r", [10, 48])
def test_cfg5_fused_step_on_sampled_entries(cfg5, r):
    import torch

    from paper_1810_06860_b200 import completion, device

    o, obs, A = cfg5
    eng = completion.DeviceEngine(obs)
    eng.m_norm = eng.observed_norm()
    assert abs(eng.m_norm - np.linalg.norm(o.values)) <= 1e-12 * eng.m_norm
    eng.start(1.5)
    rng = np.random.default_rng(r)
    U, V = rng.standard_normal((o.m, r)) * 0.3, rng.standard_normal((o.n, r)) * 0.3
    S = rng.random(r) + 0.5
    pick = np.sort(rng.choice(A.nnz, 200_000, replace=False))
    i, j = o.rows[pick], o.cols[pick]  # cfg5's COO is already row-major sorted: slot e of the CSR is entry e
    pick_d = torch.from_numpy(pick).cuda()
    y0 = device.to_host(eng.Y.device_values()[0][pick_d])
    assert np.array_equal(y0, 1.5 * o.values[pick])
    step = 0.37
    resid, _ = eng.step(device.to_device(U), S, device.to_device(V), r, step)
    x = np.einsum("er,er->e", U[i] * S, V[j])
    y1 = device.to_host(eng.Y.device_values()[0][pick_d])
    ref = y0 + step * (o.values[pick] - x)
    assert np.max(np.abs(y1 - ref)) <= 1e-13 * np.max(np.abs(ref))
    # the CSC copy is refreshed to the same values
    yc, yt = eng.Y.device_values()
    assert bool((yt == yc[eng.dp.perm.long()]).all())
    # the residual against a 200k-entry estimate of ||x - m|| / ||m|| (sampling error ~ 1 %)
    est = np.linalg.norm(x - o.values[pick]) / np.linalg.norm(o.values[pick])
    assert abs(resid - est) <= 0.03 * est
