"""GPU parity of the individual kernels against the CPU oracle (oracle/),
on seeded inputs.  Tolerances are the reference's own:
SpMM 1e-12 * ||ref||, SDDMM 1e-12, eigSVD values 1e-10 relative,
projectors 1e-8..1e-10; integer/structural results exact."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

lr = pytest.importorskip("paper_1810_06860_b200")


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def rand_pattern(m, n, nnz, seed, long_rows=0, long_cols=0):
    rng = np.random.default_rng(seed)
    flat = rng.choice(m * n, size=nnz, replace=False)
    i, j = np.divmod(flat, n)
    extra_i, extra_j = [], []
    for r in range(long_rows):  # fully dense rows (exercise the split schedule)
        extra_i.append(np.full(n, r))
        extra_j.append(np.arange(n))
    for c in range(long_cols):
        extra_i.append(np.arange(m))
        extra_j.append(np.full(m, n - 1 - c))
    if extra_i:
        i = np.concatenate([i] + extra_i)
        j = np.concatenate([j] + extra_j)
        key = np.unique(i * n + j)
        i, j = np.divmod(key, n)
    v = rng.standard_normal(i.shape[0])
    return i, j, v


@pytest.mark.parametrize("w", [1, 2, 3, 7, 16, 33, 64, 65, 110, 131, 200])
def test_spmm_and_spmm_t_match_oracle(w):
    from paper_1810_06860_b200.sparse import SparseMatrix, spmm, spmm_t

    m, n = 700, 1300
    i, j, v = rand_pattern(m, n, 20000, seed=w, long_rows=2, long_cols=1)
    A = SparseMatrix.from_coo(m, n, i, j, v)
    P = oracle.csr_from_triples(m, n, i, j, v)
    rng = np.random.default_rng(100 + w)
    X = rng.standard_normal((n, w))
    H = rng.standard_normal((m, w))
    ref = oracle.csr_times_dense(P, X)
    assert np.linalg.norm(spmm(A, X) - ref) <= 1e-12 * np.linalg.norm(ref)
    ref_t = oracle.csr_t_times_dense(P, H)
    assert np.linalg.norm(spmm_t(A, H) - ref_t) <= 1e-12 * np.linalg.norm(ref_t)


@pytest.mark.parametrize("w", [2, 5, 16, 22, 45, 89, 132, 260])
def test_spmm_hot_rows_bit_identical(w, monkeypatch):
    """lr_spmm_hot_f64 (the most frequent block rows staged in shared memory
    by one TMA bulk copy; opt-in, LR_SPMM_HOT=1) against lr_spmm_f64 on a
    Zipf-skewed pattern with dense rows / columns (split schedule): the same
    chunks, lane map and summation order, so bit-identical on both sides;
    ranks past the staged rows go through the order lookup (w = 260: 128-column
    chunks stage ~220 of the 600 encoded rows)."""
    import torch

    from paper_1810_06860_b200 import device, sparse
    from paper_1810_06860_b200.sparse import SparseMatrix, spmm_dev, spmm_t_dev

    m, n, nnz = 3000, 600, 150000
    rng = np.random.default_rng(w)
    pj = 1.0 / np.arange(1, n + 1) ** 0.9
    pi = 1.0 / np.arange(1, m + 1)
    j = rng.permutation(n)[rng.choice(n, size=nnz, p=pj / pj.sum())]
    i = rng.permutation(m)[rng.choice(m, size=nnz, p=pi / pi.sum())]
    key = np.unique(np.concatenate([i * n + j, np.arange(n), (m - 1) * n + np.arange(n), np.arange(m) * n + 7]))
    i, j = np.divmod(key, n)
    A = SparseMatrix.from_coo(m, n, i, j, rng.standard_normal(i.shape[0]))
    X = device.to_device(rng.standard_normal((n, w)))
    H = device.to_device(rng.standard_normal((m, w)))
    y0, t0 = spmm_dev(A, X), spmm_t_dev(A, H)
    monkeypatch.setattr(sparse, "HOT_ROWS", True)
    monkeypatch.setattr(sparse, "HOT_MIN_NNZ", 0)
    monkeypatch.setattr(sparse, "HOT_MIN_SHARE", 0.0)
    dp = A.pattern()
    dp.csr._hot = dp.csc._hot = False  # examine the sides again under the opt-in
    assert dp.csr.hot() is not None and dp.csc.hot() is not None
    hot_c = dp.csr.hot()
    assert int((hot_c[0] < 0).sum()) == int(round(hot_c[3][-1] * A.nnz))  # encoded entries = the top ranks' share
    calls = []
    from paper_1810_06860_b200 import _native
    real = _native.call
    monkeypatch.setattr(_native, "call", lambda name, *a, **k: (calls.append(name), real(name, *a, **k))[1])
    y1, t1 = spmm_dev(A, X), spmm_t_dev(A, H)
    assert calls == ["lr_spmm_hot_f64", "lr_spmm_hot_f64"]
    assert torch.equal(y0, y1) and torch.equal(t0, t1)


@pytest.mark.parametrize("w,off", [(5, 1), (11, 3), (22, 7), (45, 45), (45, 90), (89, 1), (131, 5)])
def test_spmm_column_slice_at_odd_offset_is_bit_identical(w, off):
    """Y X and Y^T X with X a column slice of a wider block starting at an
    odd column (the Krylov blocks H_i of rsvd_bki for odd k + s): the
    line-aligned group kernel reads the chunks from the row's 128-byte line,
    so the slice need not start a 16-byte chunk; same bits as the product with
    a contiguous copy of the slice."""
    import torch

    from paper_1810_06860_b200 import device
    from paper_1810_06860_b200.sparse import SparseMatrix, spmm_dev, spmm_t_dev

    m, n = 1500, 900
    i, j, v = rand_pattern(m, n, 40000, seed=w + off, long_rows=1, long_cols=1)
    A = SparseMatrix.from_coo(m, n, i, j, v)
    rng = np.random.default_rng(off)
    Xw = device.to_device(rng.standard_normal((n, off + w + 3)))
    Hw = device.to_device(rng.standard_normal((m, off + w + 3)))
    Xs, Hs = Xw[:, off:off + w], Hw[:, off:off + w]
    Xc, Hc = device.empty(n, w), device.empty(m, w)
    Xc.copy_(Xs)
    Hc.copy_(Hs)
    assert torch.equal(spmm_dev(A, Xs), spmm_dev(A, Xc))
    assert torch.equal(spmm_t_dev(A, Hs), spmm_t_dev(A, Hc))
    out = device.empty(m, off + w + 3)  # and into a column slice of a wider block
    spmm_dev(A, Xs, out=out[:, off:off + w])
    assert torch.equal(out[:, off:off + w], spmm_dev(A, Xc))


def test_spmm_golden(golden):
    from paper_1810_06860_b200.sparse import SparseMatrix, spmm, spmm_t

    A = SparseMatrix.from_coo(60, 45, golden["sp_i"], golden["sp_j"], golden["sp_v"])
    assert np.array_equal(A.indptr, golden["sp_indptr"]) and np.array_equal(A.indices, golden["sp_indices"])
    perm, tip, tix = A._transpose_index()
    assert np.array_equal(perm, golden["sp_tperm"]) and np.array_equal(tix, golden["sp_tindices"])
    assert rel(spmm(A, golden["sp_X"]), golden["sp_spmm"]) <= 1e-12
    assert rel(spmm_t(A, golden["sp_H"]), golden["sp_spmm_t"]) <= 1e-12


def test_spmm_empty_rows_and_identity():
    from paper_1810_06860_b200.sparse import SparseMatrix, spmm, spmm_t

    A = SparseMatrix.from_coo(5, 4, [0, 4], [1, 3], [2.0, -1.0])  # rows 1..3 empty
    X = np.arange(12.0).reshape(4, 3)
    np.testing.assert_array_equal(spmm(A, X), A.densify() @ X)
    H = np.arange(15.0).reshape(5, 3)
    np.testing.assert_array_equal(spmm_t(A, H), A.densify().T @ H)
    I = SparseMatrix.identity(9)
    Z = np.random.default_rng(0).standard_normal((9, 4))
    np.testing.assert_array_equal(spmm(I, Z), Z)
    with pytest.raises(ValueError, match="dimension mismatch"):
        spmm(A, np.ones((5, 2)))


def test_sddmm_and_frobenius(golden):
    from paper_1810_06860_b200.sparse import SparseMatrix, frobenius, project_pattern

    A = SparseMatrix.from_coo(60, 45, golden["sp_i"], golden["sp_j"], golden["sp_v"])
    x = project_pattern(golden["sp_U"], golden["sp_S"], golden["sp_V"], A)
    assert rel(x, golden["sp_project"]) <= 1e-12
    assert abs(frobenius(A.data) - float(golden["sp_frob"])) <= 1e-14 * float(golden["sp_frob"])
    assert frobenius(np.array([3.0, 4.0])) == 5.0
    assert frobenius(np.zeros(0)) == 0.0 and frobenius(np.zeros(7)) == 0.0
    assert abs(frobenius(np.array([3e200, 4e200])) - 5e200) <= 1e-14 * 5e200


def test_update_pattern_values_both_copies():
    from paper_1810_06860_b200.sparse import SparseMatrix, spmm, spmm_t, update_pattern_values

    i, j, v = rand_pattern(80, 50, 900, seed=3)
    A = SparseMatrix.from_coo(80, 50, i, j, v)
    data_id = id(A.data)
    X = np.random.default_rng(1).standard_normal((50, 4))
    spmm(A, X)  # materialise device copies
    delta = np.random.default_rng(2).standard_normal(A.nnz)
    update_pattern_values(A, delta)
    assert id(A.data) == data_id
    np.testing.assert_allclose(A.data, v[np.lexsort((j, i))] + delta, rtol=0, atol=0)
    D = A.densify()
    np.testing.assert_allclose(spmm(A, X), D @ X, rtol=1e-12, atol=1e-12)
    H = np.random.default_rng(3).standard_normal((80, 4))
    np.testing.assert_allclose(spmm_t(A, H), D.T @ H, rtol=1e-12, atol=1e-12)


def test_spectral_norm_matches_oracle(golden):
    from paper_1810_06860_b200.rng import RngState
    from paper_1810_06860_b200.sparse import SparseMatrix, spectral_norm_est

    A = SparseMatrix.from_coo(60, 45, golden["sp_i"], golden["sp_j"], golden["sp_v"])
    got = spectral_norm_est(A, RngState(3))
    assert abs(got - float(golden["sp_norm2"])) <= 1e-12 * got


@pytest.mark.parametrize("M,N,K,transA", [(64, 64, 64, 0), (100, 37, 129, 0), (1000, 110, 110, 0),
                                          (7, 5, 3, 0), (660, 660, 5000, 1), (33, 17, 100000, 1),
                                          (1, 1, 1, 1)])
def test_gemm_matches_numpy(M, N, K, transA):
    import torch

    from paper_1810_06860_b200 import device
    from paper_1810_06860_b200.linalg import matmul_dev, matmul_tn_dev

    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((K, M) if transA else (M, K))
    B = rng.standard_normal((K, N))
    ref = (A.T if transA else A) @ B
    got = device.to_host((matmul_tn_dev if transA else matmul_dev)(device.to_device(A), device.to_device(B)))
    assert rel(got, ref) <= 1e-14 * max(1.0, np.sqrt(K) / 10)
    del torch


def test_gram_is_exactly_symmetric_and_accurate():
    from paper_1810_06860_b200 import device
    from paper_1810_06860_b200.linalg import gram_dev

    A = np.random.default_rng(5).standard_normal((20000, 131))
    G = device.to_host(gram_dev(device.to_device(A)))
    assert np.array_equal(G, G.T)
    assert rel(G, A.T @ A) <= 1e-14


def test_upper_triangular_b_and_potrf_inverse():
    from paper_1810_06860_b200 import device
    from paper_1810_06860_b200.linalg import matmul_dev, potrf_inv_dev

    for n in (1, 5, 31, 32, 33, 64, 65, 130, 300, 660, 1220, 2048, 2050):
        X = np.random.default_rng(n).standard_normal((3 * n + 10, n))
        G = X.T @ X
        Gd = device.to_device(G)
        info, Rinv = potrf_inv_dev(Gd)
        assert info == 0
        R = device.to_host(Gd)
        Rref = np.linalg.cholesky(G).T
        assert np.allclose(np.tril(R, -1), 0.0)
        assert rel(R, Rref) <= 1e-12
        Ri = device.to_host(Rinv)
        assert rel(Ri @ R, np.eye(n)) <= 1e-10
        Q = device.to_host(matmul_dev(device.to_device(X), Rinv, b_upper=True))
        assert rel(Q.T @ Q, np.eye(n)) <= 1e-9
    # breakdown is reported, not raised (1-based column of the first bad pivot)
    info, _ = potrf_inv_dev(device.to_device(np.array([[1.0, 2.0], [2.0, 1.0]])))
    assert info == 2
    for n, bad in ((100, 70), (660, 33), (660, 659)):
        X = np.random.default_rng(bad).standard_normal((2 * n, n))
        X[:, bad] = X[:, :bad] @ np.random.default_rng(1).standard_normal(bad)  # dependent column
        G = X.T @ X
        G[bad, bad] -= 1e-6 * G[bad, bad]  # push the Schur complement negative
        info, _ = potrf_inv_dev(device.to_device(G))
        assert info == bad + 1, (n, bad, info)
    # shifted factorization (shifted CholeskyQR3): R^T R = G + shift I
    X = np.random.default_rng(7).standard_normal((500, 200))
    G = X.T @ X
    Gd = device.to_device(G)
    info, Rinv = potrf_inv_dev(Gd, 3.5)
    R = device.to_host(Gd)
    assert info == 0 and rel(R.T @ R, G + 3.5 * np.eye(200)) <= 1e-13


@pytest.mark.parametrize("m,n", [(25, 7), (300, 40), (5000, 110), (100000, 110), (138493, 65), (40, 40),
                                 (20000, 300), (60000, 305), (3000, 17)])
def test_lu_pl_structure_and_span(m, n):
    from paper_1810_06860_b200.linalg import lu_pl

    X = np.random.default_rng(m + n).standard_normal((m, n))
    PL = lu_pl(X)
    assert PL.shape == (m, n)
    assert np.max(np.abs(PL)) <= 1.0 + 1e-12
    ref = oracle.pivoted_lower(X)
    # same pivots (no near ties in Gaussian data) -> same factor to rounding
    assert rel(PL, ref) <= 1e-10
    Qa, _ = np.linalg.qr(PL)
    Qb, _ = np.linalg.qr(X)
    assert np.linalg.norm(Qa @ (Qa.T @ Qb) - Qb) <= 1e-8 * np.sqrt(n)


def test_lu_pl_golden(golden):
    from paper_1810_06860_b200.linalg import lu_pl

    assert rel(lu_pl(golden["lu_X"]), golden["lu_PL"]) <= 1e-12
    assert rel(lu_pl(golden["lu2_X"]), golden["lu2_PL"]) <= 1e-12


def test_lu_pl_errors():
    from paper_1810_06860_b200.errors import RankDeficiencyError
    from paper_1810_06860_b200.linalg import lu_pl

    with pytest.raises(RankDeficiencyError, match="zero matrix"):
        lu_pl(np.zeros((10, 3)))
    X = np.random.default_rng(0).standard_normal((30, 5))
    X[:, 3] = X[:, 1]
    with pytest.raises(RankDeficiencyError, match="zero pivot at column 3"):
        lu_pl(X)
    with pytest.raises(ValueError):
        lu_pl(np.ones((3, 5)))
    # the cooperative (multi-CTA) kernel reports the same column
    Z = np.random.default_rng(1).standard_normal((60000, 70))
    Z[:, 41] = Z[:, 7] - 2.0 * Z[:, 30]
    with pytest.raises(RankDeficiencyError, match="zero pivot at column 41"):
        lu_pl(Z)
    Y = np.ones((6, 2))
    Y[1, 1] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        lu_pl(Y)


@pytest.mark.parametrize("n", [1, 2, 3, 11, 50, 96, 97, 130, 260, 400, 700, 1400])
def test_sym_eig_matches_numpy(n):
    from paper_1810_06860_b200.linalg import sym_eig

    X = np.random.default_rng(n).standard_normal((n + 20, n))
    B = X.T @ X
    V, d = sym_eig(B)
    dref = np.linalg.eigvalsh(B)
    assert np.all(np.diff(d) >= 0)
    assert np.max(np.abs(d - dref)) <= 1e-12 * dref[-1]
    assert rel(V.T @ V, np.eye(n)) <= 1e-12 * max(1, n / 10)
    assert rel(B @ V, V * d) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("n,groups", [(40, [1, 1, 1, 2, 3, 3]), (300, None), (660, "big")])
def test_sym_eig_clusters(n, groups):
    """Repeated eigenvalues: the device cluster finder + MGS keep V orthonormal
    (n = 300: 150 equal pairs, more clusters than the MGS grid; n = 660: one
    600-fold cluster, the O(k^2) worst case of the one-CTA-per-cluster MGS)."""
    import ctypes

    import torch

    from paper_1810_06860_b200 import _native, device
    from paper_1810_06860_b200.linalg import sym_eig

    rng = np.random.default_rng(n)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    if groups is None:
        d0 = np.repeat(np.arange(1.0, n // 2 + 1), 2)
    elif groups == "big":
        d0 = np.concatenate([np.full(600, 5.0), 10.0 + np.arange(n - 600)])
    else:
        d0 = np.concatenate([groups, 10.0 + np.arange(n - len(groups))])
    B = (Q * d0) @ Q.T
    B = (B + B.T) / 2
    V, d = sym_eig(B)
    assert np.max(np.abs(d - np.sort(d0))) <= 1e-12 * d0.max() * 10
    assert rel(V.T @ V, np.eye(n)) <= 1e-12 * max(1, n / 10)
    assert rel(B @ V, V * d) <= 1e-12
    # raw ABI with the optional host count
    A = device.to_device(B)
    dd, VV = device.vector(n), device.empty(n, n)
    work = torch.empty(int(_native.load().lr_syevd_workspace_doubles(n)), dtype=torch.float64, device="cuda")
    ncl = ctypes.c_int(-1)
    _native.call("lr_syevd_f64", n, device.ptr(A), device.ld(A), device.ptr(dd), device.ptr(VV), device.ld(VV),
                 device.ptr(work), ctypes.byref(ncl), device.stream())
    expect = n // 2 if groups is None else (1 if groups == "big" else 2)
    assert ncl.value == expect


def test_eig_svd_golden_and_acceptance_01(golden):
    from paper_1810_06860_b200.linalg import eig_svd

    r = eig_svd(golden["eig_A"])
    assert r.order == "ascending"
    assert rel(r.S, golden["eig_S"]) <= 1e-12
    assert rel(r.V, golden["eig_V"]) <= 1e-9  # same sign rule
    assert rel(r.U, golden["eig_U"]) <= 1e-9
    worst_val = worst_rec = 0.0
    for seed in range(30):  # test_acceptance.py:92-110 contract on 30 seeds
        rng = np.random.default_rng(seed)
        n = int(rng.integers(5, 61))
        m = int(rng.integers(n, 301))
        A = rng.standard_normal((m, n))
        got = eig_svd(A).descending()
        ref = np.linalg.svd(A, compute_uv=False)
        worst_val = max(worst_val, float(np.max(np.abs(got.S - ref)) / ref[0]))
        worst_rec = max(worst_rec, np.linalg.norm(A - (got.U * got.S) @ got.V.T) / np.linalg.norm(A))
    assert worst_val <= 1e-10 and worst_rec < 1e-8


def test_eig_svd_rank_errors():
    from paper_1810_06860_b200.errors import RankDeficiencyError
    from paper_1810_06860_b200.linalg import eig_svd

    X = np.random.default_rng(0).standard_normal((20, 5))
    X[:, 4] = X[:, 0]
    with pytest.raises(RankDeficiencyError, match="eigenvalue"):
        eig_svd(X)
    with pytest.raises(RankDeficiencyError, match="no positive eigenvalue"):
        eig_svd(np.zeros((6, 3)))
    with pytest.raises(ValueError):
        eig_svd(np.ones((2, 4)))


def test_orth_golden_and_rank_checks(golden):
    from paper_1810_06860_b200.errors import RankDeficiencyError
    from paper_1810_06860_b200.linalg import orth

    Q = orth(golden["orth_X"])
    Qr = golden["orth_Q"]
    assert rel(Q @ Q.T, Qr @ Qr.T) <= 1e-12
    assert rel(Q.T @ Q, np.eye(Q.shape[1])) <= 1e-13
    X = np.random.default_rng(0).standard_normal((20, 5))
    X[:, 4] = X[:, 0]
    with pytest.raises(RankDeficiencyError):
        orth(X)
    with pytest.raises(RankDeficiencyError, match="zero matrix"):
        orth(np.zeros((10, 3)))
    # an ill-conditioned Krylov-like block (cond ~ 1e10) still orthonormalizes
    rng = np.random.default_rng(7)
    U, _ = np.linalg.qr(rng.standard_normal((3000, 40)))
    W, _ = np.linalg.qr(rng.standard_normal((40, 40)))
    Xc = (U * np.logspace(0, -10, 40)) @ W
    Q = orth(Xc)
    assert rel(Q.T @ Q, np.eye(40)) <= 1e-12
    assert np.linalg.norm(Q @ (Q.T @ U) - U) <= 1e-6 * np.sqrt(40)


def test_oracle_svd_matches_lapack(golden):
    from paper_1810_06860_b200.linalg import oracle_svd

    r = oracle_svd(golden["eig_A"])
    assert rel(r.S, golden["osvd_S"]) <= 1e-12
    assert rel((r.U * r.S) @ r.V.T, golden["eig_A"]) <= 1e-12
    rw = oracle_svd(golden["eig_A"].T)  # wide input
    assert rel(rw.S, golden["osvd_S"]) <= 1e-12
    assert rel((rw.U * rw.S) @ rw.V.T, golden["eig_A"].T) <= 1e-12
    # rank-deficient input: orthonormal U, and every singular value -- the null
    # one included -- to dgesdd's absolute accuracy (the Gram route alone
    # resolves it only to ~sqrt(eps) * s_max)
    X = np.random.default_rng(4).standard_normal((50, 6))
    X[:, 5] = X[:, 1]
    r = oracle_svd(X)
    S_ref = np.linalg.svd(X, compute_uv=False)
    assert rel(r.U.T @ r.U, np.eye(6)) <= 1e-12
    assert np.max(np.abs(r.S - S_ref)) <= 1e-12 * S_ref[0]
    assert r.S[-1] <= 1e-14 * r.S[0]
    assert rel((r.U * r.S) @ r.V.T, X) <= 1e-13
    # a tall block with exactly dependent columns (the BKI fallback's case): the
    # noise-level columns need not converge among themselves
    rng4 = np.random.default_rng(5)
    Xt = rng4.standard_normal((60000, 40))
    Xt[:, 30:] = Xt[:, :10] * 3.0
    r = oracle_svd(Xt)
    S_ref = np.linalg.svd(Xt, compute_uv=False)
    assert np.max(np.abs(r.S - S_ref)) <= 1e-12 * S_ref[0]
    assert rel(r.U.T @ r.U, np.eye(40)) <= 1e-12 and rel(r.V.T @ r.V, np.eye(40)) <= 1e-12
    assert rel((r.U * r.S) @ r.V.T, Xt) <= 1e-13
    # graded spectrum down to 1e-14 s_max, tall and wide
    rng = np.random.default_rng(9)
    Uq, _ = np.linalg.qr(rng.standard_normal((400, 30)))
    Wq, _ = np.linalg.qr(rng.standard_normal((30, 30)))
    Xg = (Uq * np.logspace(0, -14, 30)) @ Wq.T
    for M in (Xg, Xg.T):
        r = oracle_svd(M)
        S_ref = np.linalg.svd(M, compute_uv=False)
        assert np.max(np.abs(r.S - S_ref)) <= 1e-13 * S_ref[0]
        assert rel(r.U.T @ r.U, np.eye(30)) <= 1e-12 and rel(r.V.T @ r.V, np.eye(30)) <= 1e-12
        assert rel((r.U * r.S) @ r.V.T, M) <= 1e-13


def test_device_gaussian_matches_host():
    from paper_1810_06860_b200 import device
    from paper_1810_06860_b200.rng import RngState, gaussian_matrix, gaussian_matrix_device

    for seed, rows, cols in ((0, 1, 1), (5, 4, 3), (7, 37, 11), (2**62 + 7, 1001, 65), (12345, 50000, 110)):
        host = gaussian_matrix(RngState(seed), rows, cols)
        dev = device.to_host(gaussian_matrix_device(seed, rows, cols))
        # uniform words are bit-exact; log/sincos differ by a few ulp
        np.testing.assert_allclose(dev, host, rtol=4e-15, atol=4e-15)


def _patterns():
    rng = np.random.default_rng(11)
    yield "uniform", 3000, 2000, rng.choice(3000 * 2000, 40000, replace=False)
    yield "tiny", 1, 1, np.array([0])
    yield "empty rows/cols", 500, 700, rng.choice(250 * 700, 3000, replace=False) * 2 % (500 * 700)
    # long rows (> SPLIT_CHUNK) and a dense column
    rows = np.r_[np.full(1500, 7), np.arange(0, 900, 1), rng.integers(0, 900, 4000)]
    cols = np.r_[np.arange(1500), np.full(900, 3), rng.integers(0, 1600, 4000)]
    yield "long rows", 900, 1600, np.unique(rows * 1600 + cols)
    # Zipf-ish columns
    z = np.minimum(rng.zipf(1.3, 60000), 5000) - 1
    r = rng.integers(0, 20000, 60000)
    yield "zipf cols", 20000, 5000, np.unique(r * 5000 + z)


@pytest.mark.parametrize("case", list(range(5)))
def test_device_transpose_matches_host_stable_argsort(case):
    """The CSC built on the device (lr_csr_transpose_i32) is bit-identical to
    the reference's host transpose index (stable argsort, sparse.py:129-139)."""
    from paper_1810_06860_b200 import device
    from paper_1810_06860_b200.sparse import SparseMatrix

    name, m, n, flat = list(_patterns())[case]
    flat = np.asarray(flat, dtype=np.int64)
    i, j = np.divmod(flat, n)
    A = SparseMatrix.from_coo(m, n, i, j, np.arange(flat.size, dtype=np.float64) + 0.5)
    dp = A.pattern()
    perm, t_ptr, t_idx = A._transpose_index()
    assert np.array_equal(device.to_host(dp.csc.ptr), t_ptr), name
    assert np.array_equal(device.to_host(dp.csc.idx)[:A.nnz], t_idx), name
    assert np.array_equal(device.to_host(dp.perm)[:A.nnz], perm), name
    inv = np.empty(A.nnz, dtype=np.int64)
    inv[perm] = np.arange(A.nnz)
    assert np.array_equal(device.to_host(dp.inv_perm)[:A.nnz], inv), name
    vc, vt = A.device_values()
    assert np.array_equal(device.to_host(vt)[:A.nnz], A.data[perm]), name


@pytest.mark.parametrize("w", [2, 3, 16, 45, 110, 300])
def test_spmm_f32_matches_rounded_product(w):
    """fp32 mode kernel: against the fp64 product of the fp32-rounded inputs,
    within fp32 accumulation error (long rows and split items included)."""
    import torch

    from paper_1810_06860_b200 import device
    from paper_1810_06860_b200.sparse import SparseMatrix, spmm_dev32, spmm_t_dev32

    m, n = 700, 1300
    i, j, v = rand_pattern(m, n, 20000, seed=w, long_rows=2, long_cols=1)
    A = SparseMatrix.from_coo(m, n, i, j, v)
    P = oracle.csr_from_triples(m, n, i, j, v)
    P32 = oracle.csr_from_triples(m, n, i, j, np.asarray(v, dtype=np.float32).astype(np.float64))
    rng = np.random.default_rng(200 + w)
    X = rng.standard_normal((n, w)).astype(np.float32)
    H = rng.standard_normal((m, w)).astype(np.float32)
    Y32 = spmm_dev32(A, device.to_f32(device.to_device(X.astype(np.float64))))
    Yt32 = spmm_t_dev32(A, device.to_f32(device.to_device(H.astype(np.float64))))
    assert Y32.dtype == torch.float32 and Yt32.dtype == torch.float32
    ref = oracle.csr_times_dense(P32, X.astype(np.float64))
    ref_t = oracle.csr_t_times_dense(P32, H.astype(np.float64))
    got = device.to_host(device.to_f64(Y32))
    got_t = device.to_host(device.to_f64(Yt32))
    assert np.linalg.norm(got - ref) <= 2e-6 * np.linalg.norm(ref)
    assert np.linalg.norm(got_t - ref_t) <= 2e-6 * np.linalg.norm(ref_t)


def test_convert_roundtrip_and_rounding():
    from paper_1810_06860_b200 import device

    x = np.random.default_rng(3).standard_normal((37, 29)) * 1e3
    d = device.to_device(x)
    f = device.to_f32(d)
    back = device.to_host(device.to_f64(f))
    np.testing.assert_array_equal(back, x.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("r", [1, 3, 5, 9, 17, 24, 33, 48, 65, 84, 130, 200, 256])
def test_sddmm_group_kernel_matches_flat(r):
    """The line-aligned group kernel behind lr_sddmm_f64 / lr_svt_step_f64 (the
    product default) against the flat kernel (lr_sddmm_flat_f64 /
    lr_svt_step_flat_f64) and numpy: sampled entries and updated values of Y
    agree to rounding (bit-identical where the two lane maps coincide; the
    group kernel fits its map to r) -- on rows split into items, empty rows
    and a Zipf-like long row."""
    import torch

    from paper_1810_06860_b200 import _native, device
    from paper_1810_06860_b200.sparse import SparseMatrix

    m, n = 1500, 900
    i, j, v = rand_pattern(m, n, 60000, seed=700 + r, long_rows=2)
    A = SparseMatrix.from_coo(m, n, i, j, v)
    dp = A.pattern()
    rng = np.random.default_rng(r)
    U = device.to_device(rng.standard_normal((m, r)))
    V = device.to_device(rng.standard_normal((n, r)))
    S = device.f64_buffer(rng.random(r) + 0.5)
    st = device.stream()
    x_flat, x_grp = device.vector(A.nnz), device.vector(A.nnz)
    _native.call("lr_sddmm_flat_f64", device.ptr(dp.csr.ptr), device.ptr(dp.csr.idx), m, A.nnz,
                 device.ptr(dp.tile_rows()), device.ptr(U), device.ld(U), device.ptr(S), device.ptr(V), device.ld(V),
                 r, device.ptr(x_flat), st)
    _native.call("lr_sddmm_f64", device.ptr(dp.csr.ptr), device.ptr(dp.csr.idx), m, device.ptr(dp.csr.items),
                 dp.csr.n_items, device.ptr(U), device.ld(U), device.ptr(S), device.ptr(V), device.ld(V), r,
                 device.ptr(x_grp), st)
    ref = np.einsum("er,er->e", device.to_host(U)[A.coo_rows()] * device.to_host(S), device.to_host(V)[A.indices])
    assert rel(device.to_host(x_grp), ref) <= 1e-14
    assert rel(device.to_host(x_flat), device.to_host(x_grp)) <= 1e-14
    # fused step through both entry points: identical Y
    m_vals = A.device_values()[0]
    ys = []
    for name in ("lr_svt_step_flat_f64", "lr_svt_step_f64"):
        y = m_vals.clone()
        npart = int(_native.load().lr_svt_flat_partials() if "flat" in name else _native.load().lr_svt_step_partials())
        part, out2 = device.vector(npart + 8), device.vector(2)
        if "flat" in name:
            _native.call(name, device.ptr(dp.csr.ptr), device.ptr(dp.csr.idx), m, A.nnz, device.ptr(dp.tile_rows()),
                         device.ptr(U), device.ld(U), device.ptr(S), device.ptr(V), device.ld(V), r,
                         device.ptr(m_vals), device.ptr(y), None, device.ptr(dp.inv_perm), 0.37, 1, device.ptr(part),
                         npart, device.ptr(out2), st)
        else:
            _native.call(name, device.ptr(dp.csr.ptr), device.ptr(dp.csr.idx), m, device.ptr(dp.csr.items),
                         dp.csr.n_items, device.ptr(U), device.ld(U), device.ptr(S), device.ptr(V), device.ld(V), r,
                         device.ptr(m_vals), device.ptr(y), None, device.ptr(dp.inv_perm), 0.37, 1, device.ptr(part),
                         npart, device.ptr(out2), st)
        ys.append((y, float(np.sqrt(device.to_host(out2)[0]))))
    assert rel(device.to_host(ys[0][0]), device.to_host(ys[1][0])) <= 1e-15
    assert abs(ys[0][1] - ys[1][1]) <= 1e-13 * ys[0][1]


@pytest.mark.parametrize("m,n,nnz,long_rows,empty_tail,r", [
    (300, 200, 4000, 0, 0, 1), (300, 200, 4000, 2, 0, 5), (1000, 700, 30000, 3, 40, 17),
    (5000, 3000, 200000, 1, 0, 48), (700, 600, 50000, 0, 100, 84), (400, 900, 60000, 2, 0, 300),
    (2000, 1500, 100000, 0, 0, 1100)])
def test_svt_step_flat_matches_oracle_and_refreshes_csc(m, n, nnz, long_rows, empty_tail, r):
    """The fused SVT step of the product (DeviceEngine.step -> lr_svt_step_f64,
    the line-aligned group kernel; the flat kernel is bit-identical to it):
    residual and updated values against a numpy restatement of
    completion.py:373-386, the CSC copy refreshed on demand (lr_gather_f64)
    against the updated CSR values through the reference's stable argsort,
    patterns with empty rows (a tail of empty rows and scattered ones), dense
    rows, and ranks on both sides of the one-chunk limit (256) and of the
    round-1 kernels' 1024 limit."""
    import torch

    from paper_1810_06860_b200 import completion, device
    from paper_1810_06860_b200.sparse import ObservationSet

    i, j, v = rand_pattern(m, n, nnz, seed=m + r, long_rows=long_rows)
    keep = i < m - empty_tail
    i, j, v = i[keep], j[keep], v[keep]
    eng = completion.DeviceEngine(ObservationSet(m, n, i, j, v))
    eng.m_norm = eng.observed_norm()
    eng.start(1.7)
    rng = np.random.default_rng(r)
    U, V, S = rng.standard_normal((m, r)), rng.standard_normal((n, r)), rng.random(r) + 0.5
    y0 = eng.Y.data.copy()
    resid, deferred = eng.step(device.to_device(U), S, device.to_device(V), r, 0.37)
    assert deferred is None
    order = np.lexsort((j, i))
    ii, jj, mm = i[order], j[order], v[order]
    x = np.einsum("er,er->e", U[ii] * S, V[jj])
    assert abs(resid - np.linalg.norm(x - mm) / np.linalg.norm(mm)) <= 1e-12 * max(resid, 1e-300)
    y_ref = y0 + 0.37 * (mm - x)
    y_dev = eng.Y.data
    assert rel(y_dev, y_ref) <= 1e-13
    yc, yt = eng.Y.device_values()  # CSC refresh
    tperm = np.argsort(jj, kind="stable")
    assert np.array_equal(device.to_host(yt), device.to_host(yc)[tperm])
    assert torch.equal(yc.cpu(), torch.from_numpy(y_dev))


@pytest.mark.parametrize("m,n,nnz,long_rows,shuffle", [(1, 1, 1, 0, False), (300, 200, 4000, 0, True),
                                                       (2000, 9000, 60000, 2, True), (50, 5000, 0, 1, True),
                                                       (5000, 3000, 200000, 0, True)])
def test_coo_to_csr_device_matches_host_lexsort(m, n, nnz, long_rows, shuffle):
    """SparseMatrix.from_coo_device (lr_coo_to_csr_i32) against the host
    lexsort build (sparse.py:84-104): indptr, indices and values bit-exact,
    incl. empty rows and dense rows longer than the shared-memory sort (9000
    columns), entries in arbitrary input order; the split-tag selection of
    ObservationSet.train_matrix; the device values and the CSC transpose built
    from the device pattern."""
    import torch

    from paper_1810_06860_b200 import device
    from paper_1810_06860_b200.sparse import ObservationSet, SparseMatrix

    i, j, v = rand_pattern(m, n, nnz, seed=m + n, long_rows=long_rows)
    if shuffle:
        p = np.random.default_rng(1).permutation(i.size)
        i, j, v = i[p], j[p], v[p]
    H = SparseMatrix.from_coo(m, n, i, j, v)
    D = SparseMatrix.from_coo_device(m, n, i, j, v)
    assert D._dev_csr is not None
    assert np.array_equal(D.indptr, H.indptr)
    assert np.array_equal(D.indices, H.indices)
    assert np.array_equal(D.data, H.data)
    vc, vt = D.device_values()
    assert np.array_equal(device.to_host(vc), H.data)
    tperm, _, _ = H._transpose_index()
    assert np.array_equal(device.to_host(vt), H.data[tperm])
    assert torch.equal(D.pattern().csc.idx[:H.nnz].cpu(), H.pattern().csc.idx[:H.nnz].cpu())
    split = (np.random.default_rng(2).random(i.size) < 0.3).astype(np.uint8)
    obs = ObservationSet(m, n, i, j, v, split)
    T = obs.train_matrix()
    r, c, vv = obs.subset(0)
    ref = SparseMatrix.from_coo(m, n, r, c, vv)
    assert np.array_equal(T.indptr, ref.indptr) and np.array_equal(T.indices, ref.indices)
    assert np.array_equal(T.data, ref.data)


def test_coo_to_csr_device_errors():
    """The device build raises what the host build raises: out-of-range
    coordinates, the first duplicate cell in (row, col) order, non-finite
    values."""
    from paper_1810_06860_b200.errors import DataError
    from paper_1810_06860_b200.sparse import SparseMatrix

    with pytest.raises(DataError, match="out of range"):
        SparseMatrix.from_coo_device(3, 3, [0, 3], [0, 1], [1.0, 2.0])
    with pytest.raises(DataError, match="out of range"):
        SparseMatrix.from_coo_device(3, 3, [0, 1], [0, -1], [1.0, 2.0])
    i = [2, 0, 2, 1, 0, 1]
    j = [1, 2, 1, 0, 2, 2]
    with pytest.raises(DataError) as eh:
        SparseMatrix.from_coo(3, 3, i, j, np.arange(6.0))
    with pytest.raises(DataError) as ed:
        SparseMatrix.from_coo_device(3, 3, i, j, np.arange(6.0))
    assert str(ed.value) == str(eh.value) == "duplicate entry at (0, 2)"
    with pytest.raises(DataError, match="finite"):
        SparseMatrix.from_coo_device(3, 3, [0, 1], [0, 1], [1.0, np.inf])


def test_observation_set_device_validation_matches_host():
    """ObservationSet validates on the device when one is present (the
    duplicate search of each split through lr_coo_to_csr_i32) and raises the
    reference's errors in the reference's order (sparse.py:259-328); the train
    split's device CSR is handed to train_matrix() once."""
    from paper_1810_06860_b200 import device
    from paper_1810_06860_b200.errors import DataError
    from paper_1810_06860_b200.sparse import ObservationSet, SparseMatrix

    assert device.cuda_ready()
    rows, cols = np.array([0, 1, 2, 1, 0]), np.array([1, 2, 0, 2, 1])
    vals = np.arange(5.0)
    # (0, 1) twice: in the same split -> error; across splits -> fine
    with pytest.raises(DataError, match="duplicate \\(row, col\\) within train split"):
        ObservationSet(3, 3, rows[:2].tolist() + [0], cols[:2].tolist() + [1], vals[:3])
    with pytest.raises(DataError, match="within test split"):
        ObservationSet(3, 3, [0, 0, 2], [1, 1, 0], vals[:3], np.array([1, 1, 0], dtype=np.uint8))
    ok = ObservationSet(3, 3, [0, 0, 2], [1, 1, 0], vals[:3], np.array([0, 1, 0], dtype=np.uint8))
    T = ok.train_matrix()
    assert T.indptr.tolist() == [0, 1, 1, 2] and T.indices.tolist() == [1, 0] and T.data.tolist() == [0.0, 2.0]
    T2 = ok.train_matrix()  # a fresh build the second time
    assert T2 is not T and np.array_equal(T2.data, T.data)
    with pytest.raises(DataError, match="row index out of range"):
        ObservationSet(3, 3, [0, 3], [0, 9], [1.0, 2.0])
    with pytest.raises(DataError, match="col index out of range"):
        ObservationSet(3, 3, [0, 1], [0, 9], [1.0, 2.0])
    with pytest.raises(DataError, match="finite"):
        ObservationSet(3, 3, [0, 1], [0, 1], [1.0, np.nan])
    with pytest.raises(DataError, match="split tags"):
        ObservationSet(3, 3, [0, 1], [0, 1], [1.0, 2.0], np.array([0, 2], dtype=np.uint8))
    assert isinstance(T, SparseMatrix)


@pytest.mark.parametrize("K,n", [(1, 1), (37, 5), (3, 260), (1000, 128), (5000, 129), (20000, 300),
                                 (100000, 660), (300001, 40)])
def test_gram_tf32x3_tensor_core(K, n):
    """fp32 mode's eigSVD Gram on tcgen05 (kind::tf32, 3xTF32): within 1e-5
    of the fp64 Gram of the same fp32 values, entrywise relative to
    sqrt(G_ii G_jj) (the Cauchy-Schwarz scale of G_ij); exactly symmetric;
    bitwise reproducible (fixed-order chunk sum)."""
    from paper_1810_06860_b200 import device, linalg

    rng = np.random.default_rng(K + 7 * n)
    A = rng.standard_normal((K, n)) * rng.uniform(0.01, 100.0, size=n)
    A32 = device.to_f32(device.to_device(A))
    G = device.to_host(linalg.gram_tf32x3_dev(A32))
    G2 = device.to_host(linalg.gram_tf32x3_dev(A32))
    A64 = device.to_host(A32).astype(np.float64)
    ref = A64.T @ A64
    scale = np.sqrt(np.outer(np.diag(ref), np.diag(ref)))
    err = float(np.max(np.abs(G - ref) / scale))
    assert err < 1e-5, err
    assert np.array_equal(G, G.T)
    assert np.array_equal(G, G2)


@pytest.mark.parametrize("n,w_lo,w_hi", [(2677, 7, 15), (26744, 20, 28), (1000, 6, 6), (333, 1, 9)])
def test_omega_assembled_on_device_from_superset_is_bit_exact(n, w_lo, w_hi, monkeypatch):
    """The parity Omega through the device assembly (rng.Superset's Box-Muller
    halves uploaded once, lr_omega_assemble_f64 forming each width: one IEEE
    multiply per entry) against the reference draw (numpy, rng.py:38-55),
    bit for bit for every width in the range; a width outside the range takes
    the host draw."""
    from paper_1810_06860_b200 import _native, device, rng, rsvd

    seed = 1234567 + n
    rng._SUPERSETS.clear()
    rng._PREFETCH.clear()
    monkeypatch.setattr(rng, "SUPERSET_ON_DEVICE", True)  # opt-in (LR_SUPERSET_DEVICE=1)
    rng.prefetch_superset(seed, n, w_lo, w_hi)
    calls = []
    real = _native.call
    monkeypatch.setattr(_native, "call", lambda name, *a, **k: (calls.append(name), real(name, *a, **k))[1])
    for w in sorted({w_lo, (w_lo + w_hi) // 2, w_hi}):
        rng.prefetch_normals(seed, n, w)  # what the SVT loop calls once the rank is known: nothing to draw
        assert (seed, n, w) not in rng._PREFETCH
        del calls[:]
        Om = rsvd.omega_from_host(seed, n, w)
        assert calls == ["lr_omega_assemble_f64"]
        ref = rng.gaussian_matrix(rng.RngState(seed), n, w)
        assert np.array_equal(device.to_host(Om), ref)
    del calls[:]
    Om = rsvd.omega_from_host(seed, n, w_hi + 1)
    assert "lr_omega_assemble_f64" not in calls
    assert np.array_equal(device.to_host(Om), rng.gaussian_matrix(rng.RngState(seed), n, w_hi + 1))
