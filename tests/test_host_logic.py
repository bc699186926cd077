"""Host-side logic that runs without a GPU: argument validation with the
reference's error types (completion.py:44-88, rsvd.py RsvdParams,
sparse.py:84-104 / :200-246), the SpMM work-item schedule, the Gram-spectrum
rank checks (linalg.py:190-198), and the loud failure of the product path
when no CUDA device is present (no CPU fallback)."""

import numpy as np
import pytest
import torch

from paper_1810_06860_b200 import completion, linalg, rsvd, sparse, workloads
from paper_1810_06860_b200.errors import DataError, RankDeficiencyError
from paper_1810_06860_b200.sparse import SparseMatrix


@pytest.mark.parametrize("kw", [dict(tau=0.0), dict(delta=-1.0), dict(l=0), dict(epsilon=1.0), dict(epsilon=0.0),
                                dict(i_max=0), dict(i_reuse=0), dict(q_reuse=-1), dict(strategy="nope"),
                                dict(p0=0), dict(p_min=0), dict(s=-1), dict(precision="bf16")])
def test_svt_params_reject(kw):
    with pytest.raises(ValueError):
        completion.SvtParams(**kw)


def test_svt_params_defaults():
    p = completion.SvtParams()
    assert (p.l, p.epsilon, p.i_max, p.i_reuse, p.q_reuse, p.strategy, p.p0, p.p_min, p.s) == \
        (5, 0.05, 500, 100, 10, "none", 3, 1, 5)
    assert p.tau is None and p.delta is None and p.precision == "fp64"
    assert completion.SvtParams(precision="fp32").precision == "fp32"


@pytest.mark.parametrize("kw", [dict(k=0, p=1), dict(k=3, p=-1), dict(k=3, p=1, s=-1)])
def test_rsvd_params_reject(kw):
    with pytest.raises(ValueError):
        rsvd.RsvdParams(**kw)


def test_rsvd_params_width_check():
    A = SparseMatrix.from_coo(20, 12, [0, 1], [0, 1], [1.0, 2.0])
    rsvd.RsvdParams(k=2, p=1, s=1).check_against(A, krylov=True)  # (2+1)*2 = 6 <= 12
    with pytest.raises(ValueError, match="sketch width"):
        rsvd.RsvdParams(k=3, p=2, s=2).check_against(A, krylov=True)  # 15 > 12
    rsvd.RsvdParams(k=3, p=2, s=2).check_against(A, krylov=False)  # 5 <= 12


def test_sparse_validation():
    with pytest.raises(DataError):
        SparseMatrix(0, 3, [0], [], [])
    with pytest.raises(DataError):
        SparseMatrix(2, 3, [0, 1], [0], [1.0])  # indptr length
    with pytest.raises(DataError):
        SparseMatrix(2, 3, [0, 2, 1], [0, 1], [1.0, 1.0])  # not monotone
    with pytest.raises(DataError):
        SparseMatrix(2, 3, [0, 1, 2], [0, 3], [1.0, 1.0])  # column out of range
    with pytest.raises(DataError):
        SparseMatrix(1, 3, [0, 2], [1, 1], [1.0, 1.0])  # not strictly increasing
    with pytest.raises(DataError):
        SparseMatrix(1, 3, [0, 1], [1], [np.nan])
    # a new row may restart at a smaller column
    SparseMatrix(2, 3, [0, 2, 3], [1, 2, 0], [1.0, 2.0, 3.0])
    # empty pattern is legal
    SparseMatrix(2, 3, [0, 0, 0], [], [])


def test_from_coo_sorts_and_rejects_duplicates():
    A = SparseMatrix.from_coo(3, 3, [2, 0, 0], [1, 2, 0], [5.0, 2.0, 1.0])
    assert A.indptr.tolist() == [0, 2, 2, 3]
    assert A.indices.tolist() == [0, 2, 1]
    with pytest.raises(DataError):
        SparseMatrix.from_coo(3, 3, [1, 1], [2, 2], [1.0, 1.0])
    with pytest.raises(DataError):
        SparseMatrix.from_coo(3, 3, [3], [0], [1.0])


def _check_schedule(indptr, chunk):
    items, splits, n_slots = sparse._schedule(indptr, chunk)
    lens = np.diff(indptr)
    if items is None:
        assert lens.max(initial=0) <= chunk
        return
    # every stored entry is covered by exactly one item
    cover = np.zeros(int(indptr[-1]), dtype=np.int64)
    for r, b, e, s in items:
        assert indptr[r] <= b < e <= indptr[r + 1] or b == e == indptr[r]
        cover[b:e] += 1
    assert (cover == 1).all()
    # long rows own consecutive split slots, short rows write their row directly
    slots = sorted(int(s) for s in items[:, 3] if s >= 0)
    assert slots == list(range(n_slots))
    for r, sb, se, _ in splits:
        assert lens[r] > chunk and se - sb == -(-lens[r] // chunk)
    # longest first
    w = items[:, 2] - items[:, 1]
    assert (np.diff(w) <= 0).all()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_spmm_schedule_covers_pattern(seed):
    rng = np.random.default_rng(seed)
    lens = np.minimum(rng.zipf(1.6, size=500), 3000)
    lens[::37] = 0  # empty rows
    indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    for chunk in (32, 64, 256):
        _check_schedule(indptr, chunk)


def test_spmm_schedule_chunk_size():
    indptr = np.arange(0, 1001 * 200, 200, dtype=np.int64)  # cfg1: 1000 rows of 200
    assert sparse._chunk_for(indptr) == sparse.MIN_CHUNK
    big = np.array([0, 10**9], dtype=np.int64)
    assert sparse._chunk_for(big) == sparse.SPLIT_CHUNK


def test_gram_spectrum_rank_checks():
    d = np.array([1e-3, 0.5, 4.0])
    assert np.allclose(linalg.gram_spectrum(d), np.sqrt(d))
    with pytest.raises(RankDeficiencyError):
        linalg.gram_spectrum(np.array([-1.0, 0.0]))
    with pytest.raises(RankDeficiencyError):
        linalg.gram_spectrum(np.array([0.0, 1.0, 4.0]))


def test_workloads_deterministic():
    a, _ = workloads.cfg1_small()
    b, _ = workloads.cfg1_small()
    assert (a.rows == b.rows).all() and (a.cols == b.cols).all() and (a.values == b.values).all()
    assert a.rows.max() < a.m and a.cols.max() < a.n


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_product_path_fails_loudly_without_cuda():
    A = SparseMatrix.from_coo(30, 20, np.arange(20), np.arange(20), np.ones(20))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rsvd.rsvd_bki(A, rsvd.RsvdParams(k=2, p=1, s=1))
    o, _ = workloads.cfg1_small()
    obs = sparse.ObservationSet(o.m, o.n, o.rows, o.cols, o.values)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        completion.svt_fast(obs, completion.SvtParams(i_max=1))


def test_split_observations_matches_reference():
    """workloads.split_observations (cfg4's holdout) against the REAL
    reference's ingest.split_observations tags (tests/golden/make_golden_r02.py)."""
    import os

    from paper_1810_06860_b200 import workloads
    from paper_1810_06860_b200.rng import RngState

    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden_r02.npz"))
    for count, frac, seed in ((1000, 0.9, 0), (777, 0.8, 42)):
        got = workloads.split_observations(count, frac, RngState(seed))
        assert np.array_equal(got, g[f"split_{count}_{seed}"])
    with pytest.raises(ValueError, match="train fraction"):
        workloads.split_observations(10, 1.0, RngState(0))
    with pytest.raises(ValueError, match="empty split"):
        workloads.split_observations(3, 0.01, RngState(0))


@pytest.mark.parametrize("rows,cols,seed", [(50000, 110, 7), (37, 11, 3), (1001, 3, 5), (1, 1, 9),
                                            (26744, 65, 2 ** 62 + 11)])
def test_threaded_gaussian_is_bit_exact(rows, cols, seed):
    """The threaded host Omega (rng.normals_column_major, the parity default's
    producer) equals the one-thread reference draw bit for bit on this host,
    and leaves the stream where the one-thread draw leaves it."""
    from paper_1810_06860_b200 import rng as R

    ref = R.gaussian_matrix(R.RngState(seed), rows, cols)
    st = R.RngState(seed)
    got = R.gaussian_matrix_fast(st, rows, cols)
    assert np.array_equal(got, ref)
    z = R.normals_column_major(seed, rows, cols)
    assert np.array_equal(z.reshape(cols, rows).T, ref)
    st2 = R.RngState(seed)
    R.gaussian_matrix(st2, rows, cols)
    assert st.position == st2.position and np.array_equal(st.uniform(7), st2.uniform(7))


@pytest.mark.parametrize("rows,cols,seed", [(1, 1, 0), (7, 3, 5), (26744, 55, 2**62 + 9), (50000, 110, 123)])
def test_c_uniforms_and_box_muller_are_bit_exact(rows, cols, seed):
    """The C pieces of the host draw (csrc/lr_host_rng.c: Philox uniforms,
    Box-Muller with libm cos/sin; numpy's own log in between) reproduce the
    reference's all-numpy draw (rng.py:38-55) bit for bit on this host, and the
    library is the producer the parity Omega uses here."""
    from paper_1810_06860_b200 import _native
    from paper_1810_06860_b200 import rng as R

    if not __import__("os").path.exists(_native.LIB_PATH):
        pytest.fail(f"native library not built: {_native.LIB_PATH} (run make)")
    lib = R._c_draw_lib()
    assert lib, "C draw failed its self-check against numpy on this host"
    ref = R.RngState(seed).normal_pairs(rows * cols)
    assert np.array_equal(R._normals_c(lib, seed, rows, cols), ref)
    assert np.array_equal(R._normals_c(lib, seed, rows, cols, pool=R._pool()), ref)
    u = np.empty(11)
    lib.lr_host_uniforms(seed & ((1 << 64) - 1), 5, 11, u.ctypes.data)
    assert np.array_equal(u, R.RngState(seed).uniform(16)[5:])


@pytest.mark.parametrize("rows,w_lo,w_hi", [(1, 1, 3), (7, 2, 9), (26744, 9, 17), (1001, 1, 40)])
def test_superset_draw_is_bit_exact(rows, w_lo, w_hi):
    """rng.Superset (one draw serving every width in [w_lo, w_hi]) gives, for
    each width, exactly the one-width draw of the reference (rng.py:38-55)."""
    from paper_1810_06860_b200 import rng as R

    lib = R._c_draw_lib()
    assert lib
    seed = 2 ** 40 + rows
    sup = R.Superset(lib, seed, rows, w_lo, w_hi, R._pool())
    for w in range(w_lo, w_hi + 1):
        ref = R.RngState(seed).normal_pairs(rows * w)
        out = np.empty(rows * w + 1)
        assert np.array_equal(sup.normals(w, out, R._pool()), ref), w


def test_factor_container_matches_reference_format(tmp_path):
    """write_factors / read_factors: the reference's LRFC bytes
    (completion.py:449-492: magic, version, m n r, U S V little-endian),
    checked against the real reference's writer when it is importable, and its
    DataError cases."""
    import os
    import sys

    rng = np.random.default_rng(0)
    res = completion.CompletionResult(U=rng.standard_normal((7, 3)), S=np.array([3.0, 2.0, 1.0]),
                                      V=rng.standard_normal((5, 3)), rank=3, iterations=1, converged=True,
                                      residual=0.1, trace=[], events=[], svd_time=0.0, update_time=0.0,
                                      total_time=0.0)
    p = tmp_path / "f.bin"
    completion.write_factors(str(p), res)
    U, S, V = completion.read_factors(str(p))
    assert np.array_equal(U, res.U) and np.array_equal(S, res.S) and np.array_equal(V, res.V)
    ref_src = "/root/reference/pkg/src"
    if os.path.isdir(ref_src):
        sys.path.insert(0, ref_src)
        try:
            from lowrank import completion as rc

            q = tmp_path / "ref.bin"
            rc.write_factors(str(q), res)
            assert q.read_bytes() == p.read_bytes()
        finally:
            sys.path.remove(ref_src)
    raw = p.read_bytes()
    for bad, msg in ((b"XXXX" + raw[4:], "not a factor container"), (raw[:20], "truncated in header"),
                     (raw[:-8], "truncated"), (raw + b"\0", "trailing bytes")):
        q = tmp_path / "bad.bin"
        q.write_bytes(bad)
        with pytest.raises(DataError, match=msg):
            completion.read_factors(str(q))


def test_cfg5_device_generator_shape_and_pattern():
    """workloads.cfg5_device (run here on the CPU generator): distinct,
    row-major sorted in-range positions, the requested count, finite values
    of the rank-r product's scale."""
    from paper_1810_06860_b200 import workloads

    o = workloads.cfg5_device(seed=1, m=3000, n=700, nnz=50000, rank=7, noise=0.01, device="cpu")
    key = o.rows * o.n + o.cols
    assert o.rows.size == 50000 and np.all(np.diff(key) > 0)
    assert o.rows.min() >= 0 and o.rows.max() < 3000 and o.cols.min() >= 0 and o.cols.max() < 700
    assert np.all(np.isfinite(o.values)) and 1.5 < np.std(o.values) < 4.5  # var = rank


def test_superset_after_escalation_covers_the_next_calls(monkeypatch):
    """completion._speculate_after_escalation: after an escalation k_old ->
    k_new the call after the redo (svd_calls + 2) is iteration i+1's first
    call at k = r + 1, r in [k_old, k_new - 1], or another escalation at
    k_new + l: one Superset over widths [k_old + 1 + s, k_new + l + s] with
    that call's seed; nothing when a width would exceed the BKI width budget
    or the draws are not on the host."""
    from paper_1810_06860_b200 import completion, rng

    calls = []
    monkeypatch.setattr(rng, "prefetch_superset", lambda seed, rows, lo, hi: calls.append((seed, rows, lo, hi)))

    class Eng:
        m, n, omega_source = 5000, 3000, "host"

    params = completion.SvtParams(seed=7)
    state = completion.SvtState(Y=None, seed_rng=rng.RngState(7))
    state.svd_calls = 4
    completion._speculate_after_escalation(state, params, "none", Eng(), 10, 10 + params.l)
    s, l = params.s, params.l
    assert calls == [(rng.RngState(7).spawn(6).seed, 3000, 11 + s, 10 + 2 * l + s)]
    del calls[:]
    Eng.omega_source = "device"
    completion._speculate_after_escalation(state, params, "none", Eng(), 10, 10 + l)
    assert calls == []
    Eng.omega_source = "host"
    # widths past the BKI budget (min_dim // (k + s) - 1 < 1) are left out; none left -> no draw
    completion._speculate_after_escalation(state, params, "none", Eng(), 1490, 1490 + l)
    assert calls == [(rng.RngState(7).spawn(6).seed, 3000, 1491 + s, 1500)]
    del calls[:]
    completion._speculate_after_escalation(state, params, "none", Eng(), 1600, 1600 + l)
    assert calls == []
