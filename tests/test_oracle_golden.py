"""Pin the CPU oracle (oracle/) against fixtures produced by the real reference.

tests/golden/make_golden.py generated reference_golden.npz by importing
/root/reference/pkg/src/lowrank.  Integer work (patterns, permutations,
seeds) must match exactly; the RNG must match bit for bit; floating results
to 1e-12 relative (same LAPACK/BLAS builds in this image), loop traces
iteration for iteration.
"""

import numpy as np
import pytest

import oracle
from oracle import dense, sketch, svt
from oracle.csr import sampled_product
from paper_1810_06860_b200 import workloads


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def test_rng_bitexact(golden):
    for seed in (0, 1, 2, 12345, 2**62 + 7):
        assert np.array_equal(oracle.Stream(seed).normals(257), golden[f"rng_normals_{seed}"])
        assert np.array_equal(oracle.Stream(seed).uniforms(64), golden[f"rng_uniform_{seed}"])
    assert np.array_equal(oracle.gaussian_block(oracle.Stream(5), 4, 3), golden["rng_gauss_5_4x3"])
    assert np.array_equal(oracle.gaussian_block(oracle.Stream(7), 37, 11), golden["rng_gauss_7_37x11"])
    seeds = [oracle.Stream(s).derive(t).seed for s in (0, 1, 99, 2**40) for t in (0, 1, 2, 17)]
    assert np.array_equal(np.array(seeds, dtype=np.uint64), golden["rng_spawn"])


def test_pattern_build_exact(golden):
    A = oracle.csr_from_triples(3, 4, [2, 0, 0], [1, 3, 0], [5.0, 6.0, 7.0])
    assert np.array_equal(A.offsets, golden["coo_small_indptr"])
    assert np.array_equal(A.cols, golden["coo_small_indices"])
    assert np.array_equal(A.vals, golden["coo_small_data"])
    A = oracle.csr_from_triples(60, 45, golden["sp_i"], golden["sp_j"], golden["sp_v"])
    assert np.array_equal(A.offsets, golden["sp_indptr"])
    assert np.array_equal(A.cols, golden["sp_indices"])
    assert np.array_equal(A.vals, golden["sp_data"])
    perm, tip, tix = A.transpose_index()
    assert np.array_equal(perm, golden["sp_tperm"])
    assert np.array_equal(tip, golden["sp_tindptr"])
    assert np.array_equal(tix, golden["sp_tindices"])
    with pytest.raises(ValueError, match="duplicate"):
        oracle.csr_from_triples(2, 2, [0, 0], [1, 1], [1.0, 2.0])


def test_sparse_kernels(golden):
    A = oracle.csr_from_triples(60, 45, golden["sp_i"], golden["sp_j"], golden["sp_v"])
    assert rel(oracle.csr_times_dense(A, golden["sp_X"]), golden["sp_spmm"]) < 1e-14
    assert rel(oracle.csr_t_times_dense(A, golden["sp_H"]), golden["sp_spmm_t"]) < 1e-14
    assert rel(sampled_product(golden["sp_U"], golden["sp_S"], golden["sp_V"], A), golden["sp_project"]) < 1e-14
    assert oracle.scaled_norm(A.vals) == float(golden["sp_frob"])
    assert oracle.scaled_norm(np.array([3.0, 4.0])) == float(golden["frob_345"]) == 5.0
    assert abs(oracle.spectral_estimate(A, oracle.Stream(3)) - float(golden["sp_norm2"])) < 1e-12


def test_dense_layer(golden):
    assert rel(oracle.householder_basis(golden["orth_X"]), golden["orth_Q"]) < 1e-12
    assert rel(oracle.pivoted_lower(golden["lu_X"]), golden["lu_PL"]) < 1e-12
    assert rel(oracle.pivoted_lower(golden["lu2_X"]), golden["lu2_PL"]) < 1e-12
    r = oracle.gram_svd(golden["eig_A"])
    assert r.order == "ascending"
    assert rel(r.S, golden["eig_S"]) < 1e-13
    assert rel(r.U, golden["eig_U"]) < 1e-10 and rel(r.V, golden["eig_V"]) < 1e-10
    r = oracle.dense_svd(golden["eig_A"])
    assert rel(r.S, golden["osvd_S"]) < 1e-13 and rel(r.U, golden["osvd_U"]) < 1e-10


def test_dense_errors():
    X = oracle.gaussian_block(oracle.Stream(0), 20, 5)
    X[:, 4] = X[:, 0]
    with pytest.raises(oracle.RankDeficient):
        oracle.householder_basis(X)
    with pytest.raises(oracle.RankDeficient):
        oracle.householder_basis(np.zeros((10, 3)))
    with pytest.raises(oracle.RankDeficient, match="eigenvalue"):
        oracle.gram_svd(X)
    with pytest.raises(ValueError):
        oracle.pivoted_lower(np.ones((3, 5)))


@pytest.mark.parametrize("name,fn", [("pi", sketch.sketch_pi), ("bki", sketch.sketch_bki), ("basic", sketch.sketch_basic)])
def test_sketches(golden, name, fn):
    A = oracle.csr_from_triples(300, 200, golden["rs_i"], golden["rs_j"], golden["rs_v"])
    res, basis = fn(A, sketch.SketchParams(k=10, p=2, s=5, seed=3))
    assert rel(res.S, golden[f"rs_{name}_S"]) < 1e-12
    assert rel(res.product(), (golden[f"rs_{name}_U"] * golden[f"rs_{name}_S"]) @ golden[f"rs_{name}_V"].T) < 1e-10
    assert rel(basis.Q @ basis.Q.T, golden[f"rs_{name}_Q"] @ golden[f"rs_{name}_Q"].T) < 1e-10
    assert abs(sketch.relative_fit_error(A, res) - float(golden[f"rs_{name}_qb"])) < 1e-12


def test_power_rule_fixture(golden):
    loop = svt._Loop(Y=None, p=3)
    got = [svt.run_power_rule(loop, e) for e in golden["power_errs"]]
    assert got == list(golden["power_p"]) == [3, 3, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 3, 4, 4, 4, 4, 4, 4, 4]


def _check_trace(out, golden, prefix, rtol=1e-9, upto=None):
    n = len(golden[prefix + "k"]) if upto is None else upto
    assert out.iterations >= n
    tr = out.trace[:n]
    assert [t[1] for t in tr] == list(golden[prefix + "k"][:n])
    assert [t[2] for t in tr] == list(golden[prefix + "r"][:n])
    assert [t[3] for t in tr] == list(golden[prefix + "p"][:n])
    assert [t[4] for t in tr] == list(golden[prefix + "q"][:n])
    assert [t[6] for t in tr] == list(golden[prefix + "source"][:n])
    np.testing.assert_allclose([t[5] for t in tr], golden[prefix + "residual"][:n], rtol=rtol)


@pytest.mark.parametrize("prefix,kw,backend", [
    ("svt_small_bki_", dict(epsilon=1e-3, seed=4), "rsvd-bki"),
    ("svt_small_oracle_", dict(epsilon=1e-3, seed=4), "oracle"),
    ("svt_small_rq2_", dict(epsilon=0.05, seed=7, strategy="reuse-q", i_reuse=10), "rsvd-bki"),
])
def test_svt_small_traces(golden, prefix, kw, backend):
    obs, _ = workloads.cfg1_small()
    strategy = kw.get("strategy", "none")
    out = oracle.complete(obs.m, obs.n, obs.rows, obs.cols, obs.values, oracle.SvtConfig(**kw),
                          backend=backend, strategy=strategy)
    _check_trace(out, golden, prefix)
    assert out.converged == bool(golden[prefix + "converged"])
    np.testing.assert_allclose(out.S, golden[prefix + "S"], rtol=1e-9)


def test_svt_reference_test_case_recycling(golden):
    m = n = 100
    for prefix, kw in (("tc_ru_", dict(epsilon=1.21e-2, seed=7, strategy="reuse-u", i_reuse=45)),
                       ("tc_none_", dict(epsilon=1e-2, seed=7, strategy="none"))):
        out = oracle.complete(m, n, golden["tc_rows"], golden["tc_cols"], golden["tc_vals"], oracle.SvtConfig(**kw))
        _check_trace(out, golden, prefix)


def test_svt_cfg1_defaults(golden):
    obs, _ = workloads.cfg1()
    out = oracle.complete(obs.m, obs.n, obs.rows, obs.cols, obs.values, oracle.SvtConfig(seed=0))
    _check_trace(out, golden, "cfg1_")
    assert abs(out.norm2 - float(golden["cfg1_norm2"])) < 1e-10 * out.norm2
    assert out.c == 4
    assert rel((out.U * out.S) @ out.V.T, (golden["cfg1_U"] * golden["cfg1_S"]) @ golden["cfg1_V"].T) < 1e-9
