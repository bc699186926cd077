"""Generate the golden fixtures from the REAL reference package.

Run in the build container only (the reference lives at /root/reference and
does not travel to the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

It imports `lowrank` from /root/reference/pkg/src, runs it on seeded inputs,
and writes tests/golden/*.npz.  The oracle (oracle/) is pinned against these
files by tests/test_oracle_golden.py; the GPU parity tests use them too.
Known-answer items taken from the reference's own tests:
Box-Muller vs uniforms (test_rng.py:44-49), F-order fill (test_rng.py:71-76),
from_coo ordering (test_sparse.py:45-50), frobenius 3-4-5 (test_sparse.py:273),
the 20-step adapt_power trace (test_completion.py:169-176).
"""

import os
import sys

for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[v] = "1"

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import lowrank  # noqa: E402
from lowrank.completion import SvtParams, SvtState, adapt_power, svt_fast, svt_reference  # noqa: E402
from lowrank.linalg import eig_svd, lu_pl, oracle_svd, orth  # noqa: E402
from lowrank.rng import RngState, gaussian_matrix  # noqa: E402
from lowrank.rsvd import RsvdParams, qb_error, rsvd_basic, rsvd_bki, rsvd_pi  # noqa: E402
from lowrank.sparse import (ObservationSet, SparseMatrix, frobenius, project_pattern,  # noqa: E402
                            spectral_norm_est, spmm, spmm_t)

from paper_1810_06860_b200 import workloads  # noqa: E402


def random_sparse(seed, m, n, nnz):
    rng = RngState(seed)
    flat = rng.choice_without_replacement(m * n, nnz)
    i, j = np.divmod(np.asarray(flat, np.int64), n)
    return i, j, rng.normal_pairs(nnz)


def trace_arrays(res, prefix, out):
    t = res.trace
    out[prefix + "iteration"] = np.array([x.iteration for x in t])
    out[prefix + "k"] = np.array([x.k for x in t])
    out[prefix + "r"] = np.array([x.r for x in t])
    out[prefix + "p"] = np.array([x.p for x in t])
    out[prefix + "q"] = np.array([x.q for x in t])
    out[prefix + "residual"] = np.array([x.residual for x in t])
    out[prefix + "source"] = np.array([x.svd_source for x in t])
    out[prefix + "S"] = res.S
    out[prefix + "converged"] = np.array(res.converged)
    out[prefix + "hard_stops"] = np.array(res.hard_stops)


def main():
    g = {}
    # ---- rng
    for seed in (0, 1, 2, 12345, 2**62 + 7):
        g[f"rng_normals_{seed}"] = RngState(seed).normal_pairs(257)
        g[f"rng_uniform_{seed}"] = RngState(seed).uniform(64)
    g["rng_gauss_5_4x3"] = gaussian_matrix(RngState(5), 4, 3)
    g["rng_gauss_7_37x11"] = gaussian_matrix(RngState(7), 37, 11)
    g["rng_spawn"] = np.array([RngState(s).spawn(t).seed for s in (0, 1, 99, 2**40) for t in (0, 1, 2, 17)],
                              dtype=np.uint64)
    # ---- sparse structure + kernels
    g["coo_small_indptr"] = SparseMatrix.from_coo(3, 4, [2, 0, 0], [1, 3, 0], [5.0, 6.0, 7.0]).indptr
    g["coo_small_indices"] = SparseMatrix.from_coo(3, 4, [2, 0, 0], [1, 3, 0], [5.0, 6.0, 7.0]).indices
    g["coo_small_data"] = SparseMatrix.from_coo(3, 4, [2, 0, 0], [1, 3, 0], [5.0, 6.0, 7.0]).data
    i, j, v = random_sparse(3, 60, 45, 500)
    A = SparseMatrix.from_coo(60, 45, i, j, v)
    g["sp_i"], g["sp_j"], g["sp_v"] = i, j, v
    g["sp_indptr"], g["sp_indices"], g["sp_data"] = A.indptr, A.indices, A.data
    perm, tip, tix = A._transpose_index()
    g["sp_tperm"], g["sp_tindptr"], g["sp_tindices"] = perm, tip, tix
    X = gaussian_matrix(RngState(8), 45, 7)
    H = gaussian_matrix(RngState(9), 60, 7)
    g["sp_X"], g["sp_H"] = X, H
    g["sp_spmm"] = spmm(A, X)
    g["sp_spmm_t"] = spmm_t(A, H)
    U = gaussian_matrix(RngState(10), 60, 4)
    V = gaussian_matrix(RngState(11), 45, 4)
    S = np.array([3.0, 2.0, 1.5, 0.25])
    g["sp_U"], g["sp_V"], g["sp_S"] = U, V, S
    g["sp_project"] = project_pattern(U, S, V, A)
    g["sp_frob"] = np.array(frobenius(A.data))
    g["frob_345"] = np.array(frobenius(np.array([3.0, 4.0])))
    g["sp_norm2"] = np.array(spectral_norm_est(A, RngState(3)))
    # ---- dense
    Xo = gaussian_matrix(RngState(21), 40, 12)
    g["orth_X"], g["orth_Q"] = Xo, orth(Xo)
    Xl = gaussian_matrix(RngState(22), 25, 7)
    g["lu_X"], g["lu_PL"] = Xl, lu_pl(Xl)
    Xl2 = gaussian_matrix(RngState(23), 300, 40)
    g["lu2_X"], g["lu2_PL"] = Xl2, lu_pl(Xl2)
    Ae = gaussian_matrix(RngState(24), 120, 30)
    r = eig_svd(Ae)
    g["eig_A"], g["eig_U"], g["eig_S"], g["eig_V"] = Ae, r.U, r.S, r.V
    r = oracle_svd(Ae)
    g["osvd_U"], g["osvd_S"], g["osvd_V"] = r.U, r.S, r.V
    # ---- rsvd
    i, j, v = random_sparse(30, 300, 200, 6000)
    g["rs_i"], g["rs_j"], g["rs_v"] = i, j, v
    A = SparseMatrix.from_coo(300, 200, i, j, v)
    for name, fn in (("pi", rsvd_pi), ("bki", rsvd_bki), ("basic", rsvd_basic)):
        res, sub = fn(A, RsvdParams(k=10, p=2, s=5, seed=3))
        g[f"rs_{name}_U"], g[f"rs_{name}_S"], g[f"rs_{name}_V"], g[f"rs_{name}_Q"] = res.U, res.S, res.V, sub.Q
        g[f"rs_{name}_qb"] = np.array(qb_error(A, res))
    # ---- svt: small cfg1-shaped case, all routes
    obs, _ = workloads.cfg1_small()
    ob = ObservationSet(obs.m, obs.n, obs.rows, obs.cols, obs.values)
    trace_arrays(svt_reference(ob, SvtParams(epsilon=1e-3, seed=4), backend="rsvd-bki"), "svt_small_bki_", g)
    trace_arrays(svt_fast(ob, SvtParams(epsilon=1e-3, seed=4, strategy="reuse-q", i_reuse=20)), "svt_small_rq_", g)
    trace_arrays(svt_fast(ob, SvtParams(epsilon=1e-3, seed=4, strategy="reuse-u", i_reuse=20)), "svt_small_ru_", g)
    trace_arrays(svt_reference(ob, SvtParams(epsilon=1e-3, seed=4), backend="oracle"), "svt_small_oracle_", g)
    trace_arrays(svt_fast(ob, SvtParams(epsilon=0.05, seed=7, strategy="reuse-q", i_reuse=10)), "svt_small_rq2_", g)
    # the reference's own converging recycling cases, built with its test helpers
    # (test_completion.py:392-414: factor_matrix(100,100,5,20), observe(.,0.4,21))
    sys.path.insert(0, "/root/reference/pkg/tests")
    import test_completion as tc
    M = tc.factor_matrix(100, 100, 5, seed=20)
    ob2 = tc.observe(M, 0.4, 21)
    g["tc_rows"], g["tc_cols"], g["tc_vals"] = ob2.rows, ob2.cols, ob2.values
    trace_arrays(svt_fast(ob2, SvtParams(epsilon=1e-2, seed=7, strategy="reuse-q", i_reuse=25)), "tc_rq_", g)
    trace_arrays(svt_fast(ob2, SvtParams(epsilon=1.21e-2, seed=7, strategy="reuse-u", i_reuse=45)), "tc_ru_", g)
    trace_arrays(svt_fast(ob2, SvtParams(epsilon=1e-2, seed=7, strategy="none")), "tc_none_", g)
    # ---- svt cfg1 (BASELINE configs[0]) at the reference defaults and eps=1e-3
    obs, (U1, V1) = workloads.cfg1()
    ob = ObservationSet(obs.m, obs.n, obs.rows, obs.cols, obs.values)
    res = svt_reference(ob, SvtParams(seed=0), backend="rsvd-bki")
    trace_arrays(res, "cfg1_", g)
    g["cfg1_U"], g["cfg1_V"] = res.U, res.V
    phi = ob.train_matrix()
    g["cfg1_norm2"] = np.array(spectral_norm_est(phi, RngState(0).spawn(1)))
    res = svt_reference(ob, SvtParams(seed=0, epsilon=1e-3), backend="rsvd-bki")
    trace_arrays(res, "cfg1e3_", g)
    # ---- adapt_power known-answer trace (test_completion.py:169-176)
    errs = [0.9, 0.8, 0.85, 0.7, 0.6, 0.5, 0.4, 0.35, 0.3, 0.25,
            0.2, 0.18, 0.15, 0.16, 0.1, 0.09, 0.08, 0.07, 0.06, 0.05]
    st = SvtState(Y=None, p=3)
    g["power_errs"] = np.array(errs)
    g["power_p"] = np.array([adapt_power(st, e) for e in errs])
    g["versions"] = np.array([np.__version__, __import__("scipy").__version__, lowrank.__version__])
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **g)
    print("wrote", len(g), "arrays")


if __name__ == "__main__":
    main()
