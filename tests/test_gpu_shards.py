"""Sharded path on the GPU: shards.ShardedEngine with the sm_100a kernel set
(DeviceKernels) over NCCL, world size 1 with the collectives forced on
(Exchange(always_collective=True): every allgather / allreduce goes through
NCCL even with one rank), checked against the reference's golden outputs
and against the single-GPU engine.  World size > 1 is covered on the CPU by
test_shards_gloo.py (only one GPU is available to this suite)."""

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")
PREFIXES = ("svt_small_bki_", "svt_small_rq2_", "tc_ru_", "svt_small_oracle_")


@pytest.fixture(scope="module")
def nccl_run(tmp_path_factory):
    from shard_worker import spawn

    d = tmp_path_factory.mktemp("nccl1")
    runs = spawn(1, str(d), "nccl", GOLDEN, ("exchange", "bki", "svt", "cfg1"))
    assert bool(runs[0]["ok"]), str(runs[0].get("error", "worker died"))
    return runs[0]


def test_nccl_exchange(nccl_run):
    assert bool(nccl_run["ex_gather_ok"])
    np.testing.assert_array_equal(nccl_run["ex_allreduce"], np.full((4, 2), 1.0))
    np.testing.assert_array_equal(nccl_run["ex_scalars"], np.array([[0.0, 0.0]]))
    assert int(nccl_run["bytes"]) > 0


def test_nccl_bki_matches_reference(nccl_run, golden):
    r = nccl_run
    S_ref = golden["rs_bki_S"]
    assert np.max(np.abs(r["bki_S"] - S_ref)) <= 1e-10 * S_ref[0]
    ref = (golden["rs_bki_U"] * S_ref) @ golden["rs_bki_V"].T
    got = (r["bki_U"] * r["bki_S"]) @ r["bki_V"].T
    assert np.max(np.abs(got - ref)) <= 1e-9 * np.max(np.abs(ref))
    Qr = golden["rs_bki_Q"]
    np.testing.assert_allclose(r["bki_Q"] @ (r["bki_Q"].T @ Qr), Qr, atol=1e-9)


@pytest.mark.parametrize("prefix", PREFIXES)
def test_nccl_svt_matches_reference(nccl_run, golden, prefix):
    r = nccl_run
    for key in ("k", "r", "p", "q", "source"):
        assert list(r[prefix + key]) == list(golden[prefix + key]), key
    np.testing.assert_allclose(r[prefix + "residual"], golden[prefix + "residual"], rtol=1e-8)
    np.testing.assert_allclose(r[prefix + "S"], golden[prefix + "S"], rtol=1e-8)
    assert bool(r[prefix + "converged"]) == bool(golden[prefix + "converged"])


def test_nccl_svt_cfg1_defaults(nccl_run, golden):
    r = nccl_run
    for key in ("k", "r", "p", "q", "source"):
        assert list(r["cfg1_" + key]) == list(golden["cfg1_" + key]), key
    np.testing.assert_allclose(r["cfg1_residual"], golden["cfg1_residual"], rtol=1e-8)
    np.testing.assert_allclose(r["cfg1_S"], golden["cfg1_S"], rtol=1e-8)
    ref = (golden["cfg1_U"] * golden["cfg1_S"]) @ golden["cfg1_V"].T
    got = (r["cfg1_U"] * r["cfg1_S"]) @ r["cfg1_V"].T
    assert np.max(np.abs(got - ref)) <= 1e-8 * np.max(np.abs(ref))


def test_sharded_world1_equals_single_engine():
    """In-process (no process group): the sharded engine at world size 1
    runs the single-GPU kernels on the same data -> the same trace as the
    single-GPU engine, residuals to rounding."""
    from paper_1810_06860_b200 import completion, workloads
    from paper_1810_06860_b200.shards import svt_sharded
    from paper_1810_06860_b200.sparse import ObservationSet

    o, _ = workloads.cfg1_small()
    ob = ObservationSet(o.m, o.n, o.rows, o.cols, o.values)
    p = completion.SvtParams(epsilon=1e-3, seed=4)
    a = completion.svt_reference(ob, p, backend="rsvd-bki")
    b = svt_sharded(ob, p, backend="rsvd-bki", strategy="none")
    assert [t.k for t in a.trace] == [t.k for t in b.trace]
    assert [t.r for t in a.trace] == [t.r for t in b.trace]
    np.testing.assert_allclose([t.residual for t in b.trace], [t.residual for t in a.trace], rtol=1e-10)
    np.testing.assert_allclose(b.S, a.S, rtol=1e-10)


@pytest.mark.parametrize("world", [2, 3])
def test_device_cut_blocks_match_host_cut(world):
    """ShardedEngine's device setup (the train CSR built on the device, the
    row block sliced and the column block selected there) against the host
    setup (lexsort + flatnonzero) for every rank of a `world`-rank plan:
    identical plans, offsets, indices, values and split tags honoured; the
    blocks' products agree bit for bit."""
    import torch

    from paper_1810_06860_b200 import device
    from paper_1810_06860_b200.shards import DeviceKernels, Exchange, ShardedEngine
    from paper_1810_06860_b200.sparse import ObservationSet, SparseMatrix

    rng = np.random.default_rng(world)
    m, n, nnz = 900, 700, 40000
    flat = rng.choice(m * n, size=nnz, replace=False)
    i, j = np.divmod(flat, n)
    v = rng.standard_normal(nnz)
    split = (rng.random(nnz) < 0.1).astype(np.uint8)  # 10 % held out
    X = device.to_device(rng.standard_normal((n, 7)))
    H = device.to_device(rng.standard_normal((m, 7)))
    for rank in range(world):
        ex = Exchange()
        ex.rank, ex.world = rank, world  # a plan for `world` ranks; no collective runs in the setup
        eng = ShardedEngine(ObservationSet(m, n, i, j, v, split), ex)
        assert eng.phi_r._dev_csr is not None  # the device path ran
        keep = split == 0
        ref = ShardedEngine.__new__(ShardedEngine)
        ref.ex, ref.K, ref.rank, ref.world = ex, DeviceKernels(), rank, world
        ref._setup(SparseMatrix.from_coo(m, n, i[keep], j[keep], v[keep]))
        assert (eng.r0, eng.r1, eng.c0, eng.c1) == (ref.r0, ref.r1, ref.c0, ref.c1)
        assert np.array_equal(eng.plan.row_bounds, ref.plan.row_bounds)
        assert np.array_equal(eng.plan.col_bounds, ref.plan.col_bounds)
        for a, b in ((eng.phi_r, ref.phi_r), (eng.phi_c, ref.phi_c)):
            assert a.shape == b.shape
            assert np.array_equal(a.indptr, b.indptr)
            assert np.array_equal(a.indices, b.indices)
            assert np.array_equal(a.data, b.data)
            assert np.array_equal(device.to_host(a.pattern().csr.ptr), b.indptr.astype(np.int32))
        Xc = X[eng.c0:eng.c1].contiguous()
        assert torch.equal(eng.K.spmm(eng.phi_r, X, None), ref.K.spmm(ref.phi_r, X, None))
        assert torch.equal(eng.K.spmm_t(eng.phi_c, H, None), ref.K.spmm_t(ref.phi_c, H, None))
        assert torch.equal(eng.K.spmm(eng.phi_c, Xc, None), ref.K.spmm(ref.phi_c, Xc, None))
