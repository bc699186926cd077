"""Multi-rank sharded path on the CPU: world size 2 over gloo with the numpy
kernel set (tests/host_kernels.py) injected into shards.ShardedEngine.

What this pins: the shard plan, every allgather / allreduce of the
choreography, the replicated solves and the host decisions (both ranks
must produce identical results), and that the sharded SVT / rSVD-BKI
reproduce the REFERENCE's own outputs (tests/golden) -- traces, ranks,
sources, residuals and singular values.  The device kernels themselves are
pinned by the -m gpu suite (test_gpu_shards.py runs the same worker on one
GPU over NCCL)."""

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from paper_1810_06860_b200.shards import ShardPlan, balanced_bounds  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")


def test_balanced_bounds_properties():
    rng = np.random.default_rng(0)
    for _ in range(50):
        rows = int(rng.integers(1, 400))
        lens = rng.zipf(1.5, size=rows).clip(0, 5000) * rng.integers(0, 2, size=rows)
        ptr = np.r_[0, np.cumsum(lens)]
        for parts in (1, 2, 3, 8):
            if rows < parts:
                with pytest.raises(ValueError):
                    balanced_bounds(ptr, parts)
                continue
            b = balanced_bounds(ptr, parts)
            assert b[0] == 0 and b[-1] == rows
            assert np.all(np.diff(b) >= 1)
            # each cut is within one row of the ideal prefix target
            nnz = ptr[-1]
            for g in range(1, parts):
                target = g * nnz // parts
                i = int(np.searchsorted(ptr, target))
                assert b[g] == min(max(i, b[g - 1] + 1), rows - (parts - g))
            assert np.array_equal(balanced_bounds(ptr, parts), b)  # deterministic


def test_shard_plan_describe():
    ip = np.array([0, 5, 5, 6, 20, 21])
    tp = np.array([0, 1, 2, 3, 21])
    p = ShardPlan(ip, tp, 2)
    d = p.describe()
    assert d["row_bounds"][0] == 0 and d["row_bounds"][-1] == 5
    assert sum(d["row_nnz"]) == 21 and sum(d["col_nnz"]) == 21
    assert p.rows(0)[1] == p.rows(1)[0]


@pytest.fixture(scope="module")
def gloo_runs(tmp_path_factory):
    from shard_worker import spawn

    out = {}
    for world in (2, 1):
        d = tmp_path_factory.mktemp(f"gloo{world}")
        out[world] = spawn(world, str(d), "gloo", GOLDEN, ("exchange", "bki", "svt"))
    return out


def _ok(runs):
    for r in runs:
        assert bool(r["ok"]), str(r.get("error", "worker died"))


def test_gloo_exchange(gloo_runs):
    runs = gloo_runs[2]
    _ok(runs)
    for rank, r in enumerate(runs):
        assert bool(r["ex_gather_ok"])
        np.testing.assert_array_equal(r["ex_allreduce"], np.full((4, 2), 3.0))
        np.testing.assert_array_equal(r["ex_scalars"], np.array([[0.0, 0.0], [1.0, 2.0]]))


@pytest.mark.parametrize("world", [1, 2])
def test_gloo_bki_matches_reference(gloo_runs, golden, world):
    runs = gloo_runs[world]
    _ok(runs)
    r = runs[0]
    S_ref = golden["rs_bki_S"]
    assert int(r["bki_reuse"]) == 1  # Y^T Q from the Krylov products, Q's allgather deferred
    assert np.max(np.abs(r["bki_S"] - S_ref)) <= 1e-10 * S_ref[0]
    np.testing.assert_allclose(r["bki_U"], golden["rs_bki_U"], atol=1e-9)
    np.testing.assert_allclose(r["bki_V"], golden["rs_bki_V"], atol=1e-9)
    Qr = golden["rs_bki_Q"]
    # same subspace (orthonormal bases of span(H)): projectors agree
    np.testing.assert_allclose(r["bki_Q"] @ (r["bki_Q"].T @ Qr), Qr, atol=1e-9)
    for other in runs[1:]:  # every rank holds the identical result
        for key in ("bki_U", "bki_S", "bki_V", "bki_Q"):
            np.testing.assert_array_equal(other[key], r[key])


PREFIXES = ("svt_small_bki_", "svt_small_rq2_", "tc_ru_", "svt_small_oracle_")


@pytest.mark.parametrize("world", [1, 2])
@pytest.mark.parametrize("prefix", PREFIXES)
def test_gloo_svt_matches_reference(gloo_runs, golden, world, prefix):
    runs = gloo_runs[world]
    _ok(runs)
    r = runs[0]
    n = len(golden[prefix + "k"])
    assert list(r[prefix + "k"]) == list(golden[prefix + "k"])
    assert list(r[prefix + "r"]) == list(golden[prefix + "r"])
    assert list(r[prefix + "p"]) == list(golden[prefix + "p"])
    assert list(r[prefix + "q"]) == list(golden[prefix + "q"])
    assert list(r[prefix + "source"]) == list(golden[prefix + "source"])
    assert len(r[prefix + "residual"]) == n
    np.testing.assert_allclose(r[prefix + "residual"], golden[prefix + "residual"], rtol=1e-8)
    np.testing.assert_allclose(r[prefix + "S"], golden[prefix + "S"], rtol=1e-8)
    assert bool(r[prefix + "converged"]) == bool(golden[prefix + "converged"])
    if world == 2:
        rb, cb = r[prefix + "plan_rows"], r[prefix + "plan_cols"]
        m, n = (100, 100) if prefix.startswith("tc_") else (200, 150)
        assert len(rb) == 3 and rb[0] == 0 and rb[-1] == m and 0 < rb[1] < m
        assert len(cb) == 3 and cb[-1] == n
    for other in runs[1:]:
        for key in ("k", "r", "residual", "S", "U", "V"):
            np.testing.assert_array_equal(other[prefix + key], r[prefix + key])
