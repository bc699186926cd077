"""Per-rank body of the sharded-path tests (spawned by test_shards_gloo.py
on the CPU with gloo, and by test_gpu_shards.py on one GPU with NCCL).
Each rank writes its results to <outdir>/rank<r>.npz."""

from __future__ import annotations

import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)
for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import numpy as np  # noqa: E402


def _trace(res, prefix, out):
    t = res.trace
    out[prefix + "k"] = np.array([x.k for x in t])
    out[prefix + "r"] = np.array([x.r for x in t])
    out[prefix + "p"] = np.array([x.p for x in t])
    out[prefix + "q"] = np.array([x.q for x in t])
    out[prefix + "residual"] = np.array([x.residual for x in t])
    out[prefix + "source"] = np.array([x.svd_source for x in t])
    out[prefix + "S"] = res.S
    out[prefix + "U"] = res.U
    out[prefix + "V"] = res.V
    out[prefix + "converged"] = np.array(res.converged)


def run(rank, world, port, outdir, backend, golden_path, cases):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    out = {}
    try:
        if backend == "nccl":
            torch.cuda.set_device(0)
        dist.init_process_group(backend, rank=rank, world_size=world)
        from paper_1810_06860_b200 import workloads
        from paper_1810_06860_b200.completion import SvtParams
        from paper_1810_06860_b200.rsvd import RsvdParams
        from paper_1810_06860_b200.shards import Exchange, rsvd_bki_sharded, svt_sharded
        from paper_1810_06860_b200.sparse import ObservationSet, SparseMatrix

        if backend == "gloo":
            from host_kernels import HostKernels

            K = HostKernels()
            dev = torch.device("cpu")
        else:
            from paper_1810_06860_b200.shards import DeviceKernels

            K = DeviceKernels()
            dev = torch.device("cuda", 0)
        ex = Exchange(always_collective=(backend == "nccl"))
        g = dict(np.load(golden_path))

        if "exchange" in cases:
            bounds = np.array([0, 3, 10] if world == 2 else [0, 10])
            lo, hi = bounds[rank], bounds[rank + 1]
            full = torch.arange(30, dtype=torch.float64, device=dev).reshape(10, 3) * 1.5
            got = torch.zeros((10, 3), dtype=torch.float64, device=dev)
            ex.gather_rows(full[lo:hi].clone(), bounds, got)
            out["ex_gather_ok"] = np.array(bool(torch.equal(got, full)))
            t = torch.full((4, 3), float(rank + 1), dtype=torch.float64, device=dev)[:, :2]
            ex.allreduce_sum(t)
            out["ex_allreduce"] = t.cpu().numpy()
            sc = ex.gather_scalars(torch.tensor([rank, 2.0 * rank], dtype=torch.float64, device=dev))
            out["ex_scalars"] = sc

        if "bki" in cases:
            A = SparseMatrix.from_coo(300, 200, g["rs_i"], g["rs_j"], g["rs_v"])
            from paper_1810_06860_b200.rsvd import REUSE_STATS

            used0 = REUSE_STATS["used"]
            res, sub = rsvd_bki_sharded(A, RsvdParams(k=10, p=2, s=5, seed=3), exchange=ex, kernels=K)
            out["bki_reuse"] = np.array(REUSE_STATS["used"] - used0)
            out["bki_U"], out["bki_S"], out["bki_V"] = res.U, res.S, res.V
            Q = sub.Q if isinstance(sub.Q, np.ndarray) else sub.Q.cpu().numpy()
            out["bki_Q"] = np.asarray(Q)

        if "svt" in cases:
            o, _ = workloads.cfg1_small()
            ob = ObservationSet(o.m, o.n, o.rows, o.cols, o.values)
            ob2 = ObservationSet(100, 100, g["tc_rows"], g["tc_cols"], g["tc_vals"])
            for prefix, kw, be, obx in (
                    ("svt_small_bki_", dict(epsilon=1e-3, seed=4), "rsvd-bki", ob),
                    ("svt_small_rq2_", dict(epsilon=0.05, seed=7, strategy="reuse-q", i_reuse=10), "rsvd-bki", ob),
                    ("tc_ru_", dict(epsilon=1.21e-2, seed=7, strategy="reuse-u", i_reuse=45), "rsvd-bki", ob2),
                    ("svt_small_oracle_", dict(epsilon=1e-3, seed=4), "oracle", ob)):
                res = svt_sharded(obx, SvtParams(**kw), backend=be, exchange=ex, kernels=K)
                _trace(res, prefix, out)
                out[prefix + "plan_rows"] = np.array(res.plan["row_bounds"])
                out[prefix + "plan_cols"] = np.array(res.plan["col_bounds"])
        if "cfg1" in cases:
            o, _ = workloads.cfg1()
            ob = ObservationSet(o.m, o.n, o.rows, o.cols, o.values)
            res = svt_sharded(ob, SvtParams(seed=0), backend="rsvd-bki", exchange=ex, kernels=K)
            _trace(res, "cfg1_", out)
        out["bytes"] = np.array(ex.bytes)
        dist.barrier()
        dist.destroy_process_group()
        out["ok"] = np.array(True)
    except Exception:  # report to the parent test instead of hanging it
        out["ok"] = np.array(False)
        out["error"] = np.array(traceback.format_exc())
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)


def spawn(world, outdir, backend, golden_path, cases, timeout=600):
    """Run `run` on `world` fresh processes; returns the per-rank dicts."""
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=run, args=(r, world, port, outdir, backend, golden_path, cases))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout)
    for p in procs:
        if p.is_alive():
            p.kill()
            p.join()
    res = []
    for r in range(world):
        path = os.path.join(outdir, f"rank{r}.npz")
        res.append(dict(np.load(path, allow_pickle=False)) if os.path.exists(path) else {"ok": np.array(False)})
    return res
