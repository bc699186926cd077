#!/usr/bin/env python
"""Benchmark of the B200 SVT / rSVD hot path (BASELINE.json metric: "SVT
iterations/sec and rSVD-BKI time (s) at k; SpMM/SDDMM HBM GB/s vs peak").

Headline (default --mode svt): SVT iterations/s of the north-star workload,
svt_fast (rSVD-BKI inner SVDs, reuse-q recycling) on the cfg4 rating shape
(BASELINE configs[3]: 138,493 x 26,744, 20,000,263 ratings, 10 % held out by
the reference's split_observations).  One step = one complete matrix
completion job (setup excluded, run to convergence); N > 1 ranks run the SAME
job over a row/column partition of the pattern (shards.ShardedEngine, NCCL
allgather + allreduce: strong scaling).

  value   : SVT iterations/s = iterations of the K timed jobs / their device
            time (CUDA events; max over ranks), pattern and M resident in HBM
  e2e     : the same metric through the public API svt_fast(obs, params) from
            host COO arrays (page-locked): CSR build, uploads, spectral norm,
            the loop, factors downloaded -- wall clock per job
  roofline: the dominant native call of the job (CUDA events around every
            call on one extra profiled job)
  cpu_baseline: the reference's own svt_fast on the box's host cores (the
            real package from baseline/_ref, else the pinned oracle port) on
            a bounded sample (its first iterations)
  bki     : BASELINE configs[1] beside it -- rsvd_bki / rsvd_pi on the
            100,000 x 50,000 / 5M-nnz matrix: calls/s device-resident and e2e
            legs (host Omega = the parity default; device Omega; Q formed)

--mode bki makes cfg2 rsvd_bki calls/s the headline (the round-1 line);
--replicas runs N independent replicas instead of one sharded job.
--impl reference times the reference's own CPU implementation alone (rank 0).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
K_RANK, S_OVER, P_POW, SEED = 100, 10, 5, 0
WORKLOAD_BKI = "cfg2: rsvd_bki on 100000x50000, 5,000,000 uniform nnz N(0,1), k=100 s=10 p=5 (W=660)"

# cfg4 SVT settings.  The reference's defaults (tau = 5n, delta = 1.2mn/nnz
# ~ 247, completion.py:328-335) diverge on the Zipf-sampled rating pattern in
# BOTH implementations (first-iteration residual 72.05, then rank escalation
# past the 2000-column dense cap; profiles/r02_cfg4_defaults.txt).  The bench
# keeps the rating CLI's recycling defaults (reuse-q, i_reuse 50, q_reuse 10,
# cli.py:277-282) with a step inside SVT's convergence bound (delta < 2 holds
# for any sampling pattern) and tau / eps set so the job converges
# (tools/r02/cfg4_dynamics.py).
CFG4_SVT = dict(tau_div=10.0, delta=1.5, epsilon=0.40, i_reuse=50, q_reuse=10, strategy="reuse-q", seed=0,
                i_max=500)


def cfg4_params(precision="fp64"):
    from paper_1810_06860_b200 import completion

    c = CFG4_SVT
    return completion.SvtParams(tau=5.0 * 26_744 / c["tau_div"], delta=c["delta"], epsilon=c["epsilon"],
                                i_reuse=c["i_reuse"], q_reuse=c["q_reuse"], strategy=c["strategy"], seed=c["seed"],
                                i_max=c["i_max"], precision=precision)


def golden_cfg4_diff(res, mae):
    """The timed job against the REAL reference's run of the same job
    (tests/golden/reference_golden_cfg4.npz, tests/golden/make_golden_cfg4.py)."""
    path = os.path.join(ROOT, "tests", "golden", "reference_golden_cfg4.npz")
    if not os.path.exists(path):
        return None
    g = np.load(path)
    n = min(len(res.trace), int(g["k"].shape[0]))
    same_trace = [(t.k, t.r, t.p, t.q, t.svd_source) for t in res.trace[:n]] == [
        (int(g["k"][i]), int(g["r"][i]), int(g["p"][i]), int(g["q"][i]), str(g["source"][i])) for i in range(n)]
    out = {"iterations": int(g["k"].shape[0]), "converged": bool(g["converged"]),
           "residual_abs_diff": abs(res.residual - float(g["residual"][-1])),
           "heldout_mae_abs_diff": abs(mae - float(g["heldout_mae"])), "trace_identical": same_trace,
           "reference_wall_s_8_threads": float(g["total_s"])}
    if res.S.shape == g["S"].shape:
        out["S_max_rel_diff"] = float(np.max(np.abs(res.S - g["S"]) / g["S"]))
    return out


def workload_svt():
    c = CFG4_SVT
    return (f"cfg4 rating shape 138493x26744, 18,000,237 train / 2,000,026 held out; svt_fast rSVD-BKI reuse-q "
            f"(tau=5n/{c['tau_div']:g}, delta={c['delta']:g}, eps={c['epsilon']:g}, i_reuse={c['i_reuse']}, "
            f"q_reuse={c['q_reuse']}, seed {c['seed']}), one job to convergence per step")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["svt", "bki"], default="svt")
    ap.add_argument("--replicas", action="store_true", help="N independent replicas instead of one sharded job")
    ap.add_argument("--shard", action="store_true", help="the sharded engine even on one rank (collectives forced)")
    ap.add_argument("--cpu-baseline", choices=["full", "skip"], default="full")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--extras", choices=["on", "off"], default="on", help="secondary measurements (cfg2, cfg1)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def host_info(threads=None):
    info = {"cpu_count": os.cpu_count()}
    try:
        info["affinity"] = len(os.sched_getaffinity(0))
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        import subprocess

        ls = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        keep = ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU max MHz", "L3 cache")
        info["lscpu"] = {k.strip(): v.strip() for k, v in (ln.split(":", 1) for ln in ls.splitlines() if ":" in ln)
                         if k.strip() in keep}
    except Exception:
        pass
    try:
        from threadpoolctl import threadpool_info

        info["blas"] = [{"lib": d.get("internal_api"), "version": d.get("version"), "threads": d.get("num_threads"),
                         "arch": d.get("architecture")} for d in threadpool_info()]
    except Exception:
        pass
    if threads is not None:
        info["blas_threads_used"] = threads
    return info


class ClockSampler:
    """NVML samples of SM clock and throttle reasons during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        if index < 0:
            return
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            # warm the two queries (their first call is slow and holds the driver)
            pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.ok = True
        except Exception as exc:  # pragma: no cover - NVML missing
            self.err = str(exc)

    def _run(self):
        nv = self.nv
        names = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                 "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def result(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def fp64_peak_tflops():
    """Measured fp64 GEMM peak (cuBLAS DGEMM 8192^3, best of 3):
    MEASURED_PEAKS.json only carries bf16 and HBM figures."""
    import torch

    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    a @ b
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2 * 8192 ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    del a, b
    torch.cuda.empty_cache()
    return best


L2_READ_GBS = 18000.0  # tools/l2_bw.cu on this pool's B200 (profiles/r01_l2_bw.txt): gather diagnostic


def kernel_table(summary, total_ms, jobs, hbm_peak, fp64_peak):
    """Per native call: time per job, share, SURVEY 8(d) roofline fraction
    (HBM on algorithmic bytes for the sparse kernels, fp64 tensor peak for
    the GEMMs); the sparse products also get their L2-gather rate."""
    from paper_1810_06860_b200 import profiling

    kernels = []
    for name, d in sorted(summary.items(), key=lambda kv: -kv[1]["ms"]):
        entry = {"call": name, "calls_per_job": d["calls"] / jobs, "ms_per_job": d["ms"] / jobs,
                 "share": d["ms"] / total_ms}
        if name in profiling.MODELS and d["modeled_ms"] > 0:
            bound = profiling.MODELS[name][0]
            if bound == "hbm":
                ach = d["bytes"] / (d["modeled_ms"] * 1e-3) / 1e9
                entry.update(bound="hbm", achieved=ach, unit="GB/s", peak=hbm_peak, frac=ach / hbm_peak)
                if name in ("lr_spmm_f64", "lr_spmm_hot_f64", "lr_svt_step_flat_f64", "lr_svt_step_f64") and d.get("gather"):
                    g = d["gather"] / (d["modeled_ms"] * 1e-3) / 1e9
                    entry.update(l2_gather_gbs=g, l2_gather_frac_of_l2_read=g / L2_READ_GBS)
            else:
                ach = d["flops"] / (d["modeled_ms"] * 1e-3) / 1e12
                entry.update(bound="tensor", achieved=ach, unit="TFLOP/s", peak=fp64_peak, frac=ach / fp64_peak)
        kernels.append(entry)
    return kernels


def roofline_of(kernels, traffic_file=None):
    dom = next((k for k in kernels if "bound" in k), None)
    if dom is None:
        return None
    traffic = {}
    if traffic_file and os.path.exists(traffic_file):
        traffic = json.load(open(traffic_file))
    t = traffic.get(dom["call"]) or {}
    return {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"], "unit": dom["unit"],
            "frac": dom["frac"], "traffic": t.get("traffic_bytes"), "kernel": dom["call"],
            "share_of_step": dom["share"],
            "traffic_note": (f"dram read+write bytes per launch from one ncu --set full capture ({traffic_file}: "
                             f"{t.get('launch')}, algorithmic {t.get('algorithmic_bytes')} B)") if t else None,
            "l2_gather_frac_of_l2_read": dom.get("l2_gather_frac_of_l2_read"),
            "peak_source": ("MEASURED_PEAKS.json hbm_gbs (measured)" if dom["bound"] == "hbm"
                            else "fp64 cuBLAS DGEMM 8192^3 measured in this run (MEASURED_PEAKS.json has no "
                                 "fp64 figure)")}


# ------------------------------------------------------------------ reference arm

def reference_lowrank():
    """The reference package itself when it was installed into baseline/_ref
    (python -m pip install --no-deps --target baseline/_ref <reference>),
    else None (the pinned oracle port stands in)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(path, "lowrank")):
        if path not in sys.path:
            sys.path.insert(0, path)
        try:
            import lowrank  # noqa: F401
            from lowrank import completion as _c  # noqa: F401

            return sys.modules["lowrank"]
        except Exception:
            return None
    return None


def cpu_svt_sample(o4, max_iters, threads=None):
    """The reference's svt_fast on cfg4 for its first `max_iters` iterations
    (same settings as our job): iterations / loop time (setup excluded, as
    in our `value`), plus setup time."""
    from paper_1810_06860_b200 import workloads  # noqa: F401

    lr = reference_lowrank()
    c = CFG4_SVT
    ctx = None
    if threads is not None:
        from threadpoolctl import threadpool_limits

        ctx = threadpool_limits(threads)
    try:
        t0 = time.perf_counter()
        if lr is not None:
            from lowrank.completion import SvtParams, svt_fast
            from lowrank.sparse import ObservationSet as RObs

            obs = RObs(o4.m, o4.n, o4.rows, o4.cols, o4.values, o4.split)
            res = svt_fast(obs, SvtParams(tau=5.0 * o4.n / c["tau_div"], delta=c["delta"], epsilon=c["epsilon"],
                                          i_reuse=c["i_reuse"], q_reuse=c["q_reuse"], strategy=c["strategy"],
                                          seed=c["seed"], i_max=max_iters))
            trace = [(t.iteration, t.k, t.r, t.residual, t.wall_time) for t in res.trace]
            kind = "reference"
        else:
            import oracle

            r, cc, v = o4.subset(0)
            res = oracle.complete(o4.m, o4.n, r, cc, v, oracle.SvtConfig(
                epsilon=c["epsilon"], i_reuse=c["i_reuse"], q_reuse=c["q_reuse"], strategy=c["strategy"],
                seed=c["seed"], i_max=max_iters, delta=c["delta"], tau=5.0 * o4.n / c["tau_div"]))
            trace = [(t[0], t[1], t[2], t[5], float("nan")) for t in res.trace]
            kind = "port"
        total = time.perf_counter() - t0
    finally:
        if ctx is not None:
            ctx.unregister()
    loop = sum(t[4] for t in trace) if kind == "reference" else total
    return {"iterations": len(trace), "loop_s": loop, "total_s": total, "iterations_per_s": len(trace) / loop,
            "kind": kind, "residuals": [t[3] for t in trace], "ks": [t[1] for t in trace]}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    from paper_1810_06860_b200 import workloads

    if args.mode == "bki":
        lr = reference_lowrank()
        obs = workloads.cfg2()
        times = []
        budget = 150.0
        for _ in range(max(1, args.steps)):
            if lr is not None:
                from lowrank.rsvd import RsvdParams, rsvd_bki
                from lowrank.sparse import SparseMatrix as RSM

                A = RSM.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
                t0 = time.perf_counter()
                rsvd_bki(A, RsvdParams(k=K_RANK, p=P_POW, s=S_OVER, seed=SEED))
                times.append(time.perf_counter() - t0)
            else:
                import oracle

                P = oracle.csr_from_triples(obs.m, obs.n, obs.rows, obs.cols, obs.values)
                P.transpose_index()
                t0 = time.perf_counter()
                oracle.sketch_bki(P, oracle.SketchParams(k=K_RANK, p=P_POW, s=S_OVER, seed=SEED))
                times.append(time.perf_counter() - t0)
            if sum(times) > budget:
                break
        per = float(np.mean(times))
        v, unit, kind = 1.0 / per, "rSVD-BKI calls/s (cfg2, k=100)", "reference" if lr is not None else "port"
        sample = f"{len(times)} full cfg2 rsvd_bki call(s), {per:.1f} s each"
        config = {"workload": WORKLOAD_BKI}
        steps = len(times)
    else:
        o4 = workloads.cfg4()
        d = cpu_svt_sample(o4, max_iters=int(os.environ.get("BENCH_REF_ITERS", "3")))
        v, unit, kind = d["iterations_per_s"], "SVT iterations/s (cfg4)", d["kind"]
        sample = (f"first {d['iterations']} iterations of the same cfg4 job ({d['loop_s']:.1f} s loop, "
                  f"{d['total_s']:.1f} s incl. CSR build and spectral norm)")
        config = {"workload": workload_svt()}
        steps = d["iterations"]
        per = d["loop_s"] / max(1, d["iterations"])
    line = {"metric": METRIC, "value": v, "unit": unit, "impl": "reference", "n_gpus": 0, "steps": steps,
            "warmup": 0, "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "none",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators, paper_1810_06860_b200/"
                                                           "workloads.py)", "config": config,
            "cpu_baseline": {"value": v, "unit": unit, "cores": os.cpu_count(), "kind": kind, "sample": sample,
                             "host": host_info()},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": f"requested --steps {args.steps} --warmup {args.warmup}; the reference (numpy + scipy + "
                    f"OpenBLAS, default threads) on a bounded sample"}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def init_dist(ws, local, need):
    import torch

    torch.cuda.set_device(local)
    if ws > 1 or need:
        import socket

        import torch.distributed as dist

        if ws == 1:
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                os.environ.setdefault("MASTER_PORT", str(sk.getsockname()[1]))
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))


def max_over_ranks(x, ws):
    import torch

    if ws > 1:
        t = torch.tensor([float(x)], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())
    return float(x)


def barrier(ws):
    if ws > 1:
        import torch

        torch.distributed.barrier()


def bench_svt_main(args, ws, rank, local):
    import torch

    from paper_1810_06860_b200 import _native, completion, device, profiling, workloads
    from paper_1810_06860_b200.sparse import ObservationSet

    sharded = (ws > 1 and not args.replicas) or args.shard
    lib = _native.load()
    t_gen = time.perf_counter()
    o4 = workloads.cfg4()
    t_gen = time.perf_counter() - t_gen
    obs = ObservationSet(o4.m, o4.n, o4.rows, o4.cols, o4.values, o4.split)
    params = cfg4_params()
    if sharded:
        from paper_1810_06860_b200.shards import Exchange, ShardedEngine

        ex = Exchange(always_collective=args.shard)

        def make_engine():
            return ShardedEngine(obs, ex)
    else:
        ex = None

        def make_engine():
            return completion.DeviceEngine(obs)
    eng = make_engine()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2

    def job():
        return completion._svt_loop(obs, params, "rsvd-bki", params.strategy, engine=eng)

    res = None
    for _ in range(args.warmup):
        flush.zero_()
        res = job()
    torch.cuda.synchronize()
    launches0 = lib.lr_launch_count()
    barrier(ws)
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()
    iters, job_ms = [], []
    with ClockSampler(local if os.environ.get("BENCH_NO_CLOCKS") is None else -1) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
        e0.record()
        for i in range(args.steps):
            flush.zero_()
            marks[2 * i].record()
            res = job()
            marks[2 * i + 1].record()
            iters.append(res.iterations)
        e1.record()
        torch.cuda.synchronize()
    gc.enable()
    barrier(ws)
    launches = lib.lr_launch_count() - launches0
    job_ms = [marks[2 * i].elapsed_time(marks[2 * i + 1]) for i in range(args.steps)]
    ms_jobs = max_over_ranks(sum(job_ms), ws)  # device time of the K jobs (flushes excluded)
    total_iters = int(sum(iters))
    value = total_iters / (ms_jobs * 1e-3)
    if args.replicas and ws > 1:
        value *= ws

    # profiled job (events around every native call), outside the timed region
    prof = profiling.Profiler()
    _native.PROFILER = prof
    torch.cuda.synchronize()
    tp0 = time.perf_counter()
    resp = job()
    torch.cuda.synchronize()
    prof_ms = (time.perf_counter() - tp0) * 1e3
    _native.PROFILER = None
    summary = prof.summary()

    # e2e: the public API from host COO arrays (page-locked), a fresh ObservationSet per job
    pinned = [device.pinned_copy(a) for a in (o4.rows, o4.cols, o4.values)]
    split_p = device.pinned_copy(o4.split)
    e2e_s, h2d, d2h, e2e_it = [], [], [], []
    E2E_WARM = 1
    for i in range(args.e2e_steps + E2E_WARM):
        torch.cuda.synchronize()
        barrier(ws)
        th, td = device.TRAFFIC["h2d"], device.TRAFFIC["d2h"]
        t0 = time.perf_counter()
        # the user's input object is built inside the timed region: validation
        # (duplicate search on the device) and the train CSR build count
        ob = ObservationSet(o4.m, o4.n, pinned[0], pinned[1], pinned[2], split_p)
        if sharded:
            from paper_1810_06860_b200.shards import svt_sharded

            r_ = svt_sharded(ob, params, exchange=ex)
        else:
            r_ = completion.svt_fast(ob, params)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i >= E2E_WARM:
            e2e_s.append(dt)
            e2e_it.append(r_.iterations)
            h2d.append(device.TRAFFIC["h2d"] - th)
            d2h.append(device.TRAFFIC["d2h"] - td)
        del r_
    e2e_wall = max_over_ranks(float(np.mean(e2e_s)), ws) if e2e_s else float("nan")
    e2e_value = (float(np.mean(e2e_it)) / e2e_wall) if e2e_s else float("nan")

    # held-out MAE of the timed job's factors (the reference CLI's rating metric)
    rt, ct, vt = obs.subset(1)
    mae = completion.mae(res.predict(rt, ct), vt)
    if rank != 0:
        return None
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    fp64_peak = fp64_peak_tflops()
    kernels = kernel_table(summary, prof_ms, 1, hbm_peak, fp64_peak)
    roof = roofline_of(kernels, os.path.join(ROOT, "profiles", "r02_ncu_traffic.json"))
    line = {
        "metric": METRIC, "value": value, "unit": "SVT iterations/s (cfg4 rating shape, svt_fast rSVD-BKI)",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_jobs / args.steps,
        "higher_is_better": True, "scaling": "weak" if (args.replicas and ws > 1) else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cfg4 generator, workloads.py)",
        "config": {"workload": workload_svt(),
                   "parallelism": (f"sharded x{ws}: nnz-balanced row (CSR) / column (CSC) blocks, NCCL allgather "
                                   f"+ allreduce" if sharded else (f"replicas x{ws}" if ws > 1 else "one GPU")),
                   "omega": "host draw (numpy's own arithmetic, threaded), uploaded; next call's draw prefetched",
                   "l2": "256 MB flush between timed jobs", "job": "one svt_fast run to convergence"},
        "iterations_per_job": iters, "ms_per_job": job_ms, "ms_per_iteration": ms_jobs / max(1, total_iters),
        "job_result": {"iterations": res.iterations, "converged": res.converged, "rank": res.rank,
                       "residual": res.residual, "heldout_mae": mae, "ks": [t.k for t in res.trace][::5],
                       "sources": {s: sum(t.svd_source == s for t in res.trace) for s in
                                   sorted({t.svd_source for t in res.trace})},
                       "vs_reference_run": golden_cfg4_diff(res, mae)},
        "e2e": {"value": e2e_value, "unit": "SVT iterations/s (cfg4 rating shape, svt_fast rSVD-BKI)",
                "h2d_bytes_per_step": int(np.mean(h2d)) if h2d else 0,
                "d2h_bytes_per_step": int(np.mean(d2h)) if d2h else 0, "s_per_job": e2e_wall,
                "note": "ObservationSet(host COO triples, pinned) + public svt_fast(obs, params): validation "
                        "(duplicates searched on the device), CSR build on the device, pattern / values upload, "
                        "spectral norm, the loop (host Omega draws), U/V downloaded; wall clock"},
        "roofline": roof, "roofline_kernels": kernels, "gpu_launches": int(launches), "clocks": clk.result(),
        "generation_s": t_gen, "_trace": res.trace,
    }
    return line


def bench_bki(args, ws, headline):
    """cfg2 rsvd_bki / rsvd_pi (BASELINE configs[1]) on this rank's GPU."""
    import torch

    from paper_1810_06860_b200 import _native, device, profiling, workloads
    from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki, rsvd_bki_dev, rsvd_pi, rsvd_pi_dev
    from paper_1810_06860_b200.sparse import SparseMatrix

    lib = _native.load()
    obs = workloads.cfg2()
    A = SparseMatrix.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
    params = RsvdParams(k=K_RANK, p=P_POW, s=S_OVER, seed=SEED)
    A.pattern()
    A.device_values()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    steps = args.steps if headline else 5
    warm = args.warmup if headline else 3

    def timed(fn, n, w):
        out = None
        for _ in range(w):
            flush.zero_()
            out = fn()
        torch.cuda.synchronize()
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(2 * n)]
        for i in range(n):
            flush.zero_()
            marks[2 * i].record()
            out = fn()
            marks[2 * i + 1].record()
        torch.cuda.synchronize()
        return [marks[2 * i].elapsed_time(marks[2 * i + 1]) for i in range(n)], out

    launches0 = lib.lr_launch_count()
    gc.collect()
    gc.disable()
    ms_host, out = timed(lambda: rsvd_bki_dev(A, params, omega="host"), steps, warm)
    gc.enable()
    launches = lib.lr_launch_count() - launches0
    res_host = out[0]
    ms_dev, out = timed(lambda: rsvd_bki_dev(A, params, omega="device"), steps, warm)
    res_dev = out[0]
    ms_pi, out = timed(lambda: rsvd_pi_dev(A, params, omega="host"), steps, warm)
    res_pi = out[0]
    prof = profiling.Profiler()
    _native.PROFILER = prof
    t0 = time.perf_counter()
    for _ in range(2):
        flush.zero_()
        rsvd_bki_dev(A, params, omega="host")
    torch.cuda.synchronize()
    _native.PROFILER = None
    step_ms = float(np.mean(ms_host))

    # e2e legs through the public API, host matrix in pinned memory, device mirror dropped every call
    A.pin_memory()

    def e2e(fn, n=3, warm_=2):
        ts, hb, db = [], [], []
        for i in range(n + warm_):
            A.drop_device()
            torch.cuda.synchronize()
            th, td = device.TRAFFIC["h2d"], device.TRAFFIC["d2h"]
            t0 = time.perf_counter()
            r = fn()
            torch.cuda.synchronize()
            if i >= warm_:
                ts.append(time.perf_counter() - t0)
                hb.append(device.TRAFFIC["h2d"] - th)
                db.append(device.TRAFFIC["d2h"] - td)
            del r
        ms = float(np.mean(ts)) * 1e3
        return {"value": 1e3 / ms, "ms_per_call": ms, "h2d_bytes_per_step": int(np.mean(hb)),
                "d2h_bytes_per_step": int(np.mean(db))}

    def bki_q_formed():
        r, sub = rsvd_bki(A, params)
        return r, sub.Q  # Subspace.Q forms Q on the device and downloads it

    legs = {"public_default_host_omega": e2e(lambda: rsvd_bki(A, params)),
            "device_omega": e2e(lambda: rsvd_bki(A, params, omega="device")),
            "host_omega_Q_formed_and_downloaded": e2e(bki_q_formed),
            "rsvd_pi_host_omega": e2e(lambda: rsvd_pi(A, params))}
    A.drop_device()
    A.pattern()
    A.device_values()
    return {
        "workload": WORKLOAD_BKI,
        "rsvd_bki_calls_per_s": 1e3 / step_ms, "rsvd_bki_time_s": step_ms * 1e-3, "ms_per_call": ms_host,
        "rsvd_bki_device_omega_calls_per_s": 1e3 / float(np.mean(ms_dev)),
        "rsvd_pi_calls_per_s": 1e3 / float(np.mean(ms_pi)), "rsvd_pi_time_s": float(np.mean(ms_pi)) * 1e-3,
        "max_rel_S_diff_host_vs_device_omega": float(np.max(np.abs(res_dev.S_host - res_host.S_host) /
                                                            res_host.S_host)),
        "e2e_legs": legs, "gpu_launches_per_call": launches / steps,
        "profile": prof.summary(), "S_host": res_host.S_host, "S_pi": res_pi.S_host,
    }


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    import torch

    init_dist(ws, local, need=args.shard)
    if args.mode == "svt":
        line = bench_svt_main(args, ws, rank, local)
    else:
        line = None
    if rank == 0 and args.extras == "on" or (args.mode == "bki" and rank == 0):
        b = bench_bki(args, ws, headline=args.mode == "bki")
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        fp64_peak = line["roofline"]["peak"] if (line and line.get("roofline") and
                                                 line["roofline"]["bound"] == "tensor") else fp64_peak_tflops()
        kern = kernel_table(b.pop("profile"), b["rsvd_bki_time_s"] * 1e3 * 2, 2, hbm_peak, fp64_peak)
        b["roofline_kernels"] = kern
        S_host, S_pi = b.pop("S_host"), b.pop("S_pi")
        if args.cpu_baseline == "full" and ws == 1:
            lr = reference_lowrank()
            from paper_1810_06860_b200 import workloads

            o = workloads.cfg2()
            if lr is not None:
                from lowrank.rsvd import RsvdParams as RP
                from lowrank.rsvd import rsvd_bki as rbki
                from lowrank.sparse import SparseMatrix as RSM

                RA = RSM.from_coo(o.m, o.n, o.rows, o.cols, o.values)
                t0 = time.perf_counter()
                ref, _ = rbki(RA, RP(k=K_RANK, p=P_POW, s=S_OVER, seed=SEED))
                dt = time.perf_counter() - t0
                kind = "reference"
            else:
                import oracle

                P = oracle.csr_from_triples(o.m, o.n, o.rows, o.cols, o.values)
                P.transpose_index()
                t0 = time.perf_counter()
                ref, _ = oracle.sketch_bki(P, oracle.SketchParams(k=K_RANK, p=P_POW, s=S_OVER, seed=SEED))
                dt = time.perf_counter() - t0
                kind = "port"
            b["cpu_baseline"] = {"value": 1.0 / dt, "unit": "rSVD-BKI calls/s (cfg2, k=100)", "kind": kind,
                                 "cores": os.cpu_count(), "sample": f"one full cfg2 rsvd_bki call: {dt:.2f} s",
                                 "max_rel_S_diff_vs_gpu": float(np.max(np.abs(S_host - ref.S) / ref.S))}
        if line is None:  # --mode bki headline
            line = {"metric": METRIC, "value": b["rsvd_bki_calls_per_s"], "unit": "rSVD-BKI calls/s (cfg2, k=100)",
                    "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                    "ms_per_step": b["rsvd_bki_time_s"] * 1e3, "higher_is_better": True, "scaling": "weak",
                    "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cfg2 generator)",
                    "config": {"workload": WORKLOAD_BKI, "omega": "host draw (parity default)"},
                    "e2e": dict(b["e2e_legs"]["public_default_host_omega"],
                                unit="rSVD-BKI calls/s (cfg2, k=100)"),
                    "roofline": roofline_of(kern, os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")),
                    "cpu_baseline": b.get("cpu_baseline"),
                    "gpu_launches": int(b["gpu_launches_per_call"] * args.steps)}
        else:
            line["bki_cfg2"] = b
    if rank == 0 and args.mode == "svt" and line is not None:
        if args.cpu_baseline == "full" and ws == 1:
            from paper_1810_06860_b200 import workloads

            o4c = workloads.cfg4()
            d = cpu_svt_sample(o4c, max_iters=int(os.environ.get("BENCH_REF_ITERS", "3")))
            d1 = cpu_svt_sample(o4c, max_iters=1, threads=1)  # the reference's own 1-thread convention
            line["cpu_baseline_1thread"] = {"value": d1["iterations_per_s"], "unit": "SVT iterations/s (cfg4)",
                                            "cores": 1, "kind": d1["kind"],
                                            "sample": f"first iteration of the same cfg4 job, BLAS limited to "
                                                      f"1 thread ({d1['loop_s']:.1f} s loop)"}
            line["cpu_baseline"] = {"value": d["iterations_per_s"], "unit": "SVT iterations/s (cfg4)",
                                    "cores": os.cpu_count(), "kind": d["kind"],
                                    "sample": f"first {d['iterations']} iterations of the same cfg4 job "
                                              f"({d['loop_s']:.1f} s loop, {d['total_s']:.1f} s incl. setup)",
                                    "host": host_info(),
                                    "residual_rel_diff_first_iterations": [
                                        abs(a - t.residual) / a for a, t in
                                        zip(d["residuals"], line.get("_trace", []))]}
        line.pop("_trace", None)
    if rank == 0 and line is not None:
        print(json.dumps(line, default=float), flush=True)
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
