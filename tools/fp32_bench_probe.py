# Reproduce bench.py's fp32 section after the e2e phase, with per-step wall / device / native times.
import sys, time
import torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import _native, profiling, workloads
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki, rsvd_bki_dev
from paper_1810_06860_b200.sparse import SparseMatrix

obs = workloads.cfg2()
A = SparseMatrix.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
prm = RsvdParams(k=100, p=5, s=10, seed=0)
mode = sys.argv[1] if len(sys.argv) > 1 else "pinned"
for _ in range(3):
    rsvd_bki_dev(A, prm, omega="device")
if mode == "pinned":
    A.pin_memory()
    for _ in range(3):
        A.drop_device()
        rsvd_bki(A, prm)
    torch.cuda.empty_cache()
    A.drop_device()
    A.pattern()
    A.device_values()
for prec in ("fp32", "fp32", "fp32", "fp64", "fp64", "fp32"):
    torch.cuda.synchronize()
    prof = profiling.Profiler()
    _native.PROFILER = prof
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    rsvd_bki_dev(A, prm, omega="device", precision=prec)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    _native.PROFILER = None
    nat = sum(a.elapsed_time(b) for _, _, a, b in prof.records)
    top = sorted(((a.elapsed_time(b), n) for n, _, a, b in prof.records), reverse=True)[:4]
    print(f"{mode} {prec}: wall {wall:.2f} ms, device {e0.elapsed_time(e1):.2f} ms, native {nat:.2f} ms; top {[(n, round(t, 2)) for t, n in top]}", flush=True)
