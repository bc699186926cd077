# Per-call CUDA-event table of one cfg2 rsvd_bki step in fp64 and fp32 mode.
import sys
import torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import _native, profiling, workloads
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki_dev
from paper_1810_06860_b200.sparse import SparseMatrix

obs = workloads.cfg2()
A = SparseMatrix.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
prm = RsvdParams(k=100, p=5, s=10, seed=0)
for prec in ("fp64", "fp32", "fp64", "fp32"):
    rsvd_bki_dev(A, prm, precision=prec)
    torch.cuda.synchronize()
    prof = profiling.Profiler()
    _native.PROFILER = prof
    rsvd_bki_dev(A, prm, precision=prec)
    torch.cuda.synchronize()
    _native.PROFILER = None
    tot = 0.0
    for name, meta, e0, e1 in prof.records:
        ms = e0.elapsed_time(e1)
        tot += ms
        if ms > 0.05:
            print(f"{prec} {name:24s} {ms:8.3f} ms  {meta}")
    print(f"{prec} total native {tot:.2f} ms\n", flush=True)
