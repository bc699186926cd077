# Where do bench steps lose time vs the isolated timeline? per-step events, GC on/off, flush on/off.
import gc, sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads
from paper_1810_06860_b200.sparse import SparseMatrix
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki_dev
obs = workloads.cfg2()
A = SparseMatrix.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
p = RsvdParams(k=100, p=5, s=10, seed=0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(3): rsvd_bki_dev(A, p, omega="device")
for gc_on in (True, False):
    if not gc_on: gc.disable()
    for keep in (True, False):
        torch.cuda.synchronize()
        evs = []
        t0 = time.perf_counter()
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = rsvd_bki_dev(A, p, omega="device")
            e1.record(); evs.append((e0, e1))
            if not keep: del r
        torch.cuda.synchronize()
        print(f"gc={gc_on} keep={keep}: wall {(time.perf_counter()-t0)/5*1e3:.2f} ms/step, device", [round(a.elapsed_time(b), 2) for a, b in evs], flush=True)
    gc.enable()
