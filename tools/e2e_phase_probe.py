# Phases of the e2e call (pinned host matrix, device mirror dropped): pattern upload + device transpose,
# value upload + CSC gather, the rsvd_bki compute, result download.
import sys, time
import torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, workloads
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki, rsvd_bki_dev
from paper_1810_06860_b200.sparse import SparseMatrix

obs = workloads.cfg2()
A = SparseMatrix.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
prm = RsvdParams(k=100, p=5, s=10, seed=0)
A.pin_memory()
for _ in range(3):
    A.drop_device(); rsvd_bki(A, prm)
for _ in range(4):
    A.drop_device()
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    A.pattern(); torch.cuda.synchronize(); t.append(time.perf_counter())
    A.device_values(); torch.cuda.synchronize(); t.append(time.perf_counter())
    res, Q, _ = rsvd_bki_dev(A, prm); torch.cuda.synchronize(); t.append(time.perf_counter())
    h = res.to_host(); torch.cuda.synchronize(); t.append(time.perf_counter())
    d = [round((b - a) * 1e3, 2) for a, b in zip(t, t[1:])]
    print(f"pattern {d[0]} ms, values {d[1]} ms, compute {d[2]} ms, download {d[3]} ms, total {round((t[-1]-t[0])*1e3, 2)}", flush=True)
x = torch.empty(64 * 2**20 // 8, dtype=torch.float64, pin_memory=True)
g = torch.empty_like(x, device="cuda")
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); g.copy_(x, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter(); x.copy_(g, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"pinned 64 MB: H2D {64/1024/(t1-t0):.1f} GB/s, D2H {64/1024/(t2-t1):.1f} GB/s")
