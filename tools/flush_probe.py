import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads
from paper_1810_06860_b200.sparse import SparseMatrix
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki_dev
obs = workloads.cfg2()
A = SparseMatrix.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
p = RsvdParams(k=100, p=5, s=10, seed=0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(2): rsvd_bki_dev(A, p, omega="device")
for mode in ("plain", "flush", "plain", "flush"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        if mode == "flush": flush.zero_()
        rsvd_bki_dev(A, p, omega="device")
    e1.record(); torch.cuda.synchronize()
    print(mode, e0.elapsed_time(e1) / 3, "ms/step")
