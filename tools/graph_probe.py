# Repeated rsvd_bki on one small matrix (cfg1 shape): eager speculative path vs captured-graph replay
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import rsvd, workloads
from paper_1810_06860_b200.sparse import SparseMatrix
o, _ = workloads.cfg1()
A = SparseMatrix.from_coo(o.m, o.n, o.rows, o.cols, o.values)
for graphs in (False, True):
    rsvd.USE_GRAPHS = graphs
    prm = rsvd.RsvdParams(k=11, p=3, s=5, seed=0)
    t0 = time.perf_counter(); rsvd.rsvd_bki_dev(A, prm); torch.cuda.synchronize(); first = time.perf_counter() - t0
    ts = []
    for i in range(50):
        prm = rsvd.RsvdParams(k=11, p=3, s=5, seed=i)
        t0 = time.perf_counter(); rsvd.rsvd_bki_dev(A, prm); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(f"graphs={graphs}: first call {first*1e3:.2f} ms, steady median {np.median(ts)*1e3:.3f} ms")
