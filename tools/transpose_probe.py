# Device CSR->CSC transpose time on cfg2 / cfg4 patterns (median of 5), vs the host stable argsort.
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, device
from paper_1810_06860_b200.sparse import SparseMatrix, ObservationSet, _device_transpose, _Side, _HostSide
for name, gen in (("cfg2", workloads.cfg2), ("cfg4", workloads.cfg4)):
    o = gen()
    A = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split).train_matrix() if name == "cfg4" else \
        SparseMatrix.from_coo(o.m, o.n, o.rows, o.cols, o.values)
    side = _Side(_HostSide(A.indptr, A.indices, A.rows))
    ts = []
    for _ in range(6):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        _device_transpose(side, A.rows, A.cols, A.nnz); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t0 = time.perf_counter(); np.argsort(A.indices, kind="stable"); th = time.perf_counter() - t0
    print(f"{name}: device transpose {np.median(ts[1:])*1e3:.2f} ms, host stable argsort {th*1e3:.0f} ms", flush=True)
