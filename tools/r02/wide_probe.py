"""The wide Y^T Q product of the cfg4 SVT loop (W = 110 .. 330 columns): time
per call against the column-chunk width (LR_SPMM_CHUNK, read once per
process) and the L2-gather rate."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1810_06860_b200 import workloads, device
from paper_1810_06860_b200.sparse import ObservationSet, spmm_t_dev, spmm_dev

o = workloads.cfg4()
A = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split).train_matrix()
A.pattern(); A.device_values()
rng = np.random.default_rng(0)
tag = os.environ.get("LR_SPMM_CHUNK", "auto")
for W in (110, 165, 220, 330):
    H = device.to_device(rng.standard_normal((A.rows, W)))
    X = device.to_device(rng.standard_normal((A.cols, W)))
    res = []
    for name, fn in (("csc Y^T Q", lambda: spmm_t_dev(A, H)), ("csr Y X", lambda: spmm_dev(A, X))):
        ts = []
        for _ in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts[2:]))
        res.append(f"{name} {ms*1e3:7.0f} us {A.nnz*W*8/ms/1e9:6.2f} TB/s")
    print(f"chunk={tag} W={W}: " + " | ".join(res), flush=True)
