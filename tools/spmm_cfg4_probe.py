# SpMM on the cfg4 rating shape at the widths the SVT loop uses (median of 8).
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, device
from paper_1810_06860_b200.sparse import ObservationSet, spmm_dev, spmm_t_dev
o = workloads.cfg4()
A = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split).train_matrix()
A.pattern(); A.device_values()
rng = np.random.default_rng(0)
print(f"cfg4 train nnz {A.nnz}, rows {A.rows}, cols {A.cols}, csr items {A.pattern().csr.n_items}, csc items {A.pattern().csc.n_items}")
for w in tuple(int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "11,16,22,33,45,66,89,132,264".split(","))):
    X = device.to_device(rng.standard_normal((A.cols, w)))
    H = device.to_device(rng.standard_normal((A.rows, w)))
    res = []
    for name, fn in (("csr", lambda: spmm_dev(A, X)), ("csc", lambda: spmm_t_dev(A, H))):
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts[2:]))
        res.append(f"{name} {ms*1e3:7.0f}us {A.nnz*w*8/ms/1e9:6.2f}TB/s")
    print(f"w={w:3d}: " + " | ".join(res), flush=True)
