# SpMM timings on cfg2: Y*X (w=110), Y^T*H (w=110), Y^T*Q (W=660); median of 10.
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, device
from paper_1810_06860_b200.sparse import SparseMatrix, spmm_dev, spmm_t_dev
obs = workloads.cfg2()
A = SparseMatrix.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
rng = np.random.default_rng(0)
X = device.to_device(rng.standard_normal((obs.n, 110)))
H = device.to_device(rng.standard_normal((obs.m, 660)))
out_m = device.empty(obs.m, 110); out_n = device.empty(obs.n, 110); out_w = device.empty(obs.n, 660)
res = []
for name, fn, w in (("csr w=110", lambda: spmm_dev(A, X, out=out_m), 110),
                    ("csc w=110", lambda: spmm_t_dev(A, H[:, :110], out=out_n), 110),
                    ("csc W=660", lambda: spmm_t_dev(A, H, out=out_w), 660)):
    ts = []
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts[2:]))
    res.append(f"{name} {ms*1e3:.0f}us ({A.nnz*w*8/ms/1e9:.0f} GB/s gathered)")
print(sys.argv[1] if len(sys.argv) > 1 else "", " | ".join(res))
