# ncu target: the cfg4 CSR product at one width, hot-row staged (default) or plain (LR_SPMM_HOT=0).
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, device, sparse
from paper_1810_06860_b200.sparse import ObservationSet, spmm_dev
w = int(sys.argv[1]) if len(sys.argv) > 1 else 22
o = workloads.cfg4()
A = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split).train_matrix()
A.pattern(); A.device_values()
sparse.HOT_MIN_SHARE = 0.0
X = device.to_device(np.random.default_rng(0).standard_normal((A.cols, w)))
for _ in range(3):
    spmm_dev(A, X)
torch.cuda.synchronize()
print("ok")
