"""The Krylov chain of rsvd_bki on column slices of one m x W block (w = 32, p = 2), stage by stage: which stage's
output first differs between repetitions?"""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1810_06860_b200 import device, linalg, rsvd, workloads
from paper_1810_06860_b200.sparse import ObservationSet, spmm_dev, spmm_t_dev
o4 = workloads.cfg4()
A = ObservationSet(o4.m, o4.n, o4.rows, o4.cols, o4.values, o4.split).train_matrix()
A.pattern(); A.device_values()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
w, p = 32, 2
W = w * (p + 1)
Om = device.to_device(np.random.default_rng(0).standard_normal((A.cols, w)))
ref = None
bad = {}
for rep in range(n):
    H = device.empty(A.rows, W)
    T = device.empty(A.cols, w)
    st = device.vector(4 * (p + 1))
    stages = []
    spmm_dev(A, Om, out=H[:, 0:w]); stages.append(("spmm0", H[:, 0:w].clone()))
    rsvd._lu_block_async(H[:, 0:w], st[0:3]); stages.append(("lu0", H[:, 0:w].clone()))
    for i in range(1, p + 1):
        spmm_t_dev(A, H[:, (i - 1) * w:i * w], out=T); stages.append((f"spmm_t{i}", T.clone()))
        spmm_dev(A, T, out=H[:, i * w:(i + 1) * w]); stages.append((f"spmm{i}", H[:, i * w:(i + 1) * w].clone()))
        rsvd._lu_block_async(H[:, i * w:(i + 1) * w], st[4 * i:4 * i + 3]); stages.append((f"lu{i}", H[:, i * w:(i + 1) * w].clone()))
    G = linalg.gram_dev(H); stages.append(("gram", G.clone()))
    if ref is None:
        ref = stages
    else:
        for (name, a), (_, b) in zip(ref, stages):
            if not torch.equal(a, b):
                bad[name] = bad.get(name, 0) + 1
                break
print(f"w={w} p={p}: first differing stage over {n} repetitions: {bad}")
