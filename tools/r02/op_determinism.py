"""Which native op is not deterministic at w = 32 / 48?  Each op repeated on fixed inputs, outputs compared bit for bit."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1810_06860_b200 import device, linalg, workloads
from paper_1810_06860_b200.sparse import ObservationSet, spmm_dev, spmm_t_dev
o4 = workloads.cfg4()
A = ObservationSet(o4.m, o4.n, o4.rows, o4.cols, o4.values, o4.split).train_matrix()
A.pattern(); A.device_values()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
rng = np.random.default_rng(0)
for w in (32, 48):
    X = device.to_device(rng.standard_normal((A.cols, w)))
    H = device.to_device(rng.standard_normal((A.rows, w)))
    Hw = device.to_device(rng.standard_normal((A.rows, 3 * w)))
    def rep(name, fn):
        ref = fn().clone()
        bad = 0
        for _ in range(n):
            out = fn()
            bad += not torch.equal(out, ref)
        print(f"w={w} {name}: {bad} of {n} differ", flush=True)
    def lu():
        B = H.clone()
        linalg.lu_pl_dev(B)
        return B
    rep("lu_pl", lu)
    rep("gram", lambda: linalg.gram_dev(Hw))
    G = linalg.gram_dev(Hw)
    rep("potrf_inv", lambda: linalg.potrf_inv_dev(G.clone())[1])
    rep("sym_eig", lambda: linalg.sym_eig_dev(G.clone(), symmetrize=False)[0])
    R = linalg.potrf_inv_dev(G.clone())[1]
    rep("matmul upper", lambda: linalg.matmul_dev(Hw, R, b_upper=True))
    rep("matmul_tn", lambda: linalg.matmul_tn_dev(Hw, H))
