"""The tail of rsvd_bki (orth + projection + eigSVD + lifts) on a FIXED Krylov block H (w = 32, p = 2, W = 96):
which intermediate first differs between repetitions?"""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1810_06860_b200 import device, linalg, rsvd, workloads
from paper_1810_06860_b200.sparse import ObservationSet, spmm_dev, spmm_t_dev
o4 = workloads.cfg4()
A = ObservationSet(o4.m, o4.n, o4.rows, o4.cols, o4.values, o4.split).train_matrix()
A.pattern(); A.device_values()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
k, p = 27, 2
prm = rsvd.RsvdParams(k=k, p=p, s=5, seed=1261)
fb = rsvd._Fallback(True, "x")
Om = rsvd._omega(prm.seed, A.cols, k + 5, "device")
H0, Q0, lu0, probe0 = rsvd._krylov_orth(A, Om, prm, True, False, True, fb, keep_T=False)
torch.cuda.synchronize()
H0 = H0.clone()
ref = None
bad = {}
for rep in range(n):
    H = H0.clone()
    Q, probe = linalg.orth_speculative_dev(H, lazy_last=True)
    stages = [("orth.base", Q.base.clone()), ("orth.Rinv", Q.Rinv.clone()), ("orth.R1inv", Q.R1inv.clone())]
    Bt = spmm_t_dev(A, Q.base)
    stages.append(("Bt = Y^T Q1", Bt.clone()))
    W = Bt.shape[1]
    idx = np.arange(W - 1, W - k - 1, -1)
    fin, V, U, cols = linalg.eig_svd_congruent_dev(Bt, Q.Rinv, idx, defer=True)
    S = fin()
    stages += [("eig V", V.clone()), ("eig S", torch.from_numpy(S.copy())), ("eig U", U.clone())]
    if ref is None:
        ref = stages
    else:
        for (name, a), (_, b) in zip(ref, stages):
            if not torch.equal(a, b):
                d = float((a.double() - b.double()).abs().max())
                bad.setdefault(name, []).append((rep, d))
                break
print({k_: (len(v), v[:3]) for k_, v in bad.items()})
