"""Is the sketch itself reproducible?  Omega(seed, n, w) drawn repeatedly (device generator; host draw + upload +
transpose), and _krylov_orth's outputs from a freshly drawn Omega each repetition."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1810_06860_b200 import device, linalg, rsvd, workloads
from paper_1810_06860_b200.sparse import ObservationSet
o4 = workloads.cfg4()
A = ObservationSet(o4.m, o4.n, o4.rows, o4.cols, o4.values, o4.split).train_matrix()
A.pattern(); A.device_values()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
w = int(sys.argv[2]) if len(sys.argv) > 2 else 32
prm = rsvd.RsvdParams(k=w - 5, p=2, s=5, seed=1261)
fb = rsvd._Fallback(True, "x")
ref = None
bad = {}
for rep in range(n):
    Om = rsvd._omega(prm.seed, A.cols, w, "device")
    H, Q, lu, probe = rsvd._krylov_orth(A, Om, prm, True, False, True, fb, keep_T=True)
    T = Q.T_all
    st = [("Om", Om), ("H0 = LU(Y Om)", H[:, 0:w]), ("T0 = Y^T H0", T[:, 0:w]), ("H1 = LU(Y T0)", H[:, w:2 * w]),
          ("T1 = Y^T H1", T[:, w:2 * w]), ("H2 = LU(Y T1)", H[:, 2 * w:3 * w]), ("T2", T[:, 2 * w:3 * w]), ("Q.base", Q.base), ("Q.Rinv", Q.Rinv)]
    st = [(a_, b_.clone()) for a_, b_ in st]
    lus = device.to_host(lu).reshape(-1, 4)
    if ref is None:
        ref = st
    else:
        for (name, a), (_, b) in zip(ref, st):
            if not torch.equal(a, b):
                bad.setdefault(name, []).append((rep, float((a - b).abs().max()), lus[:, 0].tolist()))
                break
print(f"w={w}: krylov_orth with a fresh Omega per repetition, first differing output:", {k_: (len(v), v[:4]) for k_, v in bad.items()})
