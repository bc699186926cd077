import sys, numpy as np
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg, rsvd
from paper_1810_06860_b200.sparse import SparseMatrix
from paper_1810_06860_b200.rsvd import RsvdParams, qb_error, rsvd_bki, rsvd_pi
rng = np.random.default_rng(5)
M = rng.standard_normal((120, 5)) @ rng.standard_normal((5, 90))
i, j = np.nonzero(np.ones_like(M))
A = SparseMatrix.from_coo(120, 90, i, j, M[i, j])
for rep in range(4):
    for fn in (rsvd_pi, rsvd_bki):
        res, sub = fn(A, RsvdParams(k=5, p=1, s=3, seed=7), allow_fallback=True)
        zr = int(np.sum(np.all(res.U == 0, axis=1)))
        print(rep, fn.__name__, "qb", qb_error(A, res), "zero U rows", zr, np.flatnonzero(np.all(res.U == 0, axis=1))[:12], "fallbacks", sub.fallbacks, flush=True)
# pieces
X = np.random.default_rng(1).standard_normal((120, 8)) @ np.diag([1, 1, 1, 1, 1, 1e-20, 0, 0])
for rep in range(3):
    U, S, V = linalg.oracle_svd_dev(device.to_device(X))
    Uh = device.to_host(U)
    print("oracle_svd rank-def: zero rows", int(np.sum(np.all(Uh == 0, axis=1))), "orth", np.abs(Uh.T @ Uh - np.eye(8)).max(), flush=True)
