import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle
from paper_1810_06860_b200 import device, linalg, rsvd
from paper_1810_06860_b200.sparse import SparseMatrix, spmm, spmm_t
g = dict(np.load('/root/repo/tests/golden/reference_golden.npz'))
A = SparseMatrix.from_coo(300, 200, g["rs_i"], g["rs_j"], g["rs_v"])
D = A.densify()
X = np.random.default_rng(0).standard_normal((300, 15))
print("spmm_t err", np.abs(spmm_t(A, X) - D.T @ X).max())
Z = np.random.default_rng(1).standard_normal((200, 15))
print("spmm err", np.abs(spmm(A, Z) - D @ Z).max())
H = D @ Z
print("lu err", np.abs(linalg.lu_pl(H) - oracle.pivoted_lower(H)).max())
for om in ("host", "device"):
    res, _ = rsvd.rsvd_pi(A, rsvd.RsvdParams(k=10, p=2, s=5, seed=3), omega=om)
    print(om, "pi S", np.abs(res.S - g["rs_pi_S"]).max())
