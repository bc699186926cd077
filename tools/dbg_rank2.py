import sys, numpy as np
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg, rsvd
from paper_1810_06860_b200.errors import RankDeficiencyError
from paper_1810_06860_b200.sparse import SparseMatrix, spmm_dev, spmm_t_dev
from paper_1810_06860_b200.rsvd import RsvdParams, _Fallback, _lu_block, _omega, _windowed_small_svd
rng = np.random.default_rng(5)
M = rng.standard_normal((120, 5)) @ rng.standard_normal((5, 90))
i, j = np.nonzero(np.ones_like(M))
A = SparseMatrix.from_coo(120, 90, i, j, M[i, j])
def z(name, X):
    h = device.to_host(X)
    print(f"{name}: shape {h.shape} zero rows {int(np.sum(np.all(h == 0, axis=1)))} finite {np.isfinite(h).all()}", flush=True)
params = RsvdParams(k=5, p=1, s=3, seed=7)
fb = _Fallback(True, "x")
Om = _omega(7, 90, 8, "device"); z("Om", Om)
Q = spmm_dev(A, Om); z("Q0", Q)
T = device.empty(90, 8)
_lu_block(Q, fb); z("Q lu", Q)
spmm_t_dev(A, Q, out=T); z("T", T)
spmm_dev(A, T, out=Q); z("Q1", Q)
try:
    _, _, Q, _ = linalg.eig_svd_dev(Q)
    print("eig_svd ok")
except RankDeficiencyError as exc:
    print("eig_svd rank:", exc)
    Q = linalg.oracle_svd_dev(Q)[0]
z("Qb", Q)
Bt = spmm_t_dev(A, Q); z("Bt", Bt)
idx = np.arange(7, 2, -1)
try:
    linalg.eig_svd_dev(Bt, cols=idx)
except RankDeficiencyError as exc:
    print("eig_svd(Bt) rank:", exc)
z("Qb after eig_svd(Bt)", Q)
G = linalg.gram_dev(Bt); z("Qb after gram", Q)
Vx, dx = linalg.sym_eig_dev(G, symmetrize=False); z("Qb after sym_eig", Q)
Ud, Sd, Vd = linalg.oracle_svd_dev(Bt); z("Qb after oracle_svd(Bt)", Q)
S_sel, Vsel, Usel = _windowed_small_svd(Bt, idx, fb); z("Vsel", Vsel); z("Usel", Usel); z("Qb after windowed", Q)
U = linalg.matmul_dev(Q, Vsel); z("U", U)
print("---- bisect on a fresh process state is not possible; re-run the fallback pieces")
