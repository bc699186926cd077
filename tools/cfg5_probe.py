# cfg5 scale-up shape (1e6 x 2e5, 2e8 observed): host generation, device pattern build, one rsvd_bki at
# k=300 s=5 p=3 (W=1220) and the first SVT-step kernel; invariants checked on the device result.
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, device
from paper_1810_06860_b200.sparse import SparseMatrix
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki_dev
t0 = time.perf_counter()
o = workloads.cfg5()
t1 = time.perf_counter()
print(f"generate: {t1 - t0:.1f} s, nnz {o.rows.size}", flush=True)
# the generator already emits unique, row-major sorted keys: CSR directly
indptr = np.zeros(o.m + 1, dtype=np.int64)
np.cumsum(np.bincount(o.rows, minlength=o.m), out=indptr[1:])
A = SparseMatrix(o.m, o.n, indptr, o.cols, o.values)
del o
t2 = time.perf_counter()
print(f"csr (host): {t2 - t1:.1f} s", flush=True)
torch.cuda.synchronize(); t3 = time.perf_counter()
A.pattern(); A.device_values(); torch.cuda.synchronize()
t4 = time.perf_counter()
print(f"device pattern + values (upload + device transpose): {t4 - t3:.2f} s", flush=True)
p = RsvdParams(k=300, p=3, s=5, seed=0)
for rep in range(2):
    torch.cuda.synchronize(); t5 = time.perf_counter()
    res, Q, _ = rsvd_bki_dev(A, p)
    torch.cuda.synchronize(); t6 = time.perf_counter()
    print(f"rsvd_bki k=300 p=3 (W=1220): {t6 - t5:.3f} s  S[0]={res.S_host[0]:.6e} S[299]={res.S_host[299]:.6e}", flush=True)
S = res.S_host
U = res.U
for rep in range(2):
    torch.cuda.synchronize(); t5 = time.perf_counter()
    r32, _, _ = rsvd_bki_dev(A, p, precision="fp32")
    torch.cuda.synchronize(); t6 = time.perf_counter()
    print(f"rsvd_bki fp32 mode k=300 p=3 (W=1220): {t6 - t5:.3f} s  max rel S diff vs fp64 "
          f"{np.max(np.abs(r32.S_host - S) / S):.2e}", flush=True)
del r32
G = (U.T @ U).cpu().numpy()
print("descending:", bool(np.all(np.diff(S) <= 0)), " ||U^T U - I|| =", np.abs(G - np.eye(G.shape[0])).max(),
      " peak mem GB:", torch.cuda.max_memory_allocated() / 1e9, flush=True)
