# Targets for ncu captures.  Default: one warm rsvd_bki on cfg2 (fp64, then fp32 mode) and a few SVT
# iterations on cfg1.  NCU_ONLY=fp32: only the fp32-mode call; NCU_ONLY=gemm_nn: one H R^-1 product
# (100000 x 660 x 660, upper-triangular B) -- so a kernel-name filter plus -c 1 selects them.
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, completion, device, linalg
from paper_1810_06860_b200.sparse import SparseMatrix, ObservationSet
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki_dev
only = os.environ.get("NCU_ONLY", "")
if only == "gemm_nn":
    rng = np.random.default_rng(0)
    H = device.to_device(rng.standard_normal((100000, 660)))
    R = device.to_device(np.triu(rng.standard_normal((660, 660))))
    linalg.matmul_dev(H, R, b_upper=True)
    torch.cuda.synchronize()
    print("ok")
    sys.exit(0)
obs = workloads.cfg2()
A = SparseMatrix.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
p = RsvdParams(k=100, p=5, s=10, seed=0)
if only != "fp32":
    rsvd_bki_dev(A, p)
    torch.cuda.synchronize()
rsvd_bki_dev(A, p, precision="fp32")
torch.cuda.synchronize()
if only != "fp32":
    o, _ = workloads.cfg1()
    completion.svt_reference(ObservationSet(o.m, o.n, o.rows, o.cols, o.values),
                             completion.SvtParams(seed=0, i_max=3), backend="rsvd-bki")
    torch.cuda.synchronize()
print("ok")
