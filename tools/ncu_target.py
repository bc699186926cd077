# One warm rsvd_bki on cfg2 and a few SVT iterations on cfg1, for ncu captures.
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, completion
from paper_1810_06860_b200.sparse import SparseMatrix, ObservationSet
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki_dev
obs = workloads.cfg2()
A = SparseMatrix.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
p = RsvdParams(k=100, p=5, s=10, seed=0)
rsvd_bki_dev(A, p)
torch.cuda.synchronize()
o, _ = workloads.cfg1()
completion.svt_reference(ObservationSet(o.m, o.n, o.rows, o.cols, o.values), completion.SvtParams(seed=0, i_max=3),
                         backend="rsvd-bki")
torch.cuda.synchronize()
print("ok")
