# Host-side profile (cProfile) of the cfg1 SVT loop at eps=1e-3: where the Python time goes.
import cProfile, pstats, sys, time
import torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import completion, workloads
from paper_1810_06860_b200.sparse import ObservationSet
o, _ = workloads.cfg1()
ob = ObservationSet(o.m, o.n, o.rows, o.cols, o.values)
prm = completion.SvtParams(seed=0, epsilon=1e-3)
completion.svt_reference(ob, prm, backend="rsvd-bki"); torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = completion.svt_reference(ob, prm, backend="rsvd-bki")
torch.cuda.synchronize()
pr.disable()
print(f"{res.iterations} iterations in {time.perf_counter() - t0:.3f} s")
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
