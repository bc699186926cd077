import sys, time, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import completion, workloads
from paper_1810_06860_b200.sparse import ObservationSet
o1, _ = workloads.cfg1()
obs1 = ObservationSet(o1.m, o1.n, o1.rows, o1.cols, o1.values)
for eps in (0.05, 1e-3):
    prm = completion.SvtParams(seed=0, epsilon=eps)
    completion.svt_reference(obs1, prm, backend="rsvd-bki")
    r = []
    for _ in range(3):
        res = completion.svt_reference(obs1, prm, backend="rsvd-bki"); torch.cuda.synchronize()
        r.append(res.iterations / sum(t.wall_time for t in res.trace))
    print("cfg1", eps, [round(x) for x in r], res.iterations, res.residual, flush=True)
