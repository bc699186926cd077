import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, completion
from paper_1810_06860_b200.sparse import ObservationSet
o = workloads.cfg4()
obs = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split)
for tdiv, delta in ((10, 1.0), (40, 1.0), (40, 2.0)):
    params = completion.SvtParams(epsilon=0.17, i_reuse=5, q_reuse=10, strategy="reuse-q", seed=0, i_max=25, delta=delta, tau=5.0 * o.n / tdiv)
    torch.cuda.synchronize(); t = time.time()
    try:
        res = completion.svt_fast(obs, params)
    except Exception as e:
        print(tdiv, delta, "failed", type(e).__name__, str(e)[:80], flush=True); continue
    torch.cuda.synchronize()
    loop = sum(tr.wall_time for tr in res.trace)
    rt, ct, vt = obs.subset(1)
    print(f"tau/{tdiv} delta {delta}: {res.iterations} it resid {res.residual:.4e} rank {res.rank} loop {loop:.3f}s -> {res.iterations/loop:.1f} it/s, ks {[t.k for t in res.trace][::3]}, MAE {completion.mae(res.predict(rt, ct), vt):.4f}", flush=True)
