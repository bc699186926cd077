# SVT on cfg1 (defaults) and cfg4 (rating defaults) on the GPU: timing + trace.
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, completion
from paper_1810_06860_b200.sparse import ObservationSet
which = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
imax = int(sys.argv[2]) if len(sys.argv) > 2 else 500
if which == "cfg1":
    o, _ = workloads.cfg1()
    params = completion.SvtParams(seed=0, i_max=imax)
else:
    t = time.time(); o = workloads.cfg4(); print("gen", time.time() - t, flush=True)
    params = completion.SvtParams(epsilon=0.17, i_reuse=50, q_reuse=10, strategy="reuse-q", seed=0, i_max=imax)
obs = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split)
for rep in range(2):
    torch.cuda.synchronize(); t = time.time()
    res = completion.svt_fast(obs, params)
    torch.cuda.synchronize(); dt = time.time() - t
    loop = sum(tr.wall_time for tr in res.trace)
    print(f"{which} rep{rep}: {res.iterations} it, converged {res.converged}, resid {res.residual:.6e}, rank {res.rank}, "
          f"total {dt:.2f}s, loop {loop:.2f}s, {res.iterations/loop:.2f} it/s, svd {res.svd_time:.2f}s update {res.update_time:.2f}s", flush=True)
for tr in res.trace[:8] + res.trace[-4:]:
    print(tr.iteration, tr.k, tr.r, tr.p, tr.q, f"{tr.residual:.6e}", tr.svd_source, f"{tr.wall_time*1e3:.1f}ms")
if which != "cfg1":
    r, c, v = obs.subset(1)
    pred = res.predict(r, c)
    print("held-out MAE", completion.mae(pred, v))
