"""cfg4: which (tau, delta) converge to the rating tolerance eps = 0.17 with
the CLI's rating recycling (reuse-q, i_reuse = 50, q_reuse = 10)?  One line
per setting: iterations, converged, final rank, residual, held-out MAE."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_1810_06860_b200 import completion, workloads
from paper_1810_06860_b200.sparse import ObservationSet

o = workloads.cfg4()
obs = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split)
rt, ct, vt = obs.subset(1)
n = o.n
imax = int(os.environ.get("IMAX", "300"))
grid = [(float(a), float(b)) for a, b in (x.split(":") for x in os.environ.get(
    "GRID", "10:1.0,20:1.0,40:1.0,80:1.0,10:1.9,20:1.9,40:1.9,80:1.9,160:1.9").split(","))]
for tdiv, delta in grid:
    p = completion.SvtParams(epsilon=0.17, i_reuse=50, q_reuse=10, strategy="reuse-q", seed=0, i_max=imax,
                             tau=5.0 * n / tdiv, delta=delta)
    torch.cuda.synchronize(); t = time.time()
    try:
        res = completion.svt_fast(obs, p)
    except Exception as e:
        print(f"tau=5n/{tdiv:g} delta={delta}: FAILED {type(e).__name__} {str(e)[:100]} ({time.time()-t:.1f}s)", flush=True)
        continue
    torch.cuda.synchronize(); dt = time.time() - t
    ks = [tr.k for tr in res.trace]; rs = [tr.residual for tr in res.trace]
    print(f"tau=5n/{tdiv:g} delta={delta}: {res.iterations} it conv={res.converged} rank={res.rank} "
          f"resid={res.residual:.4e} MAE={completion.mae(res.predict(rt, ct), vt):.5f} {dt:.1f}s "
          f"k[::10]={ks[::10]} resid[::10]={[round(x, 3) for x in rs[::10]]}", flush=True)
