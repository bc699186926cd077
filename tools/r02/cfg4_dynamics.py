"""cfg4 SVT dynamics per (tau, delta, eps): the verbose trace (k, r, p, q,
residual) of the first iterations, so the rank growth against the residual
is visible.  CFG="tdiv:delta:eps[:imax]" (tau = 5n/tdiv); one run per process."""
import os, sys, time
os.environ["LR_SVT_VERBOSE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1810_06860_b200 import completion, workloads
from paper_1810_06860_b200.sparse import ObservationSet

parts = os.environ.get("CFG", "10:1.0:0.17:60").split(":")
tdiv, delta, eps = float(parts[0]), float(parts[1]), float(parts[2])
imax = int(parts[3]) if len(parts) > 3 else 60
o = workloads.cfg4()
obs = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split)
tau = 5.0 * o.n / tdiv if tdiv > 0 else None
dl = delta if delta > 0 else None
print(f"== tau={tau} delta={dl} eps={eps} imax={imax}", flush=True)
t = time.time()
try:
    res = completion.svt_fast(obs, completion.SvtParams(epsilon=eps, i_reuse=50, q_reuse=10, strategy="reuse-q",
                                                        seed=0, i_max=imax, tau=tau, delta=dl))
    rt, ct, vt = obs.subset(1)
    print(f"done {res.iterations} it conv={res.converged} rank={res.rank} resid={res.residual:.5e} "
          f"MAE={completion.mae(res.predict(rt, ct), vt):.5f} {time.time()-t:.1f}s", flush=True)
except Exception as e:
    print("FAILED", type(e).__name__, str(e)[:200], f"{time.time()-t:.1f}s", flush=True)
