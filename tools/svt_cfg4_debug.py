import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, completion
from paper_1810_06860_b200.sparse import ObservationSet
t = time.time(); o = workloads.cfg4(); print("gen", time.time() - t, flush=True)
obs = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split)
imax = int(sys.argv[1]) if len(sys.argv) > 1 else 20
params = completion.SvtParams(epsilon=0.17, i_reuse=50, q_reuse=10, strategy="reuse-q", seed=0, i_max=imax)
torch.cuda.synchronize(); t = time.time()
res = completion.svt_fast(obs, params)
torch.cuda.synchronize(); dt = time.time() - t
print(f"{res.iterations} it conv {res.converged} resid {res.residual:.6e} rank {res.rank} total {dt:.2f}s svd {res.svd_time:.2f} upd {res.update_time:.2f}")
for tr in res.trace: print(tr.iteration, tr.k, tr.r, tr.p, tr.q, f"{tr.residual:.6e}", tr.svd_source, f"{tr.wall_time*1e3:.1f}ms")
print(res.events[:20])
r, c, v = obs.subset(1)
print("held-out MAE", completion.mae(res.predict(r, c), v))
