import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, completion
from paper_1810_06860_b200.sparse import ObservationSet
import oracle
t = time.time(); o = workloads.cfg4(); print("gen", time.time() - t, flush=True)
obs = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split)
imax = int(sys.argv[1]) if len(sys.argv) > 1 else 20
params = completion.SvtParams(epsilon=0.17, i_reuse=5, q_reuse=10, strategy="reuse-q", seed=0, i_max=imax, delta=1.0)
for rep in range(2):
    torch.cuda.synchronize(); t = time.time()
    res = completion.svt_fast(obs, params)
    torch.cuda.synchronize(); dt = time.time() - t
    loop = sum(tr.wall_time for tr in res.trace)
    print(f"gpu rep{rep}: {res.iterations} it resid {res.residual:.6e} rank {res.rank} total {dt:.2f}s loop {loop:.3f}s -> {res.iterations/loop:.2f} it/s", flush=True)
for tr in res.trace: print("  ", tr.iteration, tr.k, tr.r, tr.p, tr.q, f"{tr.residual:.10e}", tr.svd_source, f"{tr.wall_time*1e3:.1f}ms")
r, c, v = obs.subset(0)
ni = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t = time.time()
out = oracle.complete(o.m, o.n, r, c, v, oracle.SvtConfig(epsilon=0.17, i_reuse=5, q_reuse=10, strategy="reuse-q", seed=0, i_max=ni, delta=1.0))
dt = time.time() - t
print(f"oracle {ni} it: {dt:.1f}s -> {ni/dt:.4f} it/s (incl setup)")
for tr in out.trace: print("  ", tr[0], tr[1], tr[2], tr[3], tr[4], f"{tr[5]:.10e}", tr[6])
