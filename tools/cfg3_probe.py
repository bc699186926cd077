# cfg3 image-inpainting shape: GPU svt_fast(reuse-u) vs the CPU oracle (timing + parity).
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import oracle
from paper_1810_06860_b200 import completion, workloads
from paper_1810_06860_b200.sparse import ObservationSet
o, X = workloads.cfg3()
ob = ObservationSet(o.m, o.n, o.rows, o.cols, o.values)
for eps in (0.05, 0.01):
    prm = completion.SvtParams(strategy="reuse-u", i_reuse=100, q_reuse=10, seed=0, epsilon=eps)
    completion.svt_fast(ob, prm); torch.cuda.synchronize()
    t0 = time.perf_counter(); res = completion.svt_fast(ob, prm); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    loop = sum(t.wall_time for t in res.trace)
    print(f"GPU eps={eps}: {res.iterations} it, loop {loop*1e3:.1f} ms ({res.iterations/loop:.1f} it/s), total {dt*1e3:.1f} ms, "
          f"rank {res.rank}, resid {res.residual:.6e}, ks {[t.k for t in res.trace][:12]}", flush=True)
    t0 = time.perf_counter()
    ref = oracle.complete(o.m, o.n, o.rows, o.cols, o.values,
                          oracle.SvtConfig(strategy="reuse-u", i_reuse=100, q_reuse=10, seed=0, epsilon=eps))
    dt = time.perf_counter() - t0
    print(f"CPU eps={eps}: {ref.iterations} it, {dt:.1f} s ({ref.iterations/dt:.2f} it/s), rank {ref.rank}, "
          f"resid {ref.residual:.6e}; residual diffs {np.max(np.abs(np.array([t.residual for t in res.trace]) - np.array([t[5] for t in ref.trace]))) if ref.iterations == res.iterations else 'iteration mismatch'}", flush=True)
