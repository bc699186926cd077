# Kernel breakdown of the cfg1 SVT loop (reference defaults and eps=1e-3), events around every native call.
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import _native, completion, profiling, workloads, linalg
from paper_1810_06860_b200.sparse import ObservationSet
o, _ = workloads.cfg1()
ob = ObservationSet(o.m, o.n, o.rows, o.cols, o.values)
for method in ("syevd", "syevj"):
    linalg.EIG_METHOD = method
    prm = completion.SvtParams(seed=0, epsilon=1e-3)
    completion.svt_reference(ob, prm, backend="rsvd-bki")
    torch.cuda.synchronize()
    t0 = time.perf_counter(); res = completion.svt_reference(ob, prm, backend="rsvd-bki"); torch.cuda.synchronize()
    loop = sum(t.wall_time for t in res.trace)
    prof = profiling.Profiler(); _native.PROFILER = prof
    completion.svt_reference(ob, prm, backend="rsvd-bki"); torch.cuda.synchronize(); _native.PROFILER = None
    summ = prof.summary()
    tot = sum(d["ms"] for d in summ.values())
    print(f"{method}: {res.iterations} it, loop {loop*1e3:.1f} ms ({res.iterations/loop:.0f} it/s); kernel time {tot:.1f} ms")
    for name, d in sorted(summ.items(), key=lambda kv: -kv[1]["ms"])[:8]:
        print(f"   {name:24s} {d['calls']:5d} calls {d['ms']:8.2f} ms")
