# SDDMM (project_pattern_dev, the SVT step's kernel family) on cfg4 at SVT ranks, median of 10.
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, device
from paper_1810_06860_b200.sparse import ObservationSet, project_pattern_dev
o = workloads.cfg4()
A = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split).train_matrix()
A.pattern(); A.device_values()
rng = np.random.default_rng(0)
out = device.vector(A.nnz)
res = []
for r in (10, 20, 40, 84, 160):
    U = device.to_device(rng.standard_normal((A.rows, r))); V = device.to_device(rng.standard_normal((A.cols, r)))
    S = device.f64_buffer(rng.random(r))
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); project_pattern_dev(U, S, V, A, out=out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts[2:]))
    res.append(f"r={r} {ms*1e3:.0f}us ({A.nnz*r*8/ms/1e9:.1f} TB/s V-gather)")
print(sys.argv[1] if len(sys.argv) > 1 else "", " | ".join(res))
