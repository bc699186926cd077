# Find what makes an occasional cfg2 step slow: per-step wall time and native-call event times.
import gc, sys, time
import torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import _native, profiling, workloads
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki_dev
from paper_1810_06860_b200.sparse import SparseMatrix

obs = workloads.cfg2()
A = SparseMatrix.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
prm = RsvdParams(k=100, p=5, s=10, seed=0)
A.pattern(); A.device_values()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(3):
    rsvd_bki_dev(A, prm, omega="device")
torch.cuda.synchronize()
gc.disable()
steps = []
for i in range(10):
    prof = profiling.Profiler()
    _native.PROFILER = prof
    flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = rsvd_bki_dev(A, prm, omega="device")
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    _native.PROFILER = None
    recs = [(n, a.elapsed_time(b)) for n, _, a, b in prof.records]
    steps.append((wall, recs))
    print(f"step {i}: wall {wall:.2f} ms native {sum(t for _, t in recs):.2f} ms  "
          f"alloc {torch.cuda.memory_allocated() / 2**30:.2f} GB reserved {torch.cuda.memory_reserved() / 2**30:.2f} GB",
          flush=True)
base = steps[-1][1]
for i, (wall, recs) in enumerate(steps):
    for k, (n, t) in enumerate(recs):
        if k < len(base) and t > 1.5 * base[k][1] + 0.2:
            print(f"  step {i} call {k} {n}: {t:.2f} ms vs {base[k][1]:.2f}")
# gaps between consecutive native calls (host time) in the slowest step
