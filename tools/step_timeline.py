# One rsvd_bki step on cfg2 with a host+device timeline of every native call.
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import _native, workloads, profiling
from paper_1810_06860_b200.sparse import SparseMatrix
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki_dev

class TL(profiling.Profiler):
    def run(self, name, meta, fn, args):
        h0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); st = fn(*args); e1.record()
        self.records.append((name, meta, e0, e1, h0, time.perf_counter()))
        return st

obs = workloads.cfg2()
A = SparseMatrix.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
p = RsvdParams(k=100, p=5, s=10, seed=0)
for _ in range(2): rsvd_bki_dev(A, p, omega="device")
torch.cuda.synchronize()
tl = TL(); _native.PROFILER = tl
base = torch.cuda.Event(enable_timing=True); base.record()
h_base = time.perf_counter()
rsvd_bki_dev(A, p, omega="device")
torch.cuda.synchronize(); h_end = time.perf_counter()
_native.PROFILER = None
print(f"host wall {1e3*(h_end-h_base):.2f} ms")
for name, meta, e0, e1, h0, h1 in tl.records:
    print(f"{name:24s} host {1e3*(h0-h_base):8.2f}..{1e3*(h1-h_base):8.2f}  gpu {base.elapsed_time(e0):8.2f}..{base.elapsed_time(e1):8.2f}  ({e0.elapsed_time(e1):.3f} ms)")
