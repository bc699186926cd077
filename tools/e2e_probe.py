# Where the e2e rsvd_bki call spends its time (pinned host matrix).
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import workloads, device
from paper_1810_06860_b200.sparse import SparseMatrix
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki_dev
obs = workloads.cfg2()
A = SparseMatrix.from_coo(obs.m, obs.n, obs.rows, obs.cols, obs.values)
p = RsvdParams(k=100, p=5, s=10, seed=0)
A.pattern(); A.device_values(); rsvd_bki_dev(A, p)
A.pin_memory()
for rep in range(3):
    A.drop_device(); torch.cuda.synchronize()
    t = [time.perf_counter()]
    A.pattern(); torch.cuda.synchronize(); t.append(time.perf_counter())
    A.device_values(); torch.cuda.synchronize(); t.append(time.perf_counter())
    res, Q, _ = rsvd_bki_dev(A, p); torch.cuda.synchronize(); t.append(time.perf_counter())
    U = device.to_host(res.U); t.append(time.perf_counter())
    V = device.to_host(res.V); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"pattern {d[0]:.2f}  values {d[1]:.2f}  compute {d[2]:.2f}  U d2h {d[3]:.2f}  V d2h {d[4]:.2f}  total {sum(d):.2f} ms", flush=True)
