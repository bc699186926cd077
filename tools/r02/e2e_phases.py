"""Phases of the e2e cfg4 job through the public API (svt_fast from host COO
arrays): where the wall clock goes outside the SVT loop."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import bench
from paper_1810_06860_b200 import completion, device, workloads
from paper_1810_06860_b200.sparse import ObservationSet, SparseMatrix

o4 = workloads.cfg4()
params = bench.cfg4_params()
pinned = [device.pinned_copy(a) for a in (o4.rows, o4.cols, o4.values)]
split_p = device.pinned_copy(o4.split)
for rep in range(2):
    T = {}
    t = time.perf_counter(); ob = ObservationSet(o4.m, o4.n, pinned[0], pinned[1], pinned[2], split_p); T["obs"] = time.perf_counter() - t
    t = time.perf_counter(); r, c, v = ob.subset(0); T["subset"] = time.perf_counter() - t
    t = time.perf_counter(); phi_h = SparseMatrix.from_coo(ob.m, ob.n, r, c, v); T["from_coo(host)"] = time.perf_counter() - t
    t = time.perf_counter(); phi = ob.train_matrix(); torch.cuda.synchronize(); T["train_matrix(device)"] = time.perf_counter() - t
    t = time.perf_counter(); phi._host_prep_dev(); T["schedule"] = time.perf_counter() - t
    t = time.perf_counter(); phi.pattern(); torch.cuda.synchronize(); T["pattern upload+transpose"] = time.perf_counter() - t
    t = time.perf_counter(); phi.device_values(); torch.cuda.synchronize(); T["values"] = time.perf_counter() - t
    t = time.perf_counter(); res = completion.svt_fast(ob, params); torch.cuda.synchronize(); T["svt_fast total"] = time.perf_counter() - t
    loop = sum(tr.wall_time for tr in res.trace)
    print(f"rep {rep}: " + ", ".join(f"{k} {v*1e3:.0f} ms" for k, v in T.items()) + f", loop (trace) {loop*1e3:.0f} ms", flush=True)
