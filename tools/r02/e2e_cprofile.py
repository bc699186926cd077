"""cProfile of one e2e cfg4 job (ObservationSet from pinned host COO + svt_fast), cumulative view."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
from paper_1810_06860_b200 import completion, device, workloads
from paper_1810_06860_b200.sparse import ObservationSet

o4 = workloads.cfg4()
params = bench.cfg4_params()
pinned = [device.pinned_copy(a) for a in (o4.rows, o4.cols, o4.values)]
split_p = device.pinned_copy(o4.split)


def job():
    ob = ObservationSet(o4.m, o4.n, pinned[0], pinned[1], pinned[2], split_p)
    r = completion.svt_fast(ob, params)
    torch.cuda.synchronize()
    return r


for _ in range(2):
    job()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = job()
pr.disable()
print(f"{res.iterations} iterations, {time.perf_counter() - t0:.3f} s e2e, loop {sum(t.wall_time for t in res.trace):.3f} s")
pstats.Stats(pr).sort_stats("cumtime").print_stats(45)
