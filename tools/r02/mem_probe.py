"""Device memory across the cfg4 SVT job: torch.cuda.memory_allocated after
every iteration (a leak shows as steady growth)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
from paper_1810_06860_b200 import completion, workloads
from paper_1810_06860_b200.sparse import ObservationSet

o4 = workloads.cfg4()
obs = ObservationSet(o4.m, o4.n, o4.rows, o4.cols, o4.values, o4.split)
params = bench.cfg4_params()
eng = completion.DeviceEngine(obs)
orig = completion._inner_svd
mem = []


def spy(state, *a, **k):
    out = orig(state, *a, **k)
    torch.cuda.synchronize()
    mem.append((state.iteration, torch.cuda.memory_allocated() / 2**30))
    return out


completion._inner_svd = spy
for rep in range(2):
    mem.clear()
    completion._svt_loop(obs, params, "rsvd-bki", params.strategy, engine=eng)
    torch.cuda.synchronize()
    print(f"job {rep}: allocated GiB after inner SVDs (iteration, GiB):", [(i, round(g, 2)) for i, g in mem[::6]],
          "end", round(torch.cuda.memory_allocated() / 2**30, 2), "max", round(torch.cuda.max_memory_allocated() / 2**30, 2),
          flush=True)
