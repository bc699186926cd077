"""cfg4 SVT job (bench.py's settings) with a host + device timeline of every
native call: GPU busy time vs job time, the largest GPU-idle gaps and the
native call that ended each gap, and a cProfile of the host side.
Usage: python tools/r02/cfg4_timeline.py [job|cprofile]"""
import cProfile
import os
import pstats
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1810_06860_b200 import _native, completion, profiling, workloads  # noqa: E402
from paper_1810_06860_b200.sparse import ObservationSet  # noqa: E402


class TL(profiling.Profiler):
    def run(self, name, meta, fn, args):
        h0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        st = fn(*args)
        e1.record()
        self.records.append((name, meta, e0, e1, h0, time.perf_counter()))
        return st


from paper_1810_06860_b200 import rng as _rng  # noqa: E402

_TN = []
_take = _rng.take_normals


def _timed_take(seed, rows, cols):
    hit = (int(seed), int(rows), int(cols)) in _rng._PREFETCH
    t0 = time.perf_counter()
    out = _take(seed, rows, cols)
    _TN.append((time.perf_counter() - t0, hit))
    return out


_rng.take_normals = _timed_take

o4 = workloads.cfg4()
obs = ObservationSet(o4.m, o4.n, o4.rows, o4.cols, o4.values, o4.split)
params = bench.cfg4_params()
if os.environ.get("SHARD"):  # the sharded engine on one rank, collectives forced (NCCL)
    import torch.distributed as dist

    from paper_1810_06860_b200.shards import Exchange, ShardedEngine

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    eng = ShardedEngine(obs, Exchange(always_collective=True))
else:
    eng = completion.DeviceEngine(obs)


def job():
    return completion._svt_loop(obs, params, "rsvd-bki", params.strategy, engine=eng)


for _ in range(2):
    job()
torch.cuda.synchronize()
mode = sys.argv[1] if len(sys.argv) > 1 else "job"
if mode == "cprofile":
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    res = job()
    torch.cuda.synchronize()
    pr.disable()
    print(f"{res.iterations} iterations in {time.perf_counter() - t0:.3f} s")
    pstats.Stats(pr).sort_stats("tottime").print_stats(30)
    pstats.Stats(pr).sort_stats("cumtime").print_stats(40)
    sys.exit(0)

_TN.clear()
t0 = time.perf_counter()
_rng.normals_column_major(12345, o4.n, 55)
print(f"one cfg4-sized host draw (26744 x 55): {1e3 * (time.perf_counter() - t0):.2f} ms")
tl = TL()
_native.PROFILER = tl
base = torch.cuda.Event(enable_timing=True)
base.record()
h_base = time.perf_counter()
res = job()
endev = torch.cuda.Event(enable_timing=True)
endev.record()
torch.cuda.synchronize()
h_end = time.perf_counter()
_native.PROFILER = None
total = base.elapsed_time(endev)
busy = 0.0
gaps = []
prev_end = 0.0
per = defaultdict(float)
for name, meta, e0, e1, h0, h1 in tl.records:
    g0, g1 = base.elapsed_time(e0), base.elapsed_time(e1)
    busy += g1 - g0
    per[name] += g1 - g0
    if g0 - prev_end > 0.02:
        gaps.append((g0 - prev_end, name, prev_end, 1e3 * (h0 - h_base)))
    prev_end = max(prev_end, g1)
print(f"{res.iterations} iterations: device span {total:.1f} ms, native busy {busy:.1f} ms "
      f"({busy / total:.2%}), host wall {1e3 * (h_end - h_base):.1f} ms, {len(tl.records)} native calls")
gsum = defaultdict(lambda: [0, 0.0])
for g, name, *_ in gaps:
    gsum[name][0] += 1
    gsum[name][1] += g
print("idle gaps > 20 us, by the native call that ended them (count, total ms):")
for name, (c, t) in sorted(gsum.items(), key=lambda kv: -kv[1][1]):
    print(f"  {name:28s} {c:5d} {t:9.2f}")
print("busy by call (ms):")
for name, t in sorted(per.items(), key=lambda kv: -kv[1]):
    print(f"  {name:28s} {t:9.2f}")
print(f"take_normals: {len(_TN)} calls, {sum(1 for t in _TN if t[1])} prefetched, waited "
      f"{1e3 * sum(t[0] for t in _TN):.1f} ms total, {1e3 * sum(t[0] for t in _TN if not t[1]):.1f} ms on misses")
from paper_1810_06860_b200 import rsvd as _rsvd  # noqa: E402

print(f"Omega sources over all jobs of this process: {_rsvd.OMEGA_STATS}")
_k = np.array(_rsvd.REUSE_STATS["kappas"])
print(f"Krylov reuse: used {_rsvd.REUSE_STATS['used']}, kappa-gated {_rsvd.REUSE_STATS['kappa_gate']}; kappa_F(H) "
      f"quantiles 10/50/90/max: {np.quantile(_k, [0.1, 0.5, 0.9, 1.0]) if _k.size else None}")
print("trace (i, source, k, r, p):", [(t.iteration, t.svd_source[0], t.k, t.r, t.p) for t in res.trace])
print("largest 15 gaps (ms, next call, gpu t, host t):")
for g in sorted(gaps, reverse=True)[:15]:
    print(f"  {g[0]:7.3f} {g[1]:28s} gpu {g[2]:9.2f} host {g[3]:9.2f}")

# LR_TL_DUMP=a:b -- every native call whose host start lies in [a, b) ms: host start / end, GPU start /
# end, and the GPU gap before it (where does the host spend the time the GPU idles?)
if os.environ.get("LR_TL_DUMP"):
    a, b = (float(x) for x in os.environ["LR_TL_DUMP"].split(":"))
    prev_end = 0.0
    prev_h1 = 0.0
    for name, meta, e0, e1, h0, h1 in tl.records:
        g0, g1 = base.elapsed_time(e0), base.elapsed_time(e1)
        hs, he = 1e3 * (h0 - h_base), 1e3 * (h1 - h_base)
        if a <= hs < b:
            print(f"{name:26s} host {hs:8.3f}..{he:8.3f} (since prev call {hs - prev_h1:6.3f})  gpu {g0:8.3f}..{g1:8.3f} "
                  f"gap {max(0.0, g0 - prev_end):6.3f}  lead {g0 - hs:7.3f}")
        prev_end = max(prev_end, g1)
        prev_h1 = he
