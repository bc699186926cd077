"""cfg5 scale-up (BASELINE configs[4]: 1e6 x 2e5, 2e8 uniform observations,
rank-100 Gaussian factor product + N(0, 0.01) noise): the SVT loop itself,
svt_fast at the reference's delta = 1.2 mn / nnz and a tau that lets the
rank grow through ~300 (below), reuse-q recycling, fp64 and the fp32 mode; per
iteration k, r, p, source, residual and wall time, the fp32 mode's residual
drift against fp64, and a spot check of the CSR product on sampled rows
against scipy (the reference's own SpMM) on the host."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import scipy.sparse as sps  # noqa: E402
import torch  # noqa: E402

from paper_1810_06860_b200 import completion, device, workloads  # noqa: E402
from paper_1810_06860_b200.sparse import ObservationSet, spmm_dev  # noqa: E402

imax = int(os.environ.get("IMAX", "45"))
t0 = time.perf_counter()
if os.environ.get("CFG5_GEN", "device") == "device":
    o = workloads.cfg5_device()
    print(f"generate (device, workloads.cfg5_device): {time.perf_counter() - t0:.1f} s, nnz {o.rows.size}", flush=True)
else:
    o = workloads.cfg5()
    print(f"generate (host numpy): {time.perf_counter() - t0:.1f} s, nnz {o.rows.size}", flush=True)
torch.cuda.empty_cache()
t0 = time.perf_counter()
obs = ObservationSet(o.m, o.n, o.rows, o.cols, o.values)
torch.cuda.synchronize()
print(f"ObservationSet (device duplicate search + CSR build): {time.perf_counter() - t0:.2f} s", flush=True)
A = obs.train_matrix()
# spot check: rows of Y X against scipy on the host
rng = np.random.default_rng(0)
X = rng.standard_normal((o.n, 40))
Yx = device.to_host(spmm_dev(A, device.to_device(X)))
rows = rng.choice(o.m, 2000, replace=False)
sub = sps.csr_matrix((o.values, (o.rows, o.cols)), shape=(o.m, o.n))[rows]
ref = sub @ X
err = np.linalg.norm(Yx[rows] - ref) / np.linalg.norm(ref)
print(f"SpMM spot check (2000 rows, w = 40) vs scipy: rel err {err:.2e}", flush=True)
del sub, Yx
# At the reference defaults (tau = 5n, delta = 1.2 mn / nnz = 1200) the first
# iteration's rank escalation ran past k = 1100 (W ~ 4600, out of memory at
# ~170 GB; profiles/r02w_cfg5_defaults_oom.txt): cfg5 sits at the detection
# threshold -- the signal's singular values in P(M) are p sigma(M) ~ 1e-3 x
# 4.5e5 ~ 450, the sampling-noise bulk edge is sqrt(p var(M)) (sqrt m + sqrt n)
# ~ 0.32 x 1447 ~ 457 -- and 2e8 samples are 1.67x the rank-100 degrees of
# freedom, below what any completion method recovers from.  With delta = 1200
# and a large tau (5e7) the loop overshoots: residuals 8, 13, 19 with the rank
# reset to 0 after each (profiles/r02cc_cfg5_delta1200.txt).  The scale-up run
# therefore uses delta = DELTA (default 1, inside SVT's delta < 2 condition)
# and tau = TAU_C * delta * S[0] (c ~ TAU_C): Y accumulates P(M - X) and the
# rank grows through the flat spectrum (S[0] / S[299] = 1.27) toward ~300 in
# ~TAU_C / 4 iterations.  KCAP stops the run (the trace so far is printed)
# before the escalation outgrows memory.
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki_dev  # noqa: E402

delta = float(os.environ.get("DELTA", "1.0"))
t0 = time.perf_counter()
r0, _, _ = rsvd_bki_dev(A, RsvdParams(k=300, p=2, s=5, seed=1))
torch.cuda.synchronize()
tau = float(os.environ.get("TAU_C", "100")) * delta * float(r0.S_host[0])
kcap = int(os.environ.get("KCAP", "420"))
print(f"rsvd_bki k=300 of P(M): {time.perf_counter() - t0:.2f} s; S[0] {r0.S_host[0]:.4e} S[100] {r0.S_host[100]:.4e} "
      f"S[299] {r0.S_host[299]:.4e}; delta {delta:.1f}, tau {tau:.4e}, c = {int(np.ceil(tau / (delta * r0.S_host[0])))}",
      flush=True)
del r0


class KCap(Exception):
    pass


_bki = completion.DeviceEngine.bki


def _capped(self, rp, *a, **kw):
    if rp.k > kcap:
        raise KCap(f"rank escalation reached k = {rp.k} > KCAP = {kcap}")
    return _bki(self, rp, *a, **kw)


completion.DeviceEngine.bki = _capped
completion.VERBOSE = True
results = {}
for prec in ("fp64", "fp32"):
    p = completion.SvtParams(tau=tau, delta=delta, epsilon=0.05, i_max=imax, strategy="reuse-q", i_reuse=4, q_reuse=10, seed=0,
                             precision=prec)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    print(f"== {prec}", flush=True)
    try:
        res = completion.svt_fast(obs, p)
        torch.cuda.synchronize()
        results[prec] = res
        print(f"== {prec}: {res.iterations} iterations in {time.perf_counter() - t0:.1f} s, rank {res.rank}, "
              f"residual {res.residual:.6e}", flush=True)
    except KCap as exc:
        torch.cuda.synchronize()
        print(f"== {prec}: stopped after {time.perf_counter() - t0:.1f} s: {exc}", flush=True)
    torch.cuda.empty_cache()
    print(f"   peak device memory {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB", flush=True)
    torch.cuda.reset_peak_memory_stats()
