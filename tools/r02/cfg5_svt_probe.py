"""cfg5 scale-up (BASELINE configs[4]: 1e6 x 2e5, 2e8 uniform observations,
rank-100 Gaussian factor product + N(0, 0.01) noise): the SVT loop itself,
svt_fast at the reference defaults (tau = 5n, delta = 1.2 mn / nnz) with
reuse-q recycling, fp64 and the fp32 mode, IMAX iterations each; per
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

imax = int(os.environ.get("IMAX", "6"))
t0 = time.perf_counter()
o = workloads.cfg5()
print(f"generate (host numpy): {time.perf_counter() - t0:.1f} s, nnz {o.rows.size}", flush=True)
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
# ~170 GB; profiles/r02w_cfg5_defaults_oom.txt).  tau is therefore placed from
# the spectrum: one rsvd_bki (k = 300) of P(M), tau = delta * S[TAU_INDEX]
# (c = 1, so ~TAU_INDEX components start above tau).
from paper_1810_06860_b200.rsvd import RsvdParams, rsvd_bki_dev  # noqa: E402

delta = 1.2 * o.m * o.n / A.nnz
t0 = time.perf_counter()
r0, _, _ = rsvd_bki_dev(A, RsvdParams(k=300, p=2, s=5, seed=1))
torch.cuda.synchronize()
tau_index = int(os.environ.get("TAU_INDEX", "150"))
tau = delta * float(r0.S_host[tau_index])
print(f"rsvd_bki k=300 of P(M): {time.perf_counter() - t0:.2f} s; S[0] {r0.S_host[0]:.4e} S[100] {r0.S_host[100]:.4e} "
      f"S[{tau_index}] {r0.S_host[tau_index]:.4e} S[299] {r0.S_host[299]:.4e}; delta {delta:.1f}, tau {tau:.4e}",
      flush=True)
del r0
results = {}
for prec in ("fp64", "fp32"):
    p = completion.SvtParams(tau=tau, epsilon=0.05, i_max=imax, strategy="reuse-q", i_reuse=4, q_reuse=10, seed=0,
                             precision=prec)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = completion.svt_fast(obs, p)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    results[prec] = res
    print(f"== {prec}: {res.iterations} iterations in {dt:.1f} s (loop {sum(t.wall_time for t in res.trace):.1f} s), "
          f"rank {res.rank}, residual {res.residual:.6e}", flush=True)
    for t in res.trace:
        print(f"   i={t.iteration} k={t.k} r={t.r} p={t.p} q={t.q} {t.svd_source} resid={t.residual:.9e} "
              f"{t.wall_time * 1e3:.0f} ms", flush=True)
a, b = results["fp64"].trace, results["fp32"].trace
d = [abs(x.residual - y.residual) / x.residual for x, y in zip(a, b)]
print(f"fp32 vs fp64 residual drift per iteration: max {max(d):.2e}; same (k, r) trajectory: "
      f"{[(x.k, x.r) for x in a] == [(y.k, y.r) for y in b]}", flush=True)
