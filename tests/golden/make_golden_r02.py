"""Round-2 golden fixtures from the REAL reference package.

Run in the build container only (imports /root/reference/pkg/src; the
reference does not travel to the GPU box):

    python tests/golden/make_golden_r02.py [cfg1rq] [cfg2] [ensembles] [split]

Writes tests/golden/reference_golden_r02.npz (merging with what is there):

* cfg1rq_*   BASELINE configs[0] at eps = 1e-3 with svt_fast(reuse-q,
             i_reuse = 50): SURVEY 0.1 item 4's instability (the streak rule
             lowers p during recycling, the forced fresh BKI at p = 1 sends the
             residual up, the run never converges).
* cfg2_*     BASELINE configs[1]: rsvd_pi and rsvd_bki with RsvdParams(k=100,
             p=5, s=10, seed=0) on the seeded 100000 x 50000 / 5M-nnz matrix:
             S, qb_error, and the first 256 rows of U and V (sign-fixed by the
             reference's own convention).
* ens_*      the reference's OWN reproducibility on the recycling traces: the
             same run repeated with every observed value perturbed by at most
             one ulp (6 seeds).  Stored per trace: iteration counts,
             convergence flags, final residuals and the first iteration whose
             residual leaves the unperturbed run by > 1e-13 / 1e-10 / 1e-8 /
             1e-6 relative.  A GPU run cannot be held to a tighter trajectory
             than the reference holds against itself.
* split_*    ingest.split_observations tags (the cfg4 holdout rule).
"""

import os
import sys
import time

for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ[v] = "1"

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from lowrank.completion import SvtParams, svt_fast  # noqa: E402
from lowrank.rsvd import RsvdParams, qb_error, rsvd_bki, rsvd_pi  # noqa: E402
from lowrank.sparse import ObservationSet, SparseMatrix  # noqa: E402

from paper_1810_06860_b200 import workloads  # noqa: E402

OUT = os.path.join(HERE, "reference_golden_r02.npz")
THRESH = (1e-13, 1e-10, 1e-8, 1e-6)


def trace_arrays(res, prefix, out):
    t = res.trace
    out[prefix + "iteration"] = np.array([x.iteration for x in t])
    out[prefix + "k"] = np.array([x.k for x in t])
    out[prefix + "r"] = np.array([x.r for x in t])
    out[prefix + "p"] = np.array([x.p for x in t])
    out[prefix + "q"] = np.array([x.q for x in t])
    out[prefix + "residual"] = np.array([x.residual for x in t])
    out[prefix + "source"] = np.array([x.svd_source for x in t])
    out[prefix + "S"] = res.S
    out[prefix + "converged"] = np.array(res.converged)
    out[prefix + "hard_stops"] = np.array(res.hard_stops)


def cfg1_obs():
    o, _ = workloads.cfg1()
    return ObservationSet(o.m, o.n, o.rows, o.cols, o.values)


def small_obs():
    o, _ = workloads.cfg1_small()
    return ObservationSet(o.m, o.n, o.rows, o.cols, o.values)


def tc_obs():
    g = np.load(os.path.join(HERE, "reference_golden.npz"))
    return ObservationSet(100, 100, g["tc_rows"], g["tc_cols"], g["tc_vals"])


CFG1RQ = dict(epsilon=1e-3, seed=0, strategy="reuse-q", i_reuse=50)
# the recycling traces whose reproducibility is measured: (name, observations, params)
ENSEMBLES = (
    ("tc_rq", tc_obs, dict(epsilon=1e-2, seed=7, strategy="reuse-q", i_reuse=25)),
    ("small_rq", small_obs, dict(epsilon=1e-3, seed=4, strategy="reuse-q", i_reuse=20)),
    ("small_ru", small_obs, dict(epsilon=1e-3, seed=4, strategy="reuse-u", i_reuse=20)),
    ("cfg1rq", cfg1_obs, CFG1RQ),
)


def do_cfg1rq(g):
    t = time.time()
    res = svt_fast(cfg1_obs(), SvtParams(**CFG1RQ))
    trace_arrays(res, "cfg1rq_", g)
    print(f"cfg1rq: {res.iterations} it conv={res.converged} resid={res.residual:.6e} ({time.time() - t:.0f}s)")


def do_cfg2(g):
    o = workloads.cfg2()
    A = SparseMatrix.from_coo(o.m, o.n, o.rows, o.cols, o.values)
    prm = RsvdParams(k=100, p=5, s=10, seed=0)
    for name, fn in (("pi", rsvd_pi), ("bki", rsvd_bki)):
        t = time.time()
        res, _ = fn(A, prm)
        g[f"cfg2_{name}_S"] = res.S
        g[f"cfg2_{name}_qb"] = np.array(qb_error(A, res))
        g[f"cfg2_{name}_U256"] = res.U[:256].copy()
        g[f"cfg2_{name}_V256"] = res.V[:256].copy()
        print(f"cfg2 {name}: S1 {res.S[0]:.9f} S100 {res.S[-1]:.9f} qb {float(g[f'cfg2_{name}_qb']):.9f} "
              f"({time.time() - t:.0f}s)")


def do_ensembles(g):
    for name, make, kw in ENSEMBLES:
        ob = make()
        base = svt_fast(ob, SvtParams(**kw))
        rb = np.array([t.residual for t in base.trace])
        its, conv, fin, first = [], [], [], []
        for s in range(6):
            rng = np.random.default_rng(100 + s)
            v = ob.values * (1.0 + 2.0 ** -52 * rng.choice([-1.0, 0.0, 1.0], ob.values.size))
            r = svt_fast(ObservationSet(ob.m, ob.n, ob.rows, ob.cols, v), SvtParams(**kw))
            rr = np.array([t.residual for t in r.trace])
            n = min(len(rr), len(rb))
            d = np.abs(rr[:n] - rb[:n]) / rb[:n]
            first.append([int(np.argmax(d > th)) + 1 if (d > th).any() else n + 1 for th in THRESH])
            its.append(r.iterations)
            conv.append(r.converged)
            fin.append(r.residual)
        g[f"ens_{name}_base_iterations"] = np.array(base.iterations)
        g[f"ens_{name}_iterations"] = np.array(its)
        g[f"ens_{name}_converged"] = np.array(conv)
        g[f"ens_{name}_final_residual"] = np.array(fin)
        g[f"ens_{name}_first_diff"] = np.array(first)  # 1-based iteration, columns = THRESH
        print(f"ensemble {name}: base {base.iterations} it; perturbed {its}; first diff (1-based) {first}")
    g["ens_thresholds"] = np.array(THRESH)


def do_split(g):
    """ingest.split_observations known answers (the cfg4 holdout rule)."""
    from lowrank.ingest import split_observations
    from lowrank.rng import RngState

    for count, frac, seed in ((1000, 0.9, 0), (777, 0.8, 42)):
        rows = np.arange(count) % 37
        cols = np.arange(count) // 37
        ob = ObservationSet(37, (count + 36) // 37, rows, cols, np.ones(count))
        tagged, cold = split_observations(ob, frac, RngState(seed))
        g[f"split_{count}_{seed}"] = tagged.split.copy()


def main():
    what = set(sys.argv[1:]) or {"cfg1rq", "cfg2", "ensembles", "split"}
    g = dict(np.load(OUT)) if os.path.exists(OUT) else {}
    if "cfg1rq" in what:
        do_cfg1rq(g)
    if "cfg2" in what:
        do_cfg2(g)
    if "ensembles" in what:
        do_ensembles(g)
    if "split" in what:
        do_split(g)
    import lowrank
    import scipy

    g["versions"] = np.array([np.__version__, scipy.__version__, lowrank.__version__])
    np.savez_compressed(OUT, **g)
    print("wrote", len(g), "arrays to", OUT)


if __name__ == "__main__":
    main()
