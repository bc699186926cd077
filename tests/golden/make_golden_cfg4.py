"""Golden cfg4 job from the REAL reference (build container only; imports
/root/reference/pkg/src): BASELINE configs[3], the rating shape
(workloads.cfg4: 138,493 x 26,744, 20,000,263 ratings, 10 % held out by the
reference's own split_observations), svt_fast with the bench's settings
(bench.CFG4_SVT): reuse-q, i_reuse 50, q_reuse 10 (the rating CLI defaults,
cli.py:277-282), tau = 5n/10, delta = 1.5, eps = 0.40, seed 0.  The
reference's own defaults (tau = 5n, delta = 1.2mn/nnz) blow up on this pattern
(tools/r02/cfg4_reference_defaults.py, profiles/r02_cfg4_defaults.txt).

Writes tests/golden/reference_golden_cfg4.npz: the trace, S, the held-out MAE
and the completed values at 4096 held-out cells.  Takes tens of minutes.

    python tests/golden/make_golden_cfg4.py
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from lowrank.completion import SvtParams, mae, svt_fast  # noqa: E402
from lowrank.sparse import ObservationSet  # noqa: E402

from paper_1810_06860_b200 import workloads  # noqa: E402

CFG = dict(tau_div=10.0, delta=1.5, epsilon=0.40, i_reuse=50, q_reuse=10, strategy="reuse-q", seed=0, i_max=500)


def main():
    o = workloads.cfg4()
    obs = ObservationSet(o.m, o.n, o.rows, o.cols, o.values, o.split)
    c = CFG
    t = time.time()
    res = svt_fast(obs, SvtParams(tau=5.0 * o.n / c["tau_div"], delta=c["delta"], epsilon=c["epsilon"],
                                  i_reuse=c["i_reuse"], q_reuse=c["q_reuse"], strategy=c["strategy"], seed=c["seed"],
                                  i_max=c["i_max"]))
    wall = time.time() - t
    tr, tc, tv = obs.subset(ObservationSet.TEST)
    pred = res.predict(tr, tc)
    rng = np.random.default_rng(7)
    pick = np.sort(rng.choice(tr.shape[0], 4096, replace=False))
    g = {"k": np.array([x.k for x in res.trace]), "r": np.array([x.r for x in res.trace]),
         "p": np.array([x.p for x in res.trace]), "q": np.array([x.q for x in res.trace]),
         "residual": np.array([x.residual for x in res.trace]),
         "source": np.array([x.svd_source for x in res.trace]),
         "wall": np.array([x.wall_time for x in res.trace]), "S": res.S, "converged": np.array(res.converged),
         "heldout_mae": np.array(mae(pred, tv)), "pred_index": pick, "pred": pred[pick],
         "cfg": np.array([c["tau_div"], c["delta"], c["epsilon"], c["i_reuse"], c["q_reuse"], c["seed"]]),
         "total_s": np.array(wall)}
    np.savez_compressed(os.path.join(HERE, "reference_golden_cfg4.npz"), **g)
    print(f"cfg4 reference: {res.iterations} it conv={res.converged} rank={res.rank} resid={res.residual:.6e} "
          f"MAE={float(g['heldout_mae']):.6f} ({wall:.0f}s)", flush=True)


if __name__ == "__main__":
    main()
