# First iterations of the CPU oracle on cfg4 (for comparison with the GPU trace).
import sys, time, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_1810_06860_b200 import workloads
o = workloads.cfg4()
r, c, v = o.subset(0)
imax = int(sys.argv[1]) if len(sys.argv) > 1 else 3
t = time.time()
out = oracle.complete(o.m, o.n, r, c, v, oracle.SvtConfig(epsilon=0.17, i_reuse=50, q_reuse=10, strategy="reuse-q", seed=0, i_max=imax))
print("oracle", time.time() - t, "s", out.c, out.norm2)
for t in out.trace: print(t)
