# grid barrier cost, LU and tridiagonalization per-column phase clocks (one B200)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gridsync tools/gridsync_bench.cu && /tmp/gridsync
LR_LU_PROFILE=1 python tools/lu_probe.py 2>&1 | tail -3
LR_LU_OCC=1 LR_LU_PROFILE=1 python tools/lu_probe.py occ1 2>&1 | tail -3
LR_SYEVD_TIMING=1 python - <<'PY' 2>&1 | tail -12
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg
X = np.random.default_rng(0).standard_normal((2000, 660)); G = device.to_device(X.T @ X)
for _ in range(2): linalg.sym_eig_dev(G); torch.cuda.synchronize()
PY
