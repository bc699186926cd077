# tridiagonalization phase clocks + syevd timing at n = 660, full and top-window (one B200)
LR_SYEVD_TIMING=1 timeout 120 python - <<'PY' 2>&1 | tail -8
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg
X = np.random.default_rng(0).standard_normal((2000, 660)); G = device.to_device(X.T @ X)
for il in (0, 0):
    linalg.sym_eig_dev(G); torch.cuda.synchronize()
PY
