# cuBLAS (torch fp64 matmul) on the BKI GEMM shapes, for comparison with lr_gemm_f64 (tools/gemm_probe.py)
import numpy as np, torch
torch.backends.cuda.matmul.allow_tf32 = False
d = torch.device("cuda")
g = torch.Generator(device=d).manual_seed(0)
H = torch.randn(100000, 660, dtype=torch.float64, device=d, generator=g)
Bt = torch.randn(50000, 660, dtype=torch.float64, device=d, generator=g)
R = torch.triu(torch.randn(660, 660, dtype=torch.float64, device=d, generator=g))
V = torch.randn(660, 100, dtype=torch.float64, device=d, generator=g)
cases = (("gram H^T H 100000x660", lambda: H.t() @ H, 2 * 100000 * 660 * 660, 100000 * 660 * 661),
         ("gram 50000x660", lambda: Bt.t() @ Bt, 2 * 50000 * 660 * 660, 50000 * 660 * 661),
         ("H R 100000x660x660 (full)", lambda: H @ R, 2 * 100000 * 660 * 660, 100000 * 660 * 661),
         ("trmm H R (triangular)", lambda: torch.linalg.solve_triangular(R + 660 * torch.eye(660, dtype=torch.float64, device=d), H, upper=True, left=False), 100000 * 660 * 660, 100000 * 660 * 661),
         ("H V 100000x660x100", lambda: H @ V, 2 * 100000 * 660 * 100, 2 * 100000 * 660 * 100))
for name, fn, issued, alg in cases:
    ts = []
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts[2:]))
    print(f"cuBLAS {name:30s} {ms:.3f} ms  {alg / ms / 1e9:.2f} TF/s algorithmic (ours' flop model), {issued / ms / 1e9:.2f} issued", flush=True)
