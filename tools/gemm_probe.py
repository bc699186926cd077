# Run the BKI-shaped dense products once each (for ncu / timing).
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_06860_b200 import device, linalg
rng = np.random.default_rng(0)
H = device.to_device(rng.standard_normal((100000, 660)))
R = device.to_device(np.triu(rng.standard_normal((660, 660))))
V = device.to_device(rng.standard_normal((660, 100)))
for rep in range(2):
    torch.cuda.synchronize()
    res = {}
    for name, fn in (("syrk 100000x660", lambda: linalg.gram_dev(H)),
                     ("nn_upper 100000x660x660", lambda: linalg.matmul_dev(H, R, b_upper=True)),
                     ("nn 100000x660x100", lambda: linalg.matmul_dev(H, V))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1)
    if rep:
        flops = {"syrk 100000x660": 100000*660*661, "nn_upper 100000x660x660": 100000*660*660, "nn 100000x660x100": 2*100000*660*100}
        for k, ms in res.items():
            print(f"{k}: {ms:.3f} ms  {flops[k]/ms/1e9:.2f} TFLOP/s")
