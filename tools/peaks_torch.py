import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2): a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(5): a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"cuBLAS DGEMM n={n}: {2*n**3/ms/1e9:.2f} TFLOP/s")
# tall gram like cfg2
A = torch.randn(100000, 660, dtype=torch.float64, device="cuda")
for _ in range(2): A.T @ A
torch.cuda.synchronize(); e0.record()
for _ in range(5): A.T @ A
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)/5
print(f"cuBLAS A^T A 100000x660: {ms:.3f} ms, {2*100000*660*660/ms/1e9:.2f} TFLOP/s (full)")
G = A.T @ A
torch.cuda.synchronize(); t=time.time()
w, V = torch.linalg.eigh(G); torch.cuda.synchronize(); print("torch eigh 660 (cusolver):", time.time()-t)
t=time.time(); w, V = torch.linalg.eigh(G); torch.cuda.synchronize(); print("torch eigh 660 (cusolver) 2nd:", time.time()-t)
