import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
for n in (1024, 4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for name, f in (("NN", lambda: a @ b), ("NT", lambda: a @ b.t())):
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        reps = 20 if n <= 4096 else 5
        e0.record()
        for _ in range(reps): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"cuBLAS DGEMM {name} n={n}: {ms:.3f} ms  {2*n**3/ms/1e9:.2f} TFLOP/s", flush=True)
