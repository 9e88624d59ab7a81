"""Measure cuBLAS DGEMM throughput (the FP64 roofline denominator) on this GPU."""
import json, sys, torch
torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda:0")
res = {}
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    reps = 5 if n < 16384 else 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[n] = 2 * n ** 3 / (best * 1e-3) / 1e12
    print(f"DGEMM n={n}: {res[n]:.2f} TFLOP/s ({best:.2f} ms)", flush=True)
json.dump(res, open(sys.argv[1] if len(sys.argv) > 1 else "/dev/stdout", "w"))
