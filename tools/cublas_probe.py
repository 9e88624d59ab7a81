"""One cuBLAS DGEMM of each reduction shape (for ncu inspection of its kernels)."""
import sys

import torch

dev = torch.device("cuda", 0)
M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (16384, 16128, 256)
A = torch.randn((K, M), dtype=torch.float64, device=dev)
B = torch.randn((N, K), dtype=torch.float64, device=dev)
C = torch.randn((N, M), dtype=torch.float64, device=dev)
for _ in range(3):
    C.addmm_(B, A)
torch.cuda.synchronize()
print("ok")
