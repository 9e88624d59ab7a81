"""Probe: which GPU eigensolver / SVD path handles n = 16384 / 32768 fp64 (test checker)."""
import time
import torch

def t(name, f):
    torch.cuda.synchronize(); t0 = time.time()
    try:
        r = f(); torch.cuda.synchronize(); print(f"{name}: ok {time.time()-t0:.1f}s", flush=True); return r
    except Exception as e:
        print(f"{name}: FAIL {time.time()-t0:.1f}s {str(e)[:200]}", flush=True)

n = 16384
A = torch.rand(n, n, dtype=torch.float64, device="cuda") * 2 - 1
t("svdvals 16384 default", lambda: torch.linalg.svdvals(A))
S = (A + A.T) / 2
t("eigvalsh 16384 cusolver", lambda: torch.linalg.eigvalsh(S))
torch.backends.cuda.preferred_linalg_library("magma")
t("eigvalsh 16384 magma", lambda: torch.linalg.eigvalsh(S))
del S, A
torch.cuda.empty_cache()
n = 32768
G = torch.randn(n, n, dtype=torch.float64, device="cuda")
G = (G + G.T) / 2
t("eigvalsh 32768 magma", lambda: torch.linalg.eigvalsh(G))
torch.backends.cuda.preferred_linalg_library("cusolver")
t("eigvalsh 32768 cusolver", lambda: torch.linalg.eigvalsh(G))
t("eigvalsh 32767 cusolver", lambda: torch.linalg.eigvalsh(G[:32767, :32767]))
