"""qr_panel against the oracle on shapes that reach every pair-step leaf
(development tool; run under gpurun with PYTHONPATH=.)."""
import sys
import numpy as np
import oracle as O
import paper_1709_00302_b200 as br


def rel(a, b, s):
    return np.linalg.norm(a - b) / s


def check(name, P0):
    Pg, Po = P0.copy(order="F"), P0.copy(order="F")
    f = br.qr_panel(Pg)
    Y, T, W, R, tau = O.qr_panel(Po)
    e = (rel(f.r_or_l, R, np.linalg.norm(P0)), rel(f.y, Y, np.linalg.norm(Y)), rel(f.t, T, np.linalg.norm(T)),
         rel(f.w, W, np.linalg.norm(W)), rel(f.tau, tau, np.linalg.norm(tau)))
    sg = np.array_equal(np.sign(np.diag(f.r_or_l)), np.sign(np.diag(R)))
    ok = sg and max(e) <= 1e-12
    print(f"{name:28s} R {e[0]:.1e} Y {e[1]:.1e} T {e[2]:.1e} W {e[3]:.1e} tau {e[4]:.1e} signs {sg} {'ok' if ok else 'FAIL'}",
          flush=True)
    return ok


rng = np.random.default_rng(7)
ok = True
for j, b in [(300, 32), (700, 31), (2016, 32), (2016, 17), (1000, 16), (1000, 9), (4000, 32), (4000, 24),
             (8000, 32), (8000, 16), (5000, 12), (16000, 16), (300, 2), (2016, 3), (3000, 128), (9000, 256)]:
    ok &= check(f"randn {j}x{b}", rng.standard_normal((j, b)))
# structured panels: zero column, zero tail, already triangular, nearly dependent neighbours
for j, b in [(2016, 32), (5000, 32)]:
    P = rng.standard_normal((j, b)); P[:, 5] = 0.0; P[:, 6] = 0.0
    ok &= check(f"zero cols {j}x{b}", P)
    P = rng.standard_normal((j, b)); P[8:, 7] = 0.0; P[9:, 8] = 0.0
    ok &= check(f"zero tails {j}x{b}", P)
    ok &= check(f"triangular {j}x{b}", np.triu(rng.standard_normal((j, b))))
    P = rng.standard_normal((j, b))
    for c in range(1, b, 2):
        P[:, c] = P[:, c - 1] + 1e-3 * rng.standard_normal(j)   # pairs that cancel: fallback steps
    ok &= check(f"near-dependent {j}x{b}", P)
    P = rng.standard_normal((j, b)) * np.logspace(0, -10, b)[None, :]
    ok &= check(f"graded cols {j}x{b}", P)
    P = rng.standard_normal((j, b)); P[:, 3] = P[:, 2]
    ok &= check(f"duplicate col {j}x{b}", P)
print("ALL OK" if ok else "FAILURES")
sys.exit(0 if ok else 1)
