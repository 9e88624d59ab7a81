import numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_00302_b200 as br, oracle as O
for (b, j) in [(64, 300), (64, 2000), (40, 500), (256, 5000), (33, 100)]:
    P0 = np.asfortranarray(np.random.default_rng(7).standard_normal((b, j)))
    f = br.lq_panel(P0.copy(order="F")); Y, T, W, L, tau = O.lq_panel(P0.copy(order="F"))
    g = br.qr_panel(np.asfortranarray(P0.T.copy()))
    e = lambda a, r: np.linalg.norm(a - r) / max(1e-300, np.linalg.norm(r))
    print(b, j, "L", e(f.r_or_l, L), "tau", e(f.tau, tau), "Y", e(f.y, Y), "T", e(f.t, T), "qrT-vs-lq L", e(g.r_or_l.T, L))
    if e(f.r_or_l, L) > 1e-12:
        d = np.abs(f.r_or_l - L); i = np.unravel_index(np.argmax(d), d.shape); print("   worst", i, f.r_or_l[i], L[i])
