"""Diagnose test_zero_column_flops_match_native: native vs devices=[0] vs oracle."""
import numpy as np
import oracle as O
import paper_1709_00302_b200 as br

n, b = 256, 32
A = np.diag(np.arange(1.0, n + 1))
A[40:, 3] = A[3, 40:] = 0.5
ev = np.linalg.eigvalsh(A)
for la in (0, 1):
    cfg = br.SevpConfig(n, b, b, br.SevpVariant.V2 if la else br.SevpVariant.REFERENCE)
    ref, _, it = O.reduce_sym_band(A, n, b, b)
    nat = br.reduce_sym_band(A, cfg).band
    mul = br.reduce_sym_band(A, cfg, devices=[0], lookahead=la).band
    na = np.linalg.norm(A)
    print("la", la, "native-oracle", np.linalg.norm(nat - ref) / na, "multi-oracle", np.linalg.norm(mul - ref) / na)
    for name, B in (("oracle", ref), ("native", nat), ("multi", mul)):
        print("  ", name, "eig err", np.max(np.abs(np.linalg.eigvalsh(B) - ev)) / np.max(np.abs(ev)))
    d = np.abs(mul - ref)
    idx = np.argwhere(d > 1e-9)
    print("  first differing entries (multi vs oracle):", idx[:5].tolist())
    d = np.abs(nat - ref)
    idx = np.argwhere(d > 1e-9)
    print("  first differing entries (native vs oracle):", idx[:5].tolist())
