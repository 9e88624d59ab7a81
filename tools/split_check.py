"""Strict-split check (run with BR_SPLIT_ROWS set): triangular band at a size that
reaches confined panels, depth 1 == depth 0 bitwise and vs the default path."""
import os, sys
import numpy as np
import paper_1709_00302_b200 as br
n, b = 3000, 96
A = np.asfortranarray(np.random.default_rng(5).standard_normal((n, n)))
r1 = br.reduce_tri_band(A, b, b, lookahead=1, return_factors=True)
r0 = br.reduce_tri_band(A, b, b, lookahead=0)
print("depth1 == depth0 bitwise:", np.array_equal(r1.band, r0.band))
sv = np.linalg.svd(A, compute_uv=False); sb = np.linalg.svd(r1.band, compute_uv=False)
print("sv err", np.max(np.abs(sv - sb)) / sv[0])
np.save(sys.argv[1], r1.band)
