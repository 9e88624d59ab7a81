import ctypes as C, numpy as np
from paper_1709_00302_b200 import _lib
import paper_1709_00302_b200 as br
lib = _lib.load()
A = np.asfortranarray(np.random.default_rng(0).standard_normal((600, 600)))
ref = br.reduce_tri_band(A, 64, 64).band
for i in range(6):   # create / use / destroy extra handles: green contexts come and go
    h = C.c_void_p()
    assert lib.br_create(0, C.byref(h)) == 0, lib.br_last_error()
    assert lib.br_destroy(h) == 0
again = br.reduce_tri_band(A, 64, 64).band
print("handles recycled, results equal:", np.array_equal(ref, again))
