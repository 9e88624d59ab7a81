"""CPU oracle for the dense->band reduction hot path (TEST INFRASTRUCTURE ONLY).

This package restates, in NumPy, the reference `bandred` algorithms that the
B200 path replaces. It exists to check the CUDA path: only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference`) may import it. The product package
`paper_1709_00302_b200` never imports it and has no CPU fallback.

Parity pinning: `tests/golden/*.npz` were produced by running the reference
package itself (`tests/golden/make_golden.py`); `tests/test_oracle_golden.py`
checks this restatement against them.
"""
from .bandred_oracle import *  # noqa: F401,F403
from .bandred_oracle import __all__  # noqa: F401
