"""Time the PURE reference (baseline/_ref, unmodified: its matmul is the
sequential rank-1 loop of ref kernels.py:39-83) on whole c1 / c2 reductions
on this host, beside the tier-B BLAS-rebound reference on the same input
(VERDICT r1 item 6). Run on the GPU box:

    python tools/cpu_pure.py [c1 c2] > gpurun_out/cpu_pure.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from baseline import ref_driver as R  # noqa: E402
import oracle as O  # noqa: E402
from bench import CONFIGS, nominal  # noqa: E402


def main():
    names = sys.argv[1:] or ["c1", "c2"]
    for name in names:
        kind, n, w, b, desc = CONFIGS[name]
        A = O.gen_config(name)
        out = {"workload": name, "desc": desc, "cores": os.cpu_count()}
        for mode in ("pure", "blas"):
            bandred = R.load(mode)
            iters = 1 << 30
            flops, sec, done = R.sample(bandred, kind, A.copy(order="F"), n, w, b, iters)
            out[mode] = {"seconds": sec, "tasks": done, "counted_gflop": flops / 1e9,
                         "gflops_nominal": nominal(kind, n) / sec / 1e9}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
