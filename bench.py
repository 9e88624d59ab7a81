"""Benchmark: fp64 GFLOP/s of the first-stage dense->band reduction on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One "step" = one full reduction of the configuration's matrix, starting from
a fresh device copy of the input (the D2D restore is inside the timed step,
like the reference's own copy of A). Workload defaults to BASELINE.json
config 4 (SVD dense -> upper triangular-band, m=n=16384, w=b=256, look-ahead
depth 1): the north-star configuration, and it fits one GPU. The metric
uses the reference's nominal counts (4/3 n^3 SEVP, 8/3 n^3 square SVD;
ref sevp.py:92-96, svd.py:127-132).

Under torchrun (N > 1) the ranks reduce ONE matrix together: 1D
block-cyclic columns with NCCL panel broadcast, X1 / Z all-reduce and LQ
row-panel all-gather (paper_1709_00302_b200/dist.py); timing
is the max over ranks, `value` the whole-job GFLOP/s ("scaling": "strong").

--impl reference times the reference algorithm's CPU implementation on the
host cores: the NumPy port in oracle/ (the reference is pure Python and does
not travel to the GPU box), on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "fp64 GFLOP/s of dense→band reduction (4/3·n³ SEVP, 8/3·n³ SVD) at 1–8 B200"

CONFIGS = {
    # name: (kind, n, w, b, description)
    "c1": ("sevp", 2048, 32, 32, "SEVP n=2048 w=b=32, A=(G+G^T)/2 N(0,1) seed 0"),
    "c2": ("tri", 2048, 32, 32, "SVD triband m=n=2048 w=b=32, N(0,1) seed 1"),
    "c3": ("sevp", 8192, 128, 128, "SEVP n=8192 w=b=128, graded spectrum 1e-8, seeds 2/3"),
    "c4": ("tri", 16384, 256, 256, "SVD triband m=n=16384 w=b=256, U(-1,1) seed 4"),
    "c5": ("sevp", 32768, 256, 256, "SEVP n=32768 w=b=256, A=(G+G^T)/2 N(0,1) seed 5"),
    # not a BASELINE config: the equal-bandwidth band form on c4's matrix
    "b4": ("band", 16384, 256, 256, "SVD band form m=n=16384 w=b=256 (Simultaneous/V2), c4 input"),
}


def nominal(kind, n):
    return 4.0 * n**3 / 3.0 if kind == "sevp" else 4.0 * (n * n * n - n**3 / 3.0)


# --------------------------------------------------------------------------
# clocks sampled during the timed region
# --------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        smax = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------
# inputs
# --------------------------------------------------------------------------
def make_input(cfg):
    import oracle as O  # input generators only (same seeds/distributions as the survey)

    return O.gen_config({"b4": "c4"}.get(cfg, cfg))


def _blas_threads():
    try:
        import threadpoolctl

        return max((i.get("num_threads", 1) for i in threadpoolctl.threadpool_info()
                    if i.get("user_api") == "blas"), default=os.cpu_count())
    except Exception:
        return os.cpu_count()


def cpu_sample(cfg, A, seconds_hint=20.0, tasks=None):
    """Time the reference's CPU implementation on the first panel tasks of the
    same workload (a bounded sample). Prefers the reference package itself
    (baseline/_ref, installed offline; its matmul rebound to multithreaded
    BLAS = SURVEY tier B, see baseline/ref_driver.py), else the oracle port.
    Returns a dict: value (GFLOP/s over the sampled tasks' counted flops),
    kind, tasks, seconds, cores, sample text."""
    from baseline import ref_driver as R

    kind, n, w, b, _ = CONFIGS[cfg]
    full = 2 * len(__import__("oracle").tri_schedule(n, n, b)) if kind == "tri" else \
        len(__import__("oracle").sevp_schedule(n, w, b))
    if R.available():
        mod = R.load("blas")

        def run(k):
            fl, dt, done = R.sample(mod, kind, A, n, w, b, k)
            return fl, dt, done

        label = ("reference package (baseline/_ref) with its matmul rebound to multithreaded "
                 "BLAS (SURVEY tier B)")
        kind_out = "reference"
    else:
        import oracle as O
        from paper_1709_00302_b200.flops import sevp_counted_flops, tri_counted_flops

        def run(k):
            t0 = time.perf_counter()
            if kind == "sevp":
                O.reduce_sym_band(A, n, w, b, max_iters=k, finalize=False)
                fl = sevp_counted_flops(n, w, b, "reference", max_iters=k)[0]["total"]
            else:
                it = (k + 1) // 2
                O.reduce_tri_band(A, w, b, max_iters=it, finalize=False)
                fl = tri_counted_flops(n, n, w, b, max_iters=it)[0]["total"]
                k = 2 * it
            return fl, time.perf_counter() - t0, k

        label = "oracle/ NumPy port + multithreaded OpenBLAS (reference package not installed)"
        kind_out = "port"
    if tasks is None:
        fl, dt, done = run(1)
        tasks = max(1, min(full, int(seconds_hint / max(dt, 1e-3))))
        if tasks > 1:
            fl, dt, done = run(tasks)
    else:
        fl, dt, done = run(tasks)
    unit = "iterations" if kind == "sevp" else "panel tasks (QR or LQ panel + its one-sided update)"
    return {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": _blas_threads(), "kind": kind_out,
            "tasks": done, "seconds": dt,
            "sample": f"first {done} of {full} {unit} of the same {n}x{n} reduction on the same "
                      f"input, {dt:.1f} s, rate = counted flops of the sample / its time; {label}"}


def same_config(cfg, la, world):
    kind, n, w, b, desc = CONFIGS[cfg]
    return {"workload": cfg, "desc": desc, "kind": kind, "n": n, "w": w, "b": b, "lookahead": la,
            "parallelism": "1 GPU" if world == 1 else f"1D block-cyclic columns x{world} (NCCL)",
            "l2": f"input {n * n * 8 / 2**30:.2f} GiB vs 126 MB L2 (no flush needed)"
            if n * n * 8 > 126e6 else "input fits L2; restored from a separate copy each step"}


def dgemm_peak(dev):
    """Measured cuBLAS DGEMM throughput (TFLOP/s): the FP64 roofline denominator
    (MEASURED_PEAKS.json carries no fp64 figure)."""
    import torch

    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(4):
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * n**3 / (best * 1e-3) / 1e12


def load_traffic(cfg):
    p = os.path.join(ROOT, "profiles", f"traffic_{cfg}.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


# --------------------------------------------------------------------------
# arms
# --------------------------------------------------------------------------
def run_reference(args, rank, world):
    """The reference's CPU implementation on the host cores (rank 0 only),
    each step one bounded sample (the first panel tasks) of the workload."""
    kind, n, w, b, desc = CONFIGS[args.config]
    if rank != 0:
        return
    A = make_input(args.config)
    first = cpu_sample(args.config, A, min(args.cpu_seconds, 8.0))  # sizing run (= warm-up)
    vals, secs = [], []
    for _ in range(args.steps):
        r = cpu_sample(args.config, A, tasks=first["tasks"])
        vals.append(r["value"])
        secs.append(r["seconds"])
    v = float(np.median(vals))
    cb = dict(r, value=v, seconds=float(np.median(secs)))
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": "GFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": float(np.median(secs)) * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": same_config(args.config, args.lookahead, world),
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "each step = the reference's first panel tasks on the full input (CPU has no "
                "warm-up state: one sizing sample replaces the warm-up steps); ms_per_step is "
                "one sample, not a whole reduction",
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_1709_00302_b200 import _lib

    kind, n, w, b, desc = CONFIGS[args.config]
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()
    h = _lib.handle(local_rank)
    peak = dgemm_peak(dev)

    A_host = make_input(args.config)  # F-order numpy
    ld = (n + 31) // 32 * 32
    A0 = torch.empty((n, ld), dtype=torch.float64, device=dev)
    A0[:, :n].copy_(torch.from_numpy(A_host.T))  # column-major on the device
    A = torch.empty_like(A0)
    # a real (non-NULL) stream shared by torch (input restore) and the library
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize(dev)
    torch.cuda.set_stream(stream)
    la = args.lookahead

    def one_step(st):
        A.copy_(A0)
        if kind == "sevp":
            rc = lib.br_reduce_sym_band(h, n, w, b, la, A.data_ptr(), ld, None, 0, None, st)
        elif kind == "band":
            rc = lib.br_reduce_band(h, n, n, w, b, 1, la, A.data_ptr(), ld, None, st)
        else:
            rc = lib.br_reduce_tri_band(h, n, n, w, b, la, A.data_ptr(), ld, None, st)
        _lib.check(rc, "reduce")

    # the library runs on its own streams: make it follow torch's stream
    lib.br_set_streams(h, C.c_void_p(stream.cuda_stream), None)
    st = _lib.BrStats()
    for _ in range(args.warmup):
        one_step(st)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    launches = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(args.steps):
        one_step(st)  # replays the CUDA graph captured during warm-up
        launches += st.launches + 1  # + the D2D restore
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    # per-kernel-class breakdown (roofline): a second timed pass with CUDA
    # events around every task on its launch stream (events cannot be timed
    # inside a graph replay, so this pass runs the same stream program eagerly)
    bsteps = max(1, args.breakdown_steps)
    lib.br_set_timing(h, 1)
    eb0, eb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eb0.record(stream)
    for _ in range(bsteps):
        one_step(st)
    eb1.record(stream)
    torch.cuda.synchronize(dev)
    ms_eager = eb0.elapsed_time(eb1) / bsteps
    timing = {}
    names = ["panel", "symm", "syr2k", "gemm"]
    for c in range(4):
        tms, tfl, tnl = C.c_double(), C.c_double(), C.c_int64()
        lib.br_get_timing(h, c, C.byref(tms), C.byref(tfl), C.byref(tnl))
        timing[names[c]] = (tms.value / bsteps, tfl.value / bsteps, tnl.value // bsteps)
    lib.br_set_timing(h, 0)
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops = nominal(kind, n)
    value = world * flops / (ms * 1e-3) / 1e9

    # ---- e2e through the C-ABI host entry point (pinned host buffers) ----
    Ah = torch.from_numpy(np.asfortranarray(A_host).T.copy()).pin_memory()  # (n, n) = col-major
    Bh = torch.empty((n, n), dtype=torch.float64).pin_memory()
    lib.br_set_streams(h, None, None)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))

    def host_call():
        if kind == "sevp":
            rc = lib.br_reduce_sym_band_host(h, n, w, b, la, Ah.data_ptr(), n, Bh.data_ptr(), n,
                                             None, 0, None, st)
        elif kind == "band":
            rc = lib.br_reduce_band_host(h, n, n, w, b, 1, la, Ah.data_ptr(), n, Bh.data_ptr(), n, None, st)
        else:
            rc = lib.br_reduce_tri_band_host(h, n, n, w, b, la, Ah.data_ptr(), n, Bh.data_ptr(), n, None, st)
        _lib.check(rc, "reduce_host")

    for _ in range(2):  # eager call sizes the staging buffers, the second captures the graph
        host_call()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        host_call()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if dist:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = world * flops / e2e_s / 1e9

    # ---- roofline of the dominant kernel class ----
    dom = max(timing, key=lambda k: timing[k][0])
    dms, dfl, dnl = timing[dom]
    achieved = dfl / (dms * 1e-3) / 1e12 if dms > 0 else 0.0
    if dom == "panel":  # report the dominant GEMM class instead: panels are latency-bound
        gem = max(("symm", "syr2k", "gemm"), key=lambda k: timing[k][0])
        dom_note = f"panel dominates ({dms:.1f} ms); roofline for {gem}"
        dms, dfl, dnl = timing[gem]
        dom = gem
        achieved = dfl / (dms * 1e-3) / 1e12 if dms > 0 else 0.0
    else:
        dom_note = None
    traffic = load_traffic(args.config)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and kind != "band":
        cpu = cpu_sample(args.config, A_host, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "GFLOP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic",
            "config": same_config(args.config, la, world),
            "clocks": clocks.summary(),
            "e2e": {"value": e2e_val, "unit": "GFLOP/s",
                    # SEVP: the host entry point copies the lower triangle only
                    "h2d_bytes_per_step": int(lib.br_sym_stage_bytes(n)) if kind == "sevp" else n * n * 8,
                    "d2h_bytes_per_step": n * n * 8, "steps": e2e_steps,
                    "path": "br_reduce_*_host (C ABI), pinned host in/out"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                         "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (MEASURED_PEAKS.json has no fp64)",
                         "traffic": traffic.get(dom) if traffic else None,
                         "note": dom_note,
                         "measured": "class flops / class CUDA-event time in the breakdown pass"},
            "breakdown_ms": {k: round(v[0], 3) for k, v in timing.items()},
            "breakdown_pass": {"steps": bsteps, "ms_per_step": ms_eager,
                               "how": "same stream program run eagerly with per-task CUDA events "
                                      "(the timed region replays it as a CUDA graph)"},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_dist(args, rank, world, local_rank):
    """N > 1: one matrix, 1D block-cyclic columns over the ranks,
    NCCL broadcast / all-reduce / all-gather inside paper_1709_00302_b200.dist."""
    import torch
    import torch.distributed as dist

    from paper_1709_00302_b200 import _lib
    from paper_1709_00302_b200 import dist as D

    kind, n, w, b, desc = CONFIGS[args.config]
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize(dev)
    torch.cuda.set_stream(stream)
    lib = _lib.load()
    peak = dgemm_peak(dev)
    lay = D.Layout(n, b, world, rank)
    ops = D.CudaOps(local_rank, torch)
    comm = D.TorchComm(dist, stream=torch.cuda.Stream(device=dev, priority=-1))
    A_host = make_input(args.config)
    L0 = D.scatter_columns(A_host, lay, ops, kind)
    L = ops.alloc(n, lay.ncols_local)
    la = args.lookahead
    fn = D.reduce_sym_band_dist if kind == "sevp" else D.reduce_tri_band_dist

    def one_step():
        L.t.copy_(L0.t)
        fn(L, lay, w, ops, comm, la)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize(dev)
    dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    l0 = lib.br_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        one_step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks.stop()
    launches = (lib.br_launch_count() - l0) // max(1, args.steps) * args.steps + args.steps
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    flops = nominal(kind, n)
    value = flops / (ms * 1e-3) / 1e9
    # e2e: host matrix -> owned columns (H2D), reduction, band gathered to rank 0 (D2H)
    dist.barrier()
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    for _ in range(e2e_steps):
        Lh = D.scatter_columns(A_host, lay, ops, kind)
        fn(Lh, lay, w, ops, comm, la)
        D.gather_band(Lh, lay, w, kind, comm, torch)
    torch.cuda.synchronize(dev)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": same_config(args.config, la, world),
            "clocks": clocks.summary(),
            "e2e": {"value": flops / e2e_s / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": n * n * 8,
                    "d2h_bytes_per_step": lay.nblk * b * (b + w) * 8, "steps": e2e_steps,
                    "path": "scatter owned columns + distributed reduction + band strips gathered to rank 0"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "tensor", "kernel": "all", "achieved": value / 1e3 / world,
                         "peak": peak, "unit": "TFLOP/s", "frac": value / 1e3 / world / peak,
                         "peak_source": "cuBLAS DGEMM 8192^3 per GPU, measured in this run",
                         "traffic": None, "note": "whole-job GFLOP/s per GPU vs one GPU's DGEMM peak"},
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--lookahead", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--breakdown-steps", type=int, default=1,
                    help="eager steps timed per kernel class for the roofline")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="run the multi-GPU (block-cyclic, NCCL) driver even at one rank")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if CONFIGS[args.config][0] == "band" and (world > 1 or args.impl == "reference"):
        sys.exit("the band-form workload is single-GPU, ours only")
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif world > 1 or args.dist:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        run_dist(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
