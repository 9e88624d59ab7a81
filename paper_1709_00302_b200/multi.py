"""Single-call multi-GPU reductions: the `ngpus` / `devices` extension of the
drop-in API.

`reduce_sym_band(A, cfg, devices=[0, 1, ...])` (or `ngpus=N`) runs the same
1D block-cyclic driver as the torchrun path (`dist.reduce_sym_band_dist` /
`dist.reduce_tri_band_dist`), but from ONE process: one host thread per
device, each with its own library handle and compute stream, and the
collectives issued as single-process NCCL group calls over all devices
(`torch.cuda.nccl`, i.e. one `ncclCommInitAll` communicator set, the plan of
SURVEY 8(e)) on per-device communication streams. The threads meet at a
rendezvous for every collective; rank 0's thread issues the NCCL call for
all of them and hands each rank an event recorded on its communication
stream, which that rank's compute stream waits on (the same event contract
as `dist.TorchComm`, so the driver code is shared unchanged).

The kernels are the same sm_100a library calls as everywhere else (ctypes
releases the GIL, so the threads enqueue concurrently); there is no CPU
path: the device runner raises without CUDA. `HostGroup` runs the identical
rendezvous on CPU tensors so the thread logic is testable without a GPU
(tests/test_multi_threads.py).
"""
from __future__ import annotations

import threading

import numpy as np

from . import dist as D


class _Rendezvous:
    """All ranks deposit a payload; rank 0 runs `lead(payloads)` and returns
    one result per rank. Any failure aborts the barrier so no thread hangs."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.out = [None] * world

    def run(self, rank, payload, lead):
        self.slots[rank] = payload
        self.barrier.wait()
        if rank == 0:
            try:
                out = lead(list(self.slots))
                self.out = list(out) if out is not None else [None] * self.world
            except BaseException:
                self.barrier.abort()
                raise
        self.barrier.wait()
        return self.out[rank]

    def abort(self):
        self.barrier.abort()


class HostGroup:
    """Collectives over CPU tensors held by the threads of one process (the
    host-logic test stand-in for `NcclGroup`). Synchronous; events are None."""

    def __init__(self, world: int):
        self.rv = _Rendezvous(world)

    def comm(self, rank: int):
        return _ThreadComm(self, rank, None)

    def broadcast(self, slots, src):
        for t, _ in slots:
            if t is not slots[src][0]:
                t.copy_(slots[src][0])

    def all_reduce(self, slots):
        total = slots[0][0].clone()
        for t, _ in slots[1:]:
            total += t
        for t, _ in slots:
            t.copy_(total)

    def all_gather(self, slots):
        for out, _ in slots:
            parts = out.view(self.rv.world, -1)
            for r, (_, inp) in enumerate(slots):
                parts[r].copy_(inp)


class NcclGroup:
    """Single-process NCCL over the listed devices (torch.cuda.nccl group
    calls), each collective on the ranks' communication streams."""

    def __init__(self, devices, torch):
        import torch.cuda.nccl as nccl

        self.torch = torch
        self.nccl = nccl
        self.devices = list(devices)
        self.rv = _Rendezvous(len(self.devices))
        self.streams = [torch.cuda.Stream(device=d, priority=-1) for d in self.devices]

    def comm(self, rank: int):
        return _ThreadComm(self, rank, self.streams[rank])

    def _events(self):
        evs = []
        for s in self.streams:
            ev = self.torch.cuda.Event()
            ev.record(s)
            evs.append(ev)
        return evs

    def broadcast(self, slots, src):
        self.nccl.broadcast([t for t, _ in slots], root=src, streams=self.streams)
        return self._events()

    def all_reduce(self, slots):
        self.nccl.all_reduce([t for t, _ in slots], streams=self.streams)
        return self._events()

    def all_gather(self, slots):
        self.nccl.all_gather([inp for _, inp in slots], [out for out, _ in slots],
                             streams=self.streams)
        return self._events()


class _ThreadComm:
    """The `comm` interface of dist.py (broadcast / all_reduce /
    all_gather_into / wait / gather_to0) for one rank thread."""

    def __init__(self, group, rank, stream):
        self.g = group
        self.rank = rank
        self.stream = stream

    def _pre(self, t):
        if self.stream is not None:  # the comm stream waits for this rank's compute stream
            import torch

            self.stream.wait_stream(torch.cuda.current_stream(t.device))

    def wait(self, ev):
        if ev is not None:
            import torch

            torch.cuda.current_stream().wait_event(ev)

    def broadcast(self, t, src: int):
        self._pre(t)
        return self.g.rv.run(self.rank, (t, None), lambda s: self.g.broadcast(s, src))

    def all_reduce(self, t):
        self._pre(t)
        return self.g.rv.run(self.rank, (t, None), self.g.all_reduce)

    def all_gather_into(self, out, inp):
        self._pre(inp)
        return self.g.rv.run(self.rank, (out, inp), self.g.all_gather)

    def gather_to0(self, inp, out_list):
        if self.stream is not None:
            import torch

            torch.cuda.current_stream(inp.device).synchronize()

        def lead(slots):
            outs = slots[0][1]
            for r, (t, _) in enumerate(slots):
                outs[r].copy_(t)  # peer copy to rank 0's device (NVLink) or a host copy
            if self.stream is not None:
                import torch

                torch.cuda.current_stream(outs[0].device).synchronize()

        self.g.rv.run(self.rank, (inp, out_list), lead)


def run_ranks(world, body):
    """Run body(rank) on `world` threads; re-raise the first failure."""
    errors = []
    results = [None] * world

    def worker(rank):
        try:
            results[rank] = body(rank)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errors.append((rank, e))
            abort = getattr(body, "abort", None)
            if abort is not None:
                abort()

    threads = [threading.Thread(target=worker, args=(r,), name=f"bandred-rank{r}") for r in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        real = [e for e in errors if not isinstance(e[1], threading.BrokenBarrierError)]
        rank, e = (real or errors)[0]
        raise e
    return results


class _Body:
    def __init__(self, fn, group):
        self.fn = fn
        self.group = group

    def __call__(self, rank):
        return self.fn(rank)

    def abort(self):
        self.group.rv.abort()


def reduce_on_ranks(A, kind, w, b, world, make_ops, group, lookahead=1,
                    chunk_rows=D.CHUNK_ROWS, finish=None):
    """Drive the block-cyclic reduction of host matrix A on `world` rank
    threads. make_ops(rank) -> rank-local ops (CudaOps / a test stand-in);
    group: NcclGroup or HostGroup. Returns (band, iterations, taus) where
    taus = (tau of the left chain, tau of the right chain or None), indexed
    by each panel's leading column (the reference's per-panel tau)."""
    n = A.shape[0]
    fn = D.reduce_sym_band_dist if kind == "sevp" else D.reduce_tri_band_dist
    out = {}

    def body(rank):
        ops = make_ops(rank)
        try:
            comm = group.comm(rank)
            lay = D.Layout(n, b, world, rank)
            L = D.scatter_columns(A, lay, ops, kind)
            tl, tr = ops.flat(n), ops.flat(n)
            its = fn(L, lay, w, ops, comm, lookahead, chunk_rows=chunk_rows,
                     tau_out=(tl, tr))
            band = D.gather_band(L, lay, w, kind, comm, ops.torch)
            # QR / SEVP taus live on each panel's owner (disjoint, zero
            # elsewhere: summing is exact); LQ taus are identical everywhere
            tl_all = comm.all_reduce(tl)
            comm.wait(tl_all)
            if rank == 0:
                out["band"] = band
                out["its"] = its
                out["taul"] = tl.cpu().numpy()[:n].copy()
                out["taur"] = tr.cpu().numpy()[:n].copy() if kind != "sevp" else None
        finally:
            if finish is not None:
                finish(ops)

    run_ranks(world, _Body(body, group))
    return out["band"], out["its"], (out["taul"], out["taur"])


def resolve_devices(ngpus, devices):
    """None -> single-GPU native path; otherwise the device list of the
    block-cyclic driver (ngpus=N means devices 0..N-1; ngpus=1 alone keeps
    the single-GPU path, devices=[d] forces the driver on one device)."""
    if devices is not None:
        devs = [int(d) for d in devices]
        if not devs:
            raise ValueError("devices must list at least one GPU")
        if len(set(devs)) != len(devs):
            raise ValueError("devices must be distinct (one rank per GPU)")
        if ngpus is not None and int(ngpus) != len(devs):
            raise ValueError(f"ngpus={ngpus} does not match devices={devs}")
        return devs
    if ngpus is None:
        return None
    ngpus = int(ngpus)
    if ngpus < 1:
        raise ValueError("ngpus must be >= 1")
    return None if ngpus == 1 else list(range(ngpus))


def check_dist_shape(n, w, b, what):
    if w != b:
        raise ValueError(f"{what} on several GPUs needs w == b (the 1D block-cyclic driver)")
    if n % b:
        raise ValueError(f"{what} on several GPUs needs n to be a multiple of b")


def reduce_devices(A, kind, w, b, devices, lookahead=1):
    """The device runner behind the `devices=` / `ngpus=` keyword: CUDA ops
    per rank thread over the library's C ABI, NCCL collectives."""
    from . import _dev
    from . import _lib

    torch = _dev.torch()
    ndev = torch.cuda.device_count()
    for d in devices:
        if d < 0 or d >= ndev:
            raise ValueError(f"device {d} does not exist ({ndev} visible)")
    group = NcclGroup(devices, torch)

    def make_ops(rank):
        dev = devices[rank]
        torch.cuda.set_device(dev)
        return D.CudaOps(dev, torch)  # a fresh thread: its own compute stream

    def finish(ops):
        ops.sync()
        _lib.check(ops.lib.br_set_streams(ops.h, None, None), "set_streams")

    return reduce_on_ranks(np.asfortranarray(A), kind, w, b, len(devices), make_ops, group,
                           lookahead, finish=finish)
