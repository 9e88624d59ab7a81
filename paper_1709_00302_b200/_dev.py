"""Host <-> device plumbing (PyTorch is used only for device memory/streams)."""
from __future__ import annotations

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        if not t.cuda.is_available():
            raise RuntimeError("paper_1709_00302_b200 needs a CUDA device (there is no CPU fallback)")
        _torch = t
    return _torch


_device = 0


def set_device(device: int):
    global _device
    _device = int(device)


def get_device() -> int:
    return _device


def ctx(device=None):
    """(handle, torch device) for the current/selected GPU."""
    d = _device if device is None else int(device)
    t = torch()
    return _lib.handle(d), t.device("cuda", d)


def call(what: str, fn, *args):
    """Run a kernel-level C-ABI call ordered after torch's pending host->device
    copies and before any device->host copy of its results (the library works
    on its own non-blocking streams)."""
    t = torch()
    t.cuda.current_stream().synchronize()
    h = args[0]
    _lib.check(fn(*args), what)
    _lib.check(_lib.load().br_sync(h), what + " (sync)")


def run_traced(h, groups, fn):
    """Run one reduction call `fn() -> rc`. If `groups` carries an EventTrace
    (ExecGroups does, like the reference's, ref runtime.py:142-160), the
    library's per-task device trace of this call is appended to it: task id
    "qr@k" / "left@k" / ..., group "seq" for the panel stream (the T_S role)
    and "par" for the main stream (T_P), start/end in microseconds."""
    trace = getattr(groups, "trace", None)
    lib = _lib.load()
    if trace is None:
        return fn()
    _lib.check(lib.br_set_timing(h, 2), "trace")
    try:
        rc = fn()
        if rc == 0:
            import ctypes as C

            buf = C.create_string_buffer(64)
            s, t0, t1 = C.c_int(), C.c_double(), C.c_double()
            for i in range(lib.br_trace_count(h)):
                _lib.check(lib.br_trace_get(h, i, buf, 64, C.byref(s), C.byref(t0), C.byref(t1)),
                           "trace")
                trace.append(buf.value.decode(), "seq" if s.value == 1 else "par", t0.value,
                             t1.value)
    finally:
        lib.br_set_timing(h, 0)
    return rc


def ld_pad(rows: int) -> int:
    """Device leading dimension: rows rounded up to 32 doubles (256 B)."""
    return max(32, (rows + 31) // 32 * 32)


class DevMat:
    """A column-major fp64 device matrix (rows x cols, leading dim ld)."""

    def __init__(self, rows, cols, dev, ld=None, zero=False):
        t = torch()
        self.rows, self.cols = int(rows), int(cols)
        self.ld = ld_pad(self.rows) if ld is None else int(ld)
        alloc = t.zeros if zero else t.empty
        self.t = alloc((max(self.cols, 1), self.ld), dtype=t.float64, device=dev)

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    @classmethod
    def from_host(cls, a: np.ndarray, dev):
        a = np.asarray(a, dtype=np.float64)
        if a.ndim == 1:
            a = a.reshape(-1, 1)
        m = cls(a.shape[0], a.shape[1], dev)
        t = torch()
        if a.size:
            host = t.from_numpy(np.asfortranarray(a).T.copy())  # (cols, rows) row-major
            m.t[: m.cols, : m.rows].copy_(host)
        return m

    def to_host(self) -> np.ndarray:
        out = self.t[: self.cols, : self.rows].cpu().numpy()
        return np.asfortranarray(out.T)
