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
