"""The 1D block-cyclic distributed driver on a real GPU with NCCL (world size
1 on the single test GPU: exercises the CUDA rank-local kernels - including
the block-column SYR2K/SYMM/GEMM views - and the NCCL plumbing; the
multi-rank logic itself is covered by tests/test_dist_gloo.py)."""
import socket

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl():
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,b,la", [("sevp", 512, 32, 1), ("sevp", 384, 64, 0),
                                         ("tri", 512, 32, 1), ("tri", 384, 64, 0)])
def test_distributed_driver_on_gpu(nccl, kind, n, b, la):
    import torch

    from paper_1709_00302_b200 import dist as D

    rng = np.random.default_rng(11)
    g = rng.standard_normal((n, n))
    A = np.asfortranarray((g + g.T) / 2 if kind == "sevp" else g)
    lay = D.Layout(n, b, 1, 0)
    ops = D.CudaOps(0, torch)
    comm = D.TorchComm(nccl)
    L = D.scatter_columns(A, lay, ops)
    if kind == "sevp":
        it = D.reduce_sym_band_dist(L, lay, b, ops, comm, la)
        ref, _, it_ref = O.reduce_sym_band(A, n, b, b)
    else:
        it = D.reduce_tri_band_dist(L, lay, b, ops, comm, la)
        ref, _, _, it_ref = O.reduce_tri_band(A, b, b)
    ops.sync()
    band = D.gather_band(L, lay, b, kind, comm, torch)
    assert it == it_ref
    assert O.band_check(band, b if kind == "sevp" else 0, b) == 0.0
    assert np.linalg.norm(band - ref) / np.linalg.norm(A) <= 1e-12 * np.sqrt(n)
