"""The real multi-process path of the tile-cyclic factorization, minus the
kernel: two processes on this one GPU exchange their replicas' CUDA-IPC
handles over a gloo group (dense.gather_handles), open each other's
allocation (spb_dense_open_peers) and read what the peer wrote into its first
L tile and flag words. No kernel waits on a peer here: the B200 profiling
guide forbids ranks whose kernels wait on one another on one GPU, so the
pushes and system-scope flags are covered by the emulated single-launch mode
(test_gpu_dense.py) and this covers the handle / offset / mapping plumbing."""

import os
import socket
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import ctypes
    import sys

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from paper_2008_01541_b200 import _native as nat
    from paper_2008_01541_b200 import dense

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = dense.DenseCholesky(300, device=0, rank=rank, nranks=world)
        handles = dense.gather_handles(d.ipc_handle(), rank, world, dense._dist_all_gather())
        d.open_peers(handles)
        nat.check(nat.lib().spb_dense_debug_replica(d._h, -1, float(10 + rank), None, None))
        dist.barrier()
        v = ctypes.c_double(0)
        f = ctypes.c_int32(0)
        nat.check(nat.lib().spb_dense_debug_replica(d._h, 0, 0.0, ctypes.byref(v), ctypes.byref(f)))
        np.save(Path(out_dir) / f"r{rank}.npy", np.array([v.value, f.value]))
        dist.barrier()  # nobody closes its allocation while the peer reads it
        d.close()
    finally:
        dist.destroy_process_group()


def test_ipc_replicas_two_processes(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        v, f = np.load(tmp_path / f"r{r}.npy")
        assert v == 10 + (1 - r) and f == 10 + (1 - r)
