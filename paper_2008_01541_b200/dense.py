"""Standalone dense Schur-complement Cholesky: BASELINE config 4.

The frame solver factors H = sigma0 + C22 inside its CUDA graph
(`linalg.dense_factor`, reference linalg.py:432-440). This module exposes
the same persistent tile kernel on its own, for:

* the config-4 scaling sweep: dense SPD orders 2K-49K, synthetic matrices
  generated on the device (exponential kernel on a
  sqrt(m) x sqrt(m) surface grid, diag ~5e3, kappa ~1e2);
* the tile-cyclic multi-GPU factorization: one process per
  GPU, tile column j owned by rank j mod P, every rank keeping a full replica
  of L that its peers write into over NVLink (CUDA-IPC mappings). There is no
  collective on the data path: each finished tile is pushed by the CTA that
  made it and released to the peers with a system-scope flag, and the peers'
  tasks wait on those per-tile flags exactly as on one GPU.

`TileCyclicCholesky` is the host side of the multi-rank case: it exchanges
the replicas' IPC handles over `torch.distributed` and runs the
reset -> barrier -> launch -> finish -> barrier protocol. The emulated mode
(`DenseCholesky(..., emulate=True)`) factors all ranks' replicas in ONE launch
on one GPU, which exercises the multi-rank data path (pushes, system-scope
flags, per-rank task lists) where only one GPU exists.

No CPU fallback: every entry point runs on the GPU or raises.
"""

from __future__ import annotations

import ctypes
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as nat
from .errors import InvalidArgumentError

IPC_BYTES = 64
MAX_RANKS = 8

# SURVEY.md §8d config 4 synthetic H: K = a exp(-d / ell) + b I on the grid,
# a + b = 5e3 (the measured sigma0 diagonal is 500-5,267), kappa ~ 1.1e2 at
# ell = 2 grid spacings (measured with numpy.linalg.eigvalsh at m = 1K-2K).
SYNTH_A, SYNTH_B, SYNTH_ELL = 4950.0, 50.0, 2.0


def chol_flops(m: int) -> float:
    """Algorithmic flops of one factorization (m^3 / 3)."""
    return float(m) ** 3 / 3.0


def rank_tasks(m: int, rank: int, nranks: int) -> np.ndarray:
    """(i, j) tile tasks of `rank` in claim order (host only, no GPU)."""
    L = nat.lib()
    cnt = ctypes.c_int64(0)
    nat.check(L.spb_dense_rank_tasks(m, rank, nranks, None, ctypes.byref(cnt)))
    out = np.zeros((cnt.value, 2), dtype=np.int32)
    nat.check(L.spb_dense_rank_tasks(m, rank, nranks, nat.ptr(out), ctypes.byref(cnt)))
    return out


def tile_owner(i: int, j: int, nranks: int) -> int:
    """Mirror of dense.cu `dense_tile_owner`: column-cyclic, except that the
    sub-diagonal partial (j+1, j) goes with diagonal j+1 (which finalizes it)."""
    return (i if i == j + 1 else j) % nranks


class DenseCholesky:
    """One dense SPD matrix on the device and its tile Cholesky factor."""

    def __init__(self, m: int, device: int = 0, rank: int = 0, nranks: int = 1, emulate: bool = False,
                 int8: Optional[bool] = None):
        if m <= 0:
            raise InvalidArgumentError("order must be positive")
        if not (1 <= nranks <= MAX_RANKS):
            raise InvalidArgumentError(f"nranks must be in [1, {MAX_RANKS}]")
        nat.require_device()
        self.m, self.rank, self.nranks, self.emulate = int(m), int(rank), int(nranks), bool(emulate)
        h = ctypes.c_void_p()
        nat.check(nat.lib().spb_dense_create(self.m, device, self.rank, self.nranks, int(self.emulate),
                                            ctypes.byref(h)))
        self._h = h
        if int8 is not None:  # default: INT8 tensor cores on one GPU (SPB_CHOL_INT8), DMMA otherwise
            nat.check(nat.lib().spb_dense_set_cholesky_kind(self._h, 1 if int8 else 0))

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            nat.lib().spb_dense_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def replicas(self) -> int:
        return self.nranks if self.emulate else 1

    @property
    def int8(self) -> bool:
        """True when the trailing updates run on the INT8 tensor cores
        (emulated FP64, one GPU); False: FP64 DMMA (tile-cyclic ranks)."""
        k = ctypes.c_int32(0)
        nat.check(nat.lib().spb_dense_cholesky_kind(self._h, ctypes.byref(k)))
        return bool(k.value)

    # -------------------------------------------------------------- matrix
    def set_matrix(self, h: np.ndarray) -> None:
        h = nat.f64(h)
        if h.shape != (self.m, self.m):
            raise InvalidArgumentError(f"matrix must be {self.m} x {self.m}")
        nat.check(nat.lib().spb_dense_set_matrix(self._h, nat.ptr(h)))

    def synthetic(self, a: float = SYNTH_A, b: float = SYNTH_B, ell: float = SYNTH_ELL) -> None:
        nat.check(nat.lib().spb_dense_synthetic(self._h, a, b, ell))

    def matrix(self) -> np.ndarray:
        out = np.zeros((self.m, self.m))
        nat.check(nat.lib().spb_dense_get_matrix(self._h, nat.ptr(out)))
        return out

    def factor_lower(self, replica: int = 0, out: Optional[np.ndarray] = None) -> np.ndarray:
        """L (row-major, strict upper zero), into `out` when given (a reused,
        page-locked buffer makes the download one direct DMA)."""
        if out is None:
            out = np.empty((self.m, self.m))
        elif out.shape != (self.m, self.m) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise InvalidArgumentError("out must be a C-contiguous float64 m x m array")
        nat.check(nat.lib().spb_dense_get_factor(self._h, replica, nat.ptr(out)))
        return out

    # -------------------------------------------------------------- factor
    def factor(self, reps: int = 1) -> float:
        """Factor `reps` times (single process); mean device ms per factorization.
        A non-positive pivot raises IndefiniteMatrixError(column=dpotrf info)."""
        ms = ctypes.c_double(0.0)
        info = ctypes.c_int64(0)
        rc = nat.lib().spb_dense_factor(self._h, reps, ctypes.byref(ms), ctypes.byref(info))
        nat.check(rc, column=int(info.value) if info.value else None)
        return float(ms.value)

    def residual(self, v: np.ndarray, replica: int = 0) -> Tuple[float, float]:
        """(||A v - L L^T v||, ||A v||) computed on the device."""
        v = nat.f64(v)
        out = np.zeros(2)
        nat.check(nat.lib().spb_dense_residual(self._h, replica, nat.ptr(v), nat.ptr(out)))
        return float(out[0]), float(out[1])

    # ---------------------------------------------------- multi-rank steps
    def ipc_handle(self) -> bytes:
        buf = (ctypes.c_uint8 * IPC_BYTES)()
        nat.check(nat.lib().spb_dense_ipc_handle(self._h, buf))
        return bytes(buf)

    def open_peers(self, handles: Sequence[bytes]) -> None:
        blob = b"".join(handles)
        buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        nat.check(nat.lib().spb_dense_open_peers(self._h, buf))

    def reset(self) -> None:
        nat.check(nat.lib().spb_dense_reset(self._h))

    def launch(self) -> None:
        nat.check(nat.lib().spb_dense_launch(self._h))

    def finish(self) -> float:
        ms = ctypes.c_double(0.0)
        info = ctypes.c_int64(0)
        rc = nat.lib().spb_dense_finish(self._h, ctypes.byref(ms), ctypes.byref(info))
        nat.check(rc, column=int(info.value) if info.value else None)
        return float(ms.value)


def gather_handles(local: bytes, rank: int, world: int,
                   all_gather: Callable[[object], List[object]]) -> List[bytes]:
    """Collect every rank's IPC handle in rank order through `all_gather`
    (object all-gather over any torch.distributed backend) and validate it."""
    if len(local) != IPC_BYTES:
        raise InvalidArgumentError(f"IPC handle must be {IPC_BYTES} bytes")
    got = all_gather((rank, local))
    if len(got) != world:
        raise InvalidArgumentError(f"expected {world} handles, got {len(got)}")
    by_rank = {}
    for r, h in got:
        if r in by_rank or not (0 <= r < world) or len(h) != IPC_BYTES:
            raise InvalidArgumentError("malformed handle exchange")
        by_rank[r] = bytes(h)
    return [by_rank[r] for r in range(world)]


def _dist_all_gather(group=None) -> Callable[[object], List[object]]:
    import torch.distributed as dist

    def ag(obj):
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, obj, group=group)
        return out

    return ag


class TileCyclicCholesky:
    """One dense factorization sharded tile-cyclically over the ranks of a
    torch.distributed group (one process per GPU, NVLink peers)."""

    def __init__(self, m: int, device: Optional[int] = None, group=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if device is None:
            device = self.rank
        self.dense = DenseCholesky(m, device=device, rank=self.rank, nranks=self.world)
        if self.world > 1:
            handles = gather_handles(self.dense.ipc_handle(), self.rank, self.world, _dist_all_gather(group))
            self.dense.open_peers(handles)
        self._barrier()

    def _barrier(self) -> None:
        import torch.distributed as dist

        if self.world > 1:
            dist.barrier(group=self.group)

    def factor(self) -> float:
        """One factorization across all ranks; returns this rank's device ms.
        Flags are reset everywhere before any rank starts, and no rank resets
        again before every peer has stopped writing into its replica."""
        self.dense.reset()
        self._barrier()
        self.dense.launch()
        ms = self.dense.finish()
        self._barrier()
        return ms
