"""ctypes binding of the C ABI (include/schurpd_b200.h) -> libschurpd_b200.so.

This is the only module that touches the native library. Status codes are
mapped to the reference's exception classes (errors.py). There is no CPU
fallback: if the library (or a CUDA device, for device entry points) is
missing, calls raise instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes
import os
import weakref
import subprocess
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

from .errors import (
    DeviceError,
    IndefiniteMatrixError,
    InvalidArgumentError,
    PartitionError,
    SchurPDError,
    SolverSetupError,
)

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "lib" / os.environ.get("SPB_LIB_NAME", "libschurpd_b200.so")
CSRC = PKG / "csrc"

SPB_OK, SPB_ERR_ARG, SPB_ERR_INDEFINITE, SPB_ERR_PARTITION, SPB_ERR_SETUP, SPB_ERR_CUDA, SPB_ERR_ALLOC = range(7)
SHAPE_KINDS = {"half_space": 0, "sphere": 1, "capsule": 2, "levelset": 3}
CADENCES = {"inner": 0, "frame": 1, "never": 2}

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
F64 = ctypes.c_double


class SceneDesc(ctypes.Structure):
    _fields_ = [
        ("num_nodes", I64), ("num_elements", I64), ("tets", P), ("dm_inverse", P), ("volume", P),
        ("mu", F64), ("mu_prime", F64), ("sigma_min", F64), ("sigma_max", F64),
        ("n1", I64), ("n2", I64), ("perm", P), ("num_alpha", I64), ("num_beta", I64),
        ("e_alpha", P), ("e_beta", P),
        ("num_attachments", I64), ("att_nodes", P), ("att_stiffness", P),
        ("num_proxies", I64), ("proxy_elements", P), ("proxy_weights", P), ("proxy_stiffness", P),
        ("k22_indptr", P), ("k22_indices", P), ("k22_data", P),
    ]


class ShapeDesc(ctypes.Structure):
    _fields_ = [("kind", I32), ("params", F64 * 7), ("dims", I64 * 3), ("values", P)]


class PosedCollider(ctypes.Structure):
    _fields_ = [("shape", I32), ("rotation", F64 * 9), ("translation", F64 * 3)]


class StepConfig(ctypes.Structure):
    _fields_ = [("outer_iters", I32), ("inner_iters", I32), ("cadence", I32), ("use_graph", I32),
                ("unused", I32), ("early_exit_residual", F64)]


class FrameIO(ctypes.Structure):
    _fields_ = [("att_targets", P), ("num_colliders", I32), ("colliders", P), ("x", P), ("active", P),
                ("target", P), ("f_tilde2", P), ("u2_accum", P)]


class FrameMetricsC(ctypes.Structure):
    _fields_ = [("t_local_ms", F64), ("t_forward_ms", F64), ("t_detect_ms", F64), ("t_dense_ms", F64),
                ("t_backward_ms", F64), ("t_total_ms", F64), ("energy", F64), ("active_proxies", I64),
                ("max_penetration", F64), ("residual", F64), ("info", I64), ("kernel_launches", I64),
                ("outer_passes", I64)]


_SIGS = {
    "spb_version": ([], I32),
    "spb_last_error": ([], ctypes.c_char_p),
    "spb_device_count": ([P], I32),
    "spb_get_device": ([P], I32),
    "spb_ctx_cholesky_kind": ([P, P], I32),
    "spb_dense_cholesky_kind": ([P, P], I32),
    "spb_dense_set_cholesky_kind": ([P, I32], I32),
    "spb_host_register": ([P, I64], I32),
    "spb_host_unregister": ([P], I32),
    "spb_set_host_blas": ([P, P, P, P, P], I32),
    "spb_factor_create": ([I64, I64, P, P, P, P, I32, I32, P, P], I32),
    "spb_factor_destroy": ([P], None),
    "spb_factor_info": ([P, P], I32),
    "spb_factor_fill_perm": ([P, P], I32),
    "spb_factor_export_l1": ([P, P, P, P], I32),
    "spb_factor_export_coupling": ([P, P, P, P], I32),
    "spb_factor_sigma0": ([P, P], I32),
    "spb_factor_supernodes": ([P, P, P, P, P, P], I32),
    "spb_fill_ordering": ([I64, P, P, P, P], I32),
    "spb_symbolic_nnz": ([I64, P, P, P], I32),
    "spb_ctx_create": ([P, P, I32, P], I32),
    "spb_ctx_destroy": ([P], None),
    "spb_ctx_add_shape": ([P, P, P], I32),
    "spb_ctx_set_pose": ([P, P, I32, P], I32),
    "spb_ctx_set_state": ([P, P, P, P, P, P, P, P], I32),
    "spb_ctx_step": ([P, P, P], I32),
    "spb_ctx_frame": ([P, P, I32, P, P, P, P, P, P, P, P], I32),
    "spb_ctx_frame_io": ([P, P, I32, P, P, P, P, P, P, P, P, P, P], I32),
    "spb_ctx_get_state": ([P, P, P, P, P, P, P, P], I32),
    "spb_ctx_bench": ([P, P, I32, P, P], I32),
    "spb_ctx_bench_cholesky": ([P, I32, P], I32),
    "spb_ctx_bench_kernel": ([P, I32, I32, P], I32),
    "spb_ctx_trace_dense_backward": ([P, P, P], I32),
    "spb_bench_batch": ([P, I32, P, I32, P], I32),
    "spb_ctx_set_concurrency": ([P, I32], I32),
    "spb_frame_batch": ([P, I32, P, P, P], I32),
    "spb_ctx_trace_cholesky": ([P, P, P, P], I32),
    "spb_op_deformation_gradients": ([I64, P, P, I64, P, I64, P, P], I32),
    "spb_op_svd": ([I64, P, P, P, P, P, P, F64, F64], I32),
    "spb_op_elastic": ([I64, P, P, P, I64, P, P, P, F64, F64, I64, P, P, P], I32),
    "spb_op_detect": ([I64, P, P, I64, P, P, I32, P, P, P, P, P], I32),
    "spb_scatter_proxies": ([P, I64, I64, P, I64, P, I32, P, P, P, P], I32),
    "spb_op_dense_factor": ([I64, P, P, P], I32),
    "spb_op_dense_solve": ([I64, P, I64, P, P], I32),
    "spb_op_forward_sub": ([P, I64, P, P, P, P], I32),
    "spb_op_backward_sub": ([P, I64, P, P, P], I32),
    "spb_ctx_set_operator": ([P, I64, P, P, P], I32),
    "spb_ctx_frame_pcg": ([P, P, I32, P, P, P, P, P, F64, I64, P, P], I32),
    "spb_dense_create": ([I64, I32, I32, I32, I32, P], I32),
    "spb_dense_destroy": ([P], None),
    "spb_dense_set_matrix": ([P, P], I32),
    "spb_dense_synthetic": ([P, F64, F64, F64], I32),
    "spb_dense_get_matrix": ([P, P], I32),
    "spb_dense_get_factor": ([P, I32, P], I32),
    "spb_dense_ipc_handle": ([P, P], I32),
    "spb_dense_open_peers": ([P, P], I32),
    "spb_dense_debug_replica": ([P, I32, F64, P, P], I32),
    "spb_dense_reset": ([P], I32),
    "spb_dense_launch": ([P], I32),
    "spb_dense_finish": ([P, P, P], I32),
    "spb_dense_factor": ([P, I32, P, P], I32),
    "spb_dense_residual": ([P, I32, P, P], I32),
    "spb_dense_rank_tasks": ([I64, I32, I32, P, P], I32),
}
EXPORTED = tuple(_SIGS)

_lib = None


def build(force: bool = False) -> Path:
    """Compile the library in-tree (make); used by __graft_entry__.build()."""
    if force or not LIB_PATH.exists() or _stale():
        subprocess.run(["make", "-s", "-j8", "-C", str(CSRC)], check=True)
    return LIB_PATH


def _stale() -> bool:
    t = LIB_PATH.stat().st_mtime
    srcs = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")) + list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh"))
    srcs.append(PKG.parent / "include" / "schurpd_b200.h")
    return any(s.stat().st_mtime > t for s in srcs if s.exists())


def lib():
    """Load the C-ABI library (raises if it was never built: no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DeviceError(f"native library {LIB_PATH} is missing; run __graft_entry__.build()")
        L = ctypes.CDLL(str(LIB_PATH))
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _register_blas(L)
        _lib = L
    return _lib


def _capsule_ptr(capsule) -> int:
    get_name = ctypes.pythonapi.PyCapsule_GetName
    get_name.restype = ctypes.c_char_p
    get_name.argtypes = [ctypes.py_object]
    get_ptr = ctypes.pythonapi.PyCapsule_GetPointer
    get_ptr.restype = ctypes.c_void_p
    get_ptr.argtypes = [ctypes.py_object, ctypes.c_char_p]
    return get_ptr(capsule, get_name(capsule))


def _register_blas(L) -> None:
    """Hand the precompute scipy's LAPACK/BLAS (Fortran ABI) function pointers."""
    import scipy.linalg.cython_blas as cb
    import scipy.linalg.cython_lapack as cl

    ptr = [_capsule_ptr(cb.__pyx_capi__[n]) for n in ("dgemm", "dsyrk", "dtrsm")]
    ptr += [_capsule_ptr(cl.__pyx_capi__[n]) for n in ("dpotrf", "dtrtri")]
    check(L.spb_set_host_blas(*[ctypes.c_void_p(p) for p in ptr]))


def last_error() -> str:
    return lib().spb_last_error().decode(errors="replace")


def check(rc: int, column: Optional[int] = None) -> None:
    if rc == SPB_OK:
        return
    msg = last_error()
    if rc == SPB_ERR_ARG:
        raise InvalidArgumentError(msg)
    if rc == SPB_ERR_INDEFINITE:
        raise IndefiniteMatrixError(msg + (f" (column {column})" if column is not None else ""), column=column)
    if rc == SPB_ERR_PARTITION:
        raise PartitionError(msg)
    if rc == SPB_ERR_SETUP:
        raise SolverSetupError(msg)
    if rc in (SPB_ERR_CUDA, SPB_ERR_ALLOC):
        raise DeviceError(msg)
    raise SchurPDError(f"native error {rc}: {msg}")


def ptr(a: Optional[np.ndarray]):
    """A c_void_p that also keeps `a` alive (call sites pass temporaries)."""
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def addr(a: Optional[np.ndarray]):
    """The bare buffer address (int) for the per-frame hot path: cheaper than
    ptr(), but the CALLER must hold a reference to `a` for the call."""
    return None if a is None else a.ctypes.data


def f64(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


# ---------------------------------------------------------- pinned reuse
_pinned: dict = {}  # data pointer -> weakref.finalize of the owning array
_seen: dict = {}    # data pointer -> id of the owning array at first sighting


def _unpin(ptr: int) -> None:
    _pinned.pop(ptr, None)
    if _lib is not None:
        _lib.spb_host_unregister(ctypes.c_void_p(ptr))


def pin_reused(arr: np.ndarray, min_bytes: int = 1 << 20) -> None:
    """Page-lock `arr`'s buffer in place the second time the same buffer is
    handed to the device path (a SolverState.x stepped frame after frame), so
    its upload/download is a direct DMA instead of a staged copy. The
    registration is dropped (finalizer on the owning array) before numpy frees
    the memory."""
    if not (isinstance(arr, np.ndarray) and arr.flags.c_contiguous and arr.nbytes >= min_bytes):
        return
    ptr = arr.ctypes.data
    if ptr in _pinned:
        return
    root = arr
    while isinstance(root.base, np.ndarray):
        root = root.base
    if root.base is not None or root.ctypes.data != ptr or root.nbytes != arr.nbytes:
        return  # memory owned elsewhere, or a sub-range: leave it to the staging path
    if _seen.get(ptr) != id(root):
        if len(_seen) > 64:
            _seen.clear()
        _seen[ptr] = id(root)
        return
    if lib().spb_host_register(ctypes.c_void_p(ptr), arr.nbytes) != SPB_OK:
        return
    _pinned[ptr] = weakref.finalize(root, _unpin, ptr)


def device_count() -> int:
    c = ctypes.c_int32(0)
    rc = lib().spb_device_count(ctypes.byref(c))
    return int(c.value) if rc == SPB_OK else 0


def default_device() -> int:
    """The GPU this process drives: SPB_DEVICE, else LOCAL_RANK (torchrun: one
    process per GPU; folded onto the visible devices when a launcher already
    restricted CUDA_VISIBLE_DEVICES per rank), else the current CUDA device."""
    for var in ("SPB_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(var)
        if v not in (None, ""):
            n = device_count()
            d = int(v)
            return d if d < n or n == 0 else d % n
    c = ctypes.c_int32(0)
    return int(c.value) if lib().spb_get_device(ctypes.byref(c)) == SPB_OK else 0


def require_device() -> None:
    if device_count() < 1:
        raise DeviceError("no CUDA device visible: the solver runs on the GPU only (no CPU fallback)")


# ------------------------------------------------------------------ factor


class NativeFactor:
    """Owns an spb_factor handle (supernodal partial factor)."""

    def __init__(self, n: int, n1: int, upper, coords=None, ordering: int = 1, relax: int = 1):
        upper = upper.tocsc()
        upper.sort_indices()
        self._keep = (i64(upper.indptr), i64(upper.indices), f64(upper.data),
                      None if coords is None else f64(coords, (-1, 3)))
        h = ctypes.c_void_p()
        bad = ctypes.c_int64(-1)
        rc = lib().spb_factor_create(n, n1, ptr(self._keep[0]), ptr(self._keep[1]), ptr(self._keep[2]),
                                     ptr(self._keep[3]), ordering, relax, ctypes.byref(h), ctypes.byref(bad))
        self.handle = h
        if rc != SPB_OK:
            self.handle = None
            check(rc, column=int(bad.value) if bad.value >= 0 else None)
        info = np.zeros(8, dtype=np.int64)
        check(lib().spb_factor_info(self.handle, ptr(info)))
        (self.n1, self.n2, self.nsuper, self.nnz_l1, self.nnz_c, self.levels,
         self.panel_values, self.panel_rows) = (int(v) for v in info)
        self._keep = None

    def fill_perm(self) -> np.ndarray:
        out = np.empty(self.n1, dtype=np.int64)
        check(lib().spb_factor_fill_perm(self.handle, ptr(out)))
        return out

    def l1_csc(self):
        ip = np.empty(self.n1 + 1, dtype=np.int64)
        ix = np.empty(self.nnz_l1, dtype=np.int64)
        dx = np.empty(self.nnz_l1, dtype=np.float64)
        check(lib().spb_factor_export_l1(self.handle, ptr(ip), ptr(ix), ptr(dx)))
        return ip, ix, dx

    def coupling_csr(self):
        ip = np.empty(self.n2 + 1, dtype=np.int64)
        ix = np.empty(self.nnz_c, dtype=np.int64)
        dx = np.empty(self.nnz_c, dtype=np.float64)
        check(lib().spb_factor_export_coupling(self.handle, ptr(ip), ptr(ix), ptr(dx)))
        return ip, ix, dx

    def sigma0(self) -> np.ndarray:
        out = np.empty((self.n2, self.n2), dtype=np.float64)
        check(lib().spb_factor_sigma0(self.handle, ptr(out)))
        return out

    def supernodes(self):
        ns = self.nsuper
        first = np.empty(ns + 1, dtype=np.int64)
        rowptr = np.empty(ns + 1, dtype=np.int64)
        rows = np.empty(self.panel_rows, dtype=np.int64)
        parent = np.empty(ns, dtype=np.int64)
        level = np.empty(ns, dtype=np.int64)
        check(lib().spb_factor_supernodes(self.handle, ptr(first), ptr(rowptr), ptr(rows), ptr(parent), ptr(level)))
        return first, rowptr, rows, parent, level

    def forward_sub(self, b1: np.ndarray, b2: np.ndarray):
        require_device()
        k = b1.shape[1]
        y1 = np.empty((self.n1, k)); y2 = np.empty((self.n2, k))
        check(lib().spb_op_forward_sub(self.handle, k, ptr(f64(b1)), ptr(f64(b2)), ptr(y1), ptr(y2)))
        return y1, y2

    def backward_sub(self, y1: np.ndarray, x2: np.ndarray):
        require_device()
        k = y1.shape[1]
        x1 = np.empty((self.n1, k))
        check(lib().spb_op_backward_sub(self.handle, k, ptr(f64(y1)), ptr(f64(x2)), ptr(x1)))
        return x1

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.spb_factor_destroy(self.handle)
            self.handle = None


def fill_ordering(n: int, upper, coords=None) -> np.ndarray:
    upper = upper.tocsc()
    ap, ai = i64(upper.indptr), i64(upper.indices)
    c = None if coords is None else f64(coords, (-1, 3))
    out = np.empty(n, dtype=np.int64)
    check(lib().spb_fill_ordering(n, ptr(ap), ptr(ai), ptr(c), ptr(out)))
    return out


def symbolic_nnz(n: int, upper) -> int:
    upper = upper.tocsc()
    upper.sort_indices()
    ap, ai = i64(upper.indptr), i64(upper.indices)
    out = ctypes.c_int64(0)
    check(lib().spb_symbolic_nnz(n, ptr(ap), ptr(ai), ctypes.byref(out)))
    return int(out.value)


# ------------------------------------------------------------------- ops


def op_deformation_gradients(tets, dm_inverse, x, elements=None) -> np.ndarray:
    require_device()
    tets = i64(tets); dmi = f64(dm_inverse); x = f64(x)
    sub = None if elements is None else i64(elements)
    k = len(tets) if sub is None else len(sub)
    F = np.empty((k, 3, 3))
    if k:
        check(lib().spb_op_deformation_gradients(len(tets), ptr(tets), ptr(dmi), len(x), ptr(x), k, ptr(sub), ptr(F)))
    return F


def op_svd(F, want=("U", "S", "V", "R", "Q"), sigma_min=0.0, sigma_max=0.0):
    require_device()
    F = f64(F, (-1, 3, 3))
    k = len(F)
    out = {n: (np.empty((k, 3)) if n == "S" else np.empty((k, 3, 3))) for n in want}
    if k:
        check(lib().spb_op_svd(k, ptr(F), ptr(out.get("U")), ptr(out.get("S")), ptr(out.get("V")),
                               ptr(out.get("R")), ptr(out.get("Q")), float(sigma_min), float(sigma_max)))
    return out


def op_elastic(tets, dm_inverse, volume, x, R, Q, mu, mu_prime, elements=None, forces=True, energy=False):
    require_device()
    tets = i64(tets); dmi = f64(dm_inverse); vol = f64(volume); x = f64(x); R = f64(R)
    Q = None if Q is None else f64(Q)
    sub = None if elements is None else i64(elements)
    fout = np.empty((len(x), 3)) if forces else None
    eout = np.zeros(1) if energy else None
    check(lib().spb_op_elastic(len(tets), ptr(tets), ptr(dmi), ptr(vol), len(x), ptr(x), ptr(R), ptr(Q),
                               float(mu), float(mu_prime), 0 if sub is None else len(sub), ptr(sub),
                               ptr(fout), ptr(eout)))
    return fout, (None if eout is None else float(eout[0]))


def shape_desc(shape) -> ShapeDesc:
    """Shape object (collision.HalfSpace/Sphere/Capsule/GridLevelset) -> ShapeDesc.
    The returned struct keeps a reference to the level-set value buffer."""
    d = ShapeDesc()
    kind = shape.KIND
    d.kind = SHAPE_KINDS[kind]
    prm = np.zeros(7)
    keep = None
    if kind == "half_space":
        prm[:3] = shape.point; prm[3:6] = shape.normal
    elif kind == "sphere":
        prm[:3] = shape.center; prm[3] = shape.radius
    elif kind == "capsule":
        prm[:3] = shape.p0; prm[3:6] = shape.p1; prm[6] = shape.radius
    else:
        prm[:3] = shape.origin; prm[3] = shape.spacing
        for a in range(3):
            d.dims[a] = shape.dims[a]
        keep = f64(shape.flat_values)
        d.values = keep.ctypes.data
    for k in range(7):
        d.params[k] = float(prm[k])
    d._keep = keep
    return d


def scatter_proxies(tets: np.ndarray, n: int, surface_tris: np.ndarray, mask: np.ndarray, per_element: int,
                    bary: np.ndarray):
    """collision.scatter_proxies on the device (spb_scatter_proxies): (elements,
    weights) of the proxies, or None when the device path does not apply
    (no GPU, node ids >= 2^21, a triangle that is no tet's face)."""
    if os.environ.get("SPB_SETUP_DEVICE", "1") == "0" or device_count() < 1:
        return None
    t = i64(tets)
    st = i64(surface_tris)
    mk = np.ascontiguousarray(mask, dtype=np.uint8)
    b = f64(bary)
    ns = len(st)
    elem = np.empty(max(ns * per_element, 1), dtype=np.int64)
    w = np.empty((max(ns * per_element, 1), 4))
    cnt = ctypes.c_int64(0)
    rc = lib().spb_scatter_proxies(ptr(t), len(t), int(n), ptr(st), ns, ptr(mk), int(per_element), ptr(b), ptr(elem),
                                   ptr(w), ctypes.byref(cnt))
    if rc == SPB_ERR_ARG:
        return None
    check(rc)
    k = int(cnt.value)
    return elem[:k], w[:k]


def posed(shape_id: int, rotation, translation) -> PosedCollider:
    p = PosedCollider()
    p.shape = shape_id
    r = f64(rotation).ravel(); t = f64(translation).ravel()
    if r.size != 9 or t.size != 3:
        raise ValueError("collider rotation must be 3 x 3 and translation 3-vector")
    ctypes.memmove(p.rotation, r.ctypes.data, 72)
    ctypes.memmove(p.translation, t.ctypes.data, 24)
    return p


def op_detect(x, tets, proxy_elements, proxy_weights, colliders: Sequence):
    """colliders: sequence of (shape, rotation, translation)."""
    require_device()
    x = f64(x); tets = i64(tets); pe = i64(proxy_elements); pw = f64(proxy_weights, (-1, 4))
    Pn = len(pe)
    active = np.zeros(Pn, dtype=np.uint8)
    target = np.zeros((Pn, 3))
    depth = np.zeros(Pn)
    if Pn == 0 or not colliders:
        return active.astype(bool), target, depth
    shapes = (ShapeDesc * len(colliders))()
    poses = (PosedCollider * len(colliders))()
    keep = []
    for i, (shape, R, t) in enumerate(colliders):
        sd = shape_desc(shape)
        keep.append(sd._keep)
        shapes[i] = sd
        poses[i] = posed(i, R, t)
    check(lib().spb_op_detect(len(x), ptr(x), ptr(tets), Pn, ptr(pe), ptr(pw), len(colliders),
                              ctypes.cast(shapes, ctypes.c_void_p), ctypes.cast(poses, ctypes.c_void_p),
                              ptr(active), ptr(target), ptr(depth)))
    return active.astype(bool), target, depth


def op_dense_factor(h: np.ndarray):
    require_device()
    h = f64(h)
    m = h.shape[0]
    chol = np.empty_like(h)
    info = ctypes.c_int64(0)
    rc = lib().spb_op_dense_factor(m, ptr(h), ptr(chol), ctypes.byref(info))
    if rc != SPB_OK:
        check(rc, column=int(info.value) - 1 if info.value > 0 else None)
    return chol


def op_dense_solve(chol: np.ndarray, g: np.ndarray) -> np.ndarray:
    require_device()
    chol = f64(chol)
    g2 = f64(g).reshape(chol.shape[0], -1)
    out = np.empty_like(g2)
    check(lib().spb_op_dense_solve(chol.shape[0], ptr(chol), g2.shape[1], ptr(g2), ptr(out)))
    return out.reshape(np.shape(g))
