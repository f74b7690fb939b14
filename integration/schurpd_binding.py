"""Reference-side binding for libschurpd_b200.so.

A maintainer of the reference package `schurpd` adds this module to route
the "schur" solver kind to the B200 library:

    from schurpd import solver
    import schurpd_binding
    schurpd_binding.install(solver)      # SOLVE_FUNCTIONS["schur"] -> B200

It is plain ctypes over include/schurpd_b200.h and touches only the fields the
reference's own types carry:
  - Model (solver.py:300-324);
  - GlobalSystem (solver.py:149-158);
  - SolverState (solver.py:117-145);
  - SolverConfig (solver.py:74-93);
  - Partition (partition.py:21-44);
  - the shapes (collision.py:57-180);
  - RigidTransform (collision.py:44-54).
Nothing here imports paper_2008_01541_b200. The GPU test
(tests/test_gpu_binding.py) drives it with that package's mirror types, which
have the same field names.

Call order per frame (what solve_frame_schur does, solver.py:387-455):
  1. set_pose: attachment targets plus posed colliders;
  2. set_state: x, active set, targets;
  3. step;
  4. get_state: x in place; active, target, f_tilde2, u2_accum, R (and Q)
     rebound;
  5. FrameMetrics is appended to state.metrics (_finish_metrics,
     solver.py:373-384).
"""

from __future__ import annotations

import ctypes
import os
import time
from pathlib import Path

import numpy as np

LIB = Path(os.environ.get("SCHURPD_B200_LIB", Path(__file__).resolve().parent.parent / "paper_2008_01541_b200"
                          / "lib" / "libschurpd_b200.so"))

P, I32, I64, F64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double


class SceneDesc(ctypes.Structure):  # spb_scene_desc
    _fields_ = [("num_nodes", I64), ("num_elements", I64), ("tets", P), ("dm_inverse", P), ("volume", P),
                ("mu", F64), ("mu_prime", F64), ("sigma_min", F64), ("sigma_max", F64),
                ("n1", I64), ("n2", I64), ("perm", P), ("num_alpha", I64), ("num_beta", I64),
                ("e_alpha", P), ("e_beta", P), ("num_attachments", I64), ("att_nodes", P), ("att_stiffness", P),
                ("num_proxies", I64), ("proxy_elements", P), ("proxy_weights", P), ("proxy_stiffness", P),
                ("k22_indptr", P), ("k22_indices", P), ("k22_data", P)]


class ShapeDesc(ctypes.Structure):  # spb_shape_desc
    _fields_ = [("kind", I32), ("params", F64 * 7), ("dims", I64 * 3), ("values", P)]


class Posed(ctypes.Structure):  # spb_posed_collider
    _fields_ = [("shape", I32), ("rotation", F64 * 9), ("translation", F64 * 3)]


class StepConfig(ctypes.Structure):  # spb_step_config
    _fields_ = [("outer_iters", I32), ("inner_iters", I32), ("cadence", I32), ("use_graph", I32),
                ("unused", I32), ("early_exit_residual", F64)]


class Metrics(ctypes.Structure):  # spb_frame_metrics
    _fields_ = [("t_local_ms", F64), ("t_forward_ms", F64), ("t_detect_ms", F64), ("t_dense_ms", F64),
                ("t_backward_ms", F64), ("t_total_ms", F64), ("energy", F64), ("active_proxies", I64),
                ("max_penetration", F64), ("residual", F64), ("info", I64), ("kernel_launches", I64),
                ("outer_passes", I64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(str(LIB))
        _lib.spb_last_error.restype = ctypes.c_char_p
        _lib.spb_factor_create.argtypes = [I64, I64, P, P, P, P, I32, I32, P, P]
        for name in ("spb_set_host_blas", "spb_ctx_create", "spb_ctx_add_shape", "spb_ctx_set_pose",
                     "spb_ctx_set_state", "spb_ctx_step", "spb_ctx_get_state"):
            getattr(_lib, name).restype = I32
        _lib.spb_ctx_set_pose.argtypes = [P, P, I32, P]
        _lib.spb_ctx_set_state.argtypes = [P] * 8
        _lib.spb_ctx_get_state.argtypes = [P] * 8
        # the multifrontal precompute calls the host BLAS/LAPACK scipy ships
        import scipy.linalg.cython_blas as cb
        import scipy.linalg.cython_lapack as cl

        cap = ctypes.pythonapi.PyCapsule_GetPointer
        cap.restype, cap.argtypes = P, [ctypes.py_object, ctypes.c_char_p]
        capi = [cb.__pyx_capi__[n] for n in ("dgemm", "dsyrk", "dtrsm")]
        capi += [cl.__pyx_capi__[n] for n in ("dpotrf", "dtrtri")]
        name = ctypes.pythonapi.PyCapsule_GetName
        name.restype, name.argtypes = ctypes.c_char_p, [ctypes.py_object]
        _ok(_lib.spb_set_host_blas(*[P(cap(c, name(c))) for c in capi]))
    return _lib


def _ok(rc, column=None):
    if rc != 0:
        msg = lib().spb_last_error().decode(errors="replace")
        raise RuntimeError(f"libschurpd_b200 status {rc}: {msg}" + (f" (column {column})" if column is not None
                                                                     else ""))


def _p(a):
    return P(a.ctypes.data) if a is not None else None


class B200Scene:
    """Device residency of one (Model, GlobalSystem): factor + context."""

    def __init__(self, model, system, device=0):
        mesh, rest, part, prm = model.mesh, model.rest, system.partition, model.params
        up = system.A.upper.tocsc()
        keep = [np.ascontiguousarray(up.indptr, np.int64), np.ascontiguousarray(up.indices, np.int64),
                np.ascontiguousarray(up.data, np.float64),
                np.ascontiguousarray(mesh.rest_positions[system.x1_ids], np.float64)]
        fac, bad = P(), I64(-1)
        _ok(lib().spb_factor_create(up.shape[0], part.n1, *[_p(a) for a in keep], 1 if part.n1 > 1 else 0, 1,
                                    ctypes.byref(fac), ctypes.byref(bad)), bad.value)
        self.factor = fac
        k22 = system.k22_beta.tocsr()
        a = dict(tets=np.ascontiguousarray(mesh.tets, np.int64), dmi=np.ascontiguousarray(rest.dm_inverse),
                 vol=np.ascontiguousarray(rest.volume), perm=np.ascontiguousarray(part.perm, np.int64),
                 ea=np.ascontiguousarray(part.e_alpha, np.int64), eb=np.ascontiguousarray(part.e_beta, np.int64),
                 an=np.array([t.node for t in model.attachments], np.int64),
                 ak=np.array([t.stiffness for t in model.attachments], np.float64),
                 pe=np.ascontiguousarray(model.proxy_elements, np.int64),
                 pw=np.ascontiguousarray(np.reshape(model.proxy_weights, (-1, 4)), np.float64),
                 pc=np.ascontiguousarray(model.proxy_stiffness, np.float64),
                 kp=k22.indptr.astype(np.int64), ki=k22.indices.astype(np.int64), kd=k22.data.astype(np.float64))
        d = SceneDesc(num_nodes=mesh.num_nodes, num_elements=mesh.num_elements, tets=_p(a["tets"]),
                      dm_inverse=_p(a["dmi"]), volume=_p(a["vol"]), mu=prm.mu, mu_prime=prm.mu_prime,
                      sigma_min=prm.sigma_min, sigma_max=prm.sigma_max, n1=part.n1, n2=part.n2,
                      perm=_p(a["perm"]), num_alpha=len(a["ea"]), num_beta=len(a["eb"]), e_alpha=_p(a["ea"]),
                      e_beta=_p(a["eb"]), num_attachments=len(a["an"]), att_nodes=_p(a["an"]),
                      att_stiffness=_p(a["ak"]), num_proxies=len(a["pe"]), proxy_elements=_p(a["pe"]),
                      proxy_weights=_p(a["pw"]), proxy_stiffness=_p(a["pc"]), k22_indptr=_p(a["kp"]),
                      k22_indices=_p(a["ki"]), k22_data=_p(a["kd"]))
        ctx = P()
        _ok(lib().spb_ctx_create(ctypes.byref(d), fac, device, ctypes.byref(ctx)))
        self.ctx = ctx
        self.shapes = {}
        self.n, self.ne, self.P, self.m = mesh.num_nodes, mesh.num_elements, len(a["pe"]), part.n2
        self.biphasic = prm.biphasic

    def __del__(self):
        if _lib is not None and getattr(self, "ctx", None):
            _lib.spb_ctx_destroy(self.ctx)
            _lib.spb_factor_destroy(self.factor)

    def shape_id(self, shape):
        sid = self.shapes.get(id(shape))
        if sid is not None:
            return sid[0]
        d, keep = ShapeDesc(), None
        kind = type(shape).__name__
        prm = np.zeros(7)
        if kind == "HalfSpace":
            d.kind, prm[:3], prm[3:6] = 0, shape.point, shape.normal
        elif kind == "Sphere":
            d.kind, prm[:3], prm[3] = 1, shape.center, shape.radius
        elif kind == "Capsule":
            d.kind, prm[:3], prm[3:6], prm[6] = 2, shape.p0, shape.p1, shape.radius
        elif kind == "GridLevelset":
            d.kind, prm[:3], prm[3] = 3, shape.origin, shape.spacing
            d.dims[:] = shape.dims
            keep = np.ascontiguousarray(np.asarray(shape.values).transpose(2, 1, 0), np.float64).ravel()
            d.values = _p(keep)  # x fastest (collision.py:142-143)
        else:
            raise TypeError(f"unsupported collider shape {kind}")
        d.params[:] = prm
        out = I32(-1)
        _ok(lib().spb_ctx_add_shape(self.ctx, ctypes.byref(d), ctypes.byref(out)))
        self.shapes[id(shape)] = (out.value, shape, keep)
        return out.value


_scenes = {}
_CAD = {"inner": 0, "frame": 1, "never": 2}


def solve_frame_schur_b200(model, system, state, config, _types):
    """solver.py:387-455 on the B200 library."""
    t0 = time.perf_counter()
    key = (id(model), id(system))
    sc = _scenes.get(key)
    if sc is None:
        _scenes.clear()
        sc = _scenes[key] = B200Scene(model, system)
    tg = np.ascontiguousarray(np.reshape([a.target for a in model.attachments], (-1, 3)), np.float64)
    cols = (Posed * max(len(model.colliders), 1))()
    for i, c in enumerate(model.colliders):
        cols[i].shape = sc.shape_id(c.shape)
        cols[i].rotation[:] = np.ravel(c.transform.rotation)
        cols[i].translation[:] = np.ravel(c.transform.translation)
    _ok(lib().spb_ctx_set_pose(sc.ctx, _p(tg), len(model.colliders), ctypes.cast(cols, P)))
    x = state.x  # (n,3) f64 C-contiguous, updated in place
    act = np.ascontiguousarray(state.active.active, np.uint8)
    tgt = np.ascontiguousarray(state.active.target, np.float64)
    _ok(lib().spb_ctx_set_state(sc.ctx, _p(x), None, None, _p(act), _p(tgt), None, None))
    early = config.early_exit_residual
    cfg = StepConfig(config.outer_iters, config.inner_iters, _CAD[config.detection_cadence], 1, 0,
                     -1.0 if early is None else float(early))
    met = Metrics()
    rc = lib().spb_ctx_step(sc.ctx, ctypes.byref(cfg), ctypes.byref(met))
    if rc == 2:  # SPB_ERR_INDEFINITE -> IndefiniteMatrixError in the reference's errors.py
        raise _types["IndefiniteMatrixError"](f"non-positive pivot at column {met.info}", column=int(met.info))
    _ok(rc)
    act_out = np.empty(sc.P, np.uint8)
    tgt_out = np.empty((sc.P, 3))
    f2, u2 = np.empty((sc.m, 3)), np.empty((sc.m, 3))
    R = np.empty((sc.ne, 3, 3))
    Q = np.empty((sc.ne, 3, 3)) if sc.biphasic else None
    _ok(lib().spb_ctx_get_state(sc.ctx, _p(x), _p(R), _p(Q), _p(act_out), _p(tgt_out), _p(f2), _p(u2)))
    state.active = _types["ActiveSet"](act_out.astype(bool), tgt_out)
    state.f_tilde2, state.u2_accum = f2, u2
    state.rotations.r[...] = R
    if Q is not None:
        state.rotations.q[...] = Q
    m = _types["FrameMetrics"](t_local_ms=met.t_local_ms, t_forward_ms=met.t_forward_ms,
                               t_detect_ms=met.t_detect_ms, t_dense_ms=met.t_dense_ms,
                               t_backward_ms=met.t_backward_ms, energy=met.energy,
                               active_proxies=int(met.active_proxies), max_penetration=met.max_penetration,
                               residual=met.residual)
    m.t_total_ms = 1e3 * (time.perf_counter() - t0)
    state.metrics.append(m)
    return m


def install(solver_module, kind: str = "schur"):
    """Register the B200 path in the reference's solver registry
    (solver.py:606-614); SolverConfig validation is unchanged."""
    errors = __import__(solver_module.__name__.rsplit(".", 1)[0] + ".errors", fromlist=["x"])
    types = {"ActiveSet": solver_module.col.ActiveSet, "FrameMetrics": solver_module.FrameMetrics,
             "IndefiniteMatrixError": errors.IndefiniteMatrixError}
    solver_module.SOLVE_FUNCTIONS[kind] = (
        lambda model, system, state, config: solve_frame_schur_b200(model, system, state, config, types))
