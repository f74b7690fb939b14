"""ORACLE — CPU restatement of the reference per-frame Schur solve.

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module,
and only as the checker or as the timed CPU baseline; the product package
(`paper_2008_01541_b200`) never imports it.

It restates, on plain arrays, the algorithm of the reference package
`schurpd` (/root/reference/pkg/src/schurpd). Each function cites the
reference file:line it follows. The numba kernels are restated in C
(oracle_c.c, built by oracle/Makefile, FP contraction off) so rotations are
bit-identical; numpy/scipy calls are the same library calls the reference
makes, so the remaining arithmetic is bit-identical on the same host too.

Parity pinning: tests/test_oracle.py checks this oracle against the golden
fixtures under tests/golden/, which were produced by running the reference
itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional

import numpy as np
import scipy.linalg
import scipy.sparse as sp

_HERE = Path(__file__).resolve().parent
_LIB = None


def build() -> Path:
    """Compile oracle_c.c (make) and return the library path."""
    so = _HERE / "_build" / "liboracle.so"
    src = _HERE / "oracle_c.c"
    if not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return so


def lib():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(str(build()))
        P = ctypes.c_void_p
        I = ctypes.c_int64
        for name, args in {
            "or_signed_svd": [I, P, P, P, P],
            "or_uvt": [I, P, P, P],
            "or_udvt": [I, P, P, P, P],
            "or_lsolve": [I, P, P, P, P],
            "or_ltsolve": [I, P, P, P, P],
            "or_lsolve3": [I, P, P, P, P],
            "or_ltsolve3": [I, P, P, P, P],
        }.items():
            fn = getattr(_LIB, name)
            fn.argtypes = args
            fn.restype = None
    return _LIB


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------ element math


def signed_svd_batch(F: np.ndarray):
    """material.py:116-221 (numba) -> C restatement."""
    F = np.ascontiguousarray(F, dtype=np.float64)
    n = len(F)
    U = np.empty_like(F); S = np.empty((n, 3)); V = np.empty_like(F)
    lib().or_signed_svd(n, _p(F), _p(U), _p(S), _p(V))
    return U, S, V


def polar_rotations(F):
    """material.py:259-269: R = U V^T of the sign-carrying SVD."""
    U, S, V = signed_svd_batch(F)
    R = np.empty_like(U)
    lib().or_uvt(len(U), _p(U), _p(V), _p(R))
    return R


def biphasic_projections(F, sigma_min, sigma_max):
    """material.py:276-290: Q = U clip(S) V^T."""
    U, S, V = signed_svd_batch(F)
    np.clip(S, sigma_min, sigma_max, out=S)
    Q = np.empty_like(U)
    lib().or_udvt(len(U), _p(U), _p(S), _p(V), _p(Q))
    return Q


def deformation_gradients(x, tets, dmi):
    """mesh.py:239-244: F = Ds Dm^-1 (numpy stacked matmul)."""
    ds = np.swapaxes(x[tets[:, 1:]] - x[tets[:, :1]], 1, 2)
    return ds @ dmi


# ------------------------------------------------------------- scene data


@dataclass
class OCollider:
    """Posed collider (collision.py:186-203): kind in half_space|sphere|capsule|levelset."""

    kind: str
    params: dict
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))


@dataclass
class OScene:
    """Frame-constant data of the reference `Model` (solver.py:299-318), as arrays."""

    tets: np.ndarray
    dm_inverse: np.ndarray
    volume: np.ndarray
    mu: float
    mu_prime: float
    sigma_min: float
    sigma_max: float
    att_nodes: np.ndarray
    att_k: np.ndarray
    att_targets: np.ndarray
    prox_elem: np.ndarray
    prox_w: np.ndarray
    prox_c: np.ndarray
    colliders: List[OCollider]
    num_nodes: int

    @property
    def biphasic(self) -> bool:
        return self.mu_prime > 0.0


@dataclass
class OSystem:
    """Reference GlobalSystem + PartialFactor fields (solver.py:148-158, linalg.py:298-319)."""

    n1: int
    n2: int
    perm: np.ndarray
    e_alpha: np.ndarray
    e_beta: np.ndarray
    l1: sp.csc_matrix  # lower, diagonal first per column (CscLower layout)
    fill_perm: np.ndarray
    coupling: sp.csr_matrix
    sigma0: np.ndarray
    k22_beta: sp.csr_matrix
    tets_beta_local: np.ndarray

    @property
    def order(self):
        inv = np.empty(len(self.perm), dtype=np.int64)
        inv[self.perm] = np.arange(len(self.perm))
        return inv

    @property
    def x1_ids(self):
        return self.order[: self.n1]

    @property
    def x2_ids(self):
        return self.order[self.n1:]


@dataclass
class OState:
    """Reference SolverState (solver.py:116-145)."""

    x: np.ndarray
    R: np.ndarray
    Q: Optional[np.ndarray]
    active: np.ndarray
    target: np.ndarray
    f_tilde2: np.ndarray
    u2_accum: np.ndarray

    def copy(self):
        return OState(self.x.copy(), self.R.copy(), None if self.Q is None else self.Q.copy(),
                      self.active.copy(), self.target.copy(), self.f_tilde2.copy(), self.u2_accum.copy())


# ---------------------------------------------------------- system build


def element_scalar_stiffness(dmi, vol, mu, mu_prime):
    """material.py:381-390: 2 (mu + mu') vol B B^T."""
    B = np.empty((len(vol), 4, 3))
    B[:, 1:, :] = dmi
    B[:, 0, :] = -dmi.sum(axis=1)
    coef = 2.0 * (mu + mu_prime) * vol
    return coef[:, None, None] * np.einsum("eaj,ebj->eab", B, B)


def system_matrix(scene: OScene, perm: np.ndarray) -> sp.csr_matrix:
    """Full permuted scalar block A (material.py:393-399 + solver.py:257-264 + partition.py:67-71)."""
    n = scene.num_nodes
    ke = element_scalar_stiffness(scene.dm_inverse, scene.volume, scene.mu, scene.mu_prime)
    rows = np.repeat(scene.tets, 4, axis=1).ravel()
    cols = np.tile(scene.tets, (1, 4)).ravel()
    K = sp.coo_matrix((ke.ravel(), (rows, cols)), shape=(n, n)).tocsr()
    K.sum_duplicates()
    diag = np.zeros(n)
    np.add.at(diag, scene.att_nodes, scene.att_k)
    A = (K + sp.diags(diag)).tocsr()
    order = np.empty(n, dtype=np.int64)
    order[perm] = np.arange(n)
    return A[order][:, order].tocsr()


def dense_partial_factor(A: sp.spmatrix, n1: int):
    """linalg.py:329-382 with the identity fill ordering, evaluated densely
    (small systems only): L1 = chol(A11), C = A21 L1^-T, sigma0 = A22 - C C^T."""
    Ad = A.toarray()
    a11 = Ad[:n1, :n1]
    a21 = Ad[n1:, :n1]
    a22 = Ad[n1:, n1:]
    L1 = np.linalg.cholesky(a11) if n1 else np.zeros((0, 0))
    C = scipy.linalg.solve_triangular(L1, a21.T, lower=True).T if n1 else np.zeros((len(a22), 0))
    sigma0 = a22 - C @ C.T
    sigma0 = 0.5 * (sigma0 + sigma0.T)
    l1 = sp.csc_matrix(np.tril(L1))
    l1.sort_indices()
    return l1, np.arange(n1, dtype=np.int64), sp.csr_matrix(C), sigma0


def build_system(scene: OScene, perm, n1, e_alpha, e_beta) -> OSystem:
    """solver.py:246-296 restated (dense partial factor: small scenes)."""
    n2 = scene.num_nodes - n1
    A = system_matrix(scene, perm)
    l1, fperm, C, sigma0 = dense_partial_factor(A, n1)
    if len(e_beta):
        ke = element_scalar_stiffness(scene.dm_inverse, scene.volume, scene.mu, scene.mu_prime)[e_beta]
        tbl = perm[scene.tets[e_beta]] - n1
        k22 = sp.coo_matrix((ke.ravel(), (np.repeat(tbl, 4, axis=1).ravel(), np.tile(tbl, (1, 4)).ravel())),
                            shape=(n2, n2)).tocsr()
        k22.sum_duplicates()
    else:
        tbl = np.zeros((0, 4), dtype=np.int64)
        k22 = sp.csr_matrix((n2, n2))
    return OSystem(n1, n2, perm, e_alpha, e_beta, l1, fperm, C, sigma0, k22, tbl)


# ------------------------------------------------------------- collision


def proxy_positions(scene: OScene, x):
    """collision.py:303-309 (einsum)."""
    if len(scene.prox_elem) == 0:
        return np.zeros((0, 3))
    return np.einsum("ma,mad->md", scene.prox_w, x[scene.tets[scene.prox_elem]])


def _sd_local(c: OCollider, q):
    """Shape signed distances in the collider frame (collision.py:57-180)."""
    p = c.params
    if c.kind == "half_space":
        return (q - np.asarray(p["point"])) @ np.asarray(p["normal"])
    if c.kind == "sphere":
        return np.linalg.norm(q - np.asarray(p["center"]), axis=-1) - p["radius"]
    if c.kind == "capsule":
        return np.linalg.norm(q - _capsule_closest(p, q), axis=-1) - p["radius"]
    return _grid_sample(p, q)


def _capsule_closest(p, q):
    p0 = np.asarray(p["p0"], dtype=np.float64); p1 = np.asarray(p["p1"], dtype=np.float64)
    axis = p1 - p0
    denom = float(axis @ axis)
    if denom == 0.0:
        return np.broadcast_to(p0, q.shape).copy()
    t = np.clip(((q - p0) @ axis) / denom, 0.0, 1.0)
    return p0 + t[..., None] * axis


def _grid_sample(p, q):
    """collision.py:145-167 (values stored x-fastest, reshaped to [ix,iy,iz])."""
    nx, ny, nz = (int(v) for v in p["dims"])
    vals = np.asarray(p["values"], dtype=np.float64).reshape(nz, ny, nx).transpose(2, 1, 0)
    g = (q - np.asarray(p["origin"], dtype=np.float64)) / float(p["spacing"])
    out = np.full(q.shape[:-1], np.inf)
    inside = ((g[..., 0] >= 0) & (g[..., 0] <= nx - 1) & (g[..., 1] >= 0) & (g[..., 1] <= ny - 1)
              & (g[..., 2] >= 0) & (g[..., 2] <= nz - 1))
    if not inside.any():
        return out
    gi = g[inside]
    i0 = np.minimum(gi.astype(np.int64), np.array([nx, ny, nz]) - 2)
    fr = gi - i0
    ix, iy, iz = i0[..., 0], i0[..., 1], i0[..., 2]
    fx, fy, fz = fr[..., 0], fr[..., 1], fr[..., 2]
    c00 = vals[ix, iy, iz] * (1 - fx) + vals[ix + 1, iy, iz] * fx
    c10 = vals[ix, iy + 1, iz] * (1 - fx) + vals[ix + 1, iy + 1, iz] * fx
    c01 = vals[ix, iy, iz + 1] * (1 - fx) + vals[ix + 1, iy, iz + 1] * fx
    c11 = vals[ix, iy + 1, iz + 1] * (1 - fx) + vals[ix + 1, iy + 1, iz + 1] * fx
    out[inside] = (c00 * (1 - fy) + c10 * fy) * (1 - fz) + (c01 * (1 - fy) + c11 * fy) * fz
    return out


def _grad_local(c: OCollider, q):
    p = c.params
    if c.kind == "half_space":
        return np.broadcast_to(np.asarray(p["normal"], dtype=np.float64), q.shape).copy()
    if c.kind in ("sphere", "capsule"):
        d = q - (np.asarray(p["center"], dtype=np.float64) if c.kind == "sphere" else _capsule_closest(p, q))
        r = np.linalg.norm(d, axis=-1, keepdims=True)
        g = np.divide(d, r, out=np.zeros_like(d), where=r > 0)
        g[(r == 0)[..., 0]] = (1.0, 0.0, 0.0)
        return g
    h = 0.5 * float(p["spacing"])
    g = np.empty_like(q)
    for a in range(3):
        dp = np.zeros(3); dp[a] = h
        g[..., a] = (_grid_sample(p, q + dp) - _grid_sample(p, q - dp)) / (2 * h)
    g[~np.isfinite(g).all(axis=-1)] = 0.0
    return g


def _to_local(c: OCollider, pts):
    return (pts - c.translation) @ c.rotation  # collision.py:50-51


def signed_distance(c: OCollider, pts):
    return _sd_local(c, _to_local(c, pts))  # collision.py:193-194


def project(c: OCollider, pts):
    """collision.py:196-203."""
    q = _to_local(c, pts)
    phi = _sd_local(c, q)
    grad = _grad_local(c, q)
    phi = np.where(np.isfinite(phi), phi, 0.0)
    return pts - phi[..., None] * (grad @ c.rotation.T)


def detect(scene: OScene, x):
    """collision.py:316-342: deepest collider wins (strict <, first listed on ties)."""
    P = len(scene.prox_elem)
    active = np.zeros(P, dtype=bool)
    target = np.zeros((P, 3))
    if P == 0 or not scene.colliders:
        return active, target
    pts = proxy_positions(scene, x)
    best = np.full(P, np.inf)
    idx = np.full(P, -1)
    for ci, c in enumerate(scene.colliders):
        phi = signed_distance(c, pts)
        deeper = phi < best
        best = np.where(deeper, phi, best)
        idx = np.where(deeper, ci, idx)
    active[:] = best < 0.0
    for ci, c in enumerate(scene.colliders):
        sel = active & (idx == ci)
        if sel.any():
            target[sel] = project(c, pts[sel])
    return active, target


def penetration_depths(scene: OScene, x):
    """collision.py:345-359."""
    P = len(scene.prox_elem)
    if P == 0 or not scene.colliders:
        return np.zeros(P)
    pts = proxy_positions(scene, x)
    best = np.full(P, np.inf)
    for c in scene.colliders:
        best = np.minimum(best, signed_distance(c, pts))
    return np.where(np.isfinite(best), np.maximum(0.0, -best), 0.0)


def c22_dense(scene: OScene, sysm: OSystem, active):
    """collision.py:401-434 + ScalarSparseSym.full() (linalg.py:46-51, 67-74) as a dense m x m."""
    m = sysm.n2
    out = sp.csr_matrix((m, m))
    if len(scene.prox_elem) == 0 or not active.any():
        return out
    local = sysm.perm[scene.tets[scene.prox_elem]] - sysm.n1
    W = scene.prox_w[active]
    c = scene.prox_c[active]
    loc = local[active]
    blocks = c[:, None, None] * (W[:, :, None] * W[:, None, :])
    rows = np.repeat(loc, 4, axis=1).ravel()
    cols = np.tile(loc, (1, 4)).ravel()
    full = sp.coo_matrix((blocks.ravel(), (rows, cols)), shape=(m, m)).tocsc()
    full.sum_duplicates()
    upper = sp.triu(full, format="csc")
    upper.sum_duplicates(); upper.sort_indices()
    d = sp.diags(upper.diagonal())
    f = (upper + upper.T - d).tocsr()
    f.sort_indices()
    return f


def collision_energy(scene: OScene, x, active, target):
    """collision.py:362-374."""
    if len(scene.prox_elem) == 0 or not active.any():
        return 0.0
    d = proxy_positions(scene, x) - target
    return float(0.5 * np.sum(scene.prox_c * active * np.einsum("md,md->m", d, d)))


def collision_forces(scene: OScene, x, active, target, out):
    """collision.py:377-398."""
    if len(scene.prox_elem) == 0 or not active.any():
        return out
    pts = proxy_positions(scene, x)
    for j in range(len(scene.prox_elem)):
        if not active[j]:
            continue
        f = -scene.prox_c[j] * (pts[j] - target[j])
        nodes = scene.tets[scene.prox_elem[j]]
        for a in range(4):
            out[nodes[a]] += scene.prox_w[j, a] * f
    return out


# --------------------------------------------------------- forces, energy


def local_step(scene: OScene, x, elements, state: OState):
    """solver.py:161-184."""
    if elements is not None and len(elements) == 0:
        return
    tets = scene.tets if elements is None else scene.tets[elements]
    dmi = scene.dm_inverse if elements is None else scene.dm_inverse[elements]
    F = deformation_gradients(x, tets, dmi)
    sel = slice(None) if elements is None else elements
    state.R[sel] = polar_rotations(F)
    if scene.biphasic:
        state.Q[sel] = biphasic_projections(F, scene.sigma_min, scene.sigma_max)


def elastic_forces(scene: OScene, x, state: OState, elements):
    """material.py:328-357 (element-order np.add.at accumulation)."""
    out = np.zeros((scene.num_nodes, 3))
    tets = scene.tets if elements is None else scene.tets[elements]
    if len(tets) == 0:
        return out
    sel = slice(None) if elements is None else elements
    F = deformation_gradients(x, tets, scene.dm_inverse[sel])
    P = 2.0 * scene.mu * (F - state.R[sel])
    if state.Q is not None and scene.biphasic:
        P += 2.0 * scene.mu_prime * (F - state.Q[sel])
    G = -scene.volume[sel][:, None, None] * (P @ np.swapaxes(scene.dm_inverse[sel], 1, 2))
    np.add.at(out, tets[:, 0], -G.sum(axis=2))
    for a in range(3):
        np.add.at(out, tets[:, a + 1], G[:, :, a])
    return out


def attachment_forces(scene: OScene, x, out):
    """solver.py:187-190 (list order)."""
    for k in range(len(scene.att_nodes)):
        i = scene.att_nodes[k]
        out[i] += scene.att_k[k] * (scene.att_targets[k] - x[i])
    return out


def elastic_energy(scene: OScene, x, state: OState):
    """material.py:360-378."""
    F = deformation_gradients(x, scene.tets, scene.dm_inverse)
    d = F - state.R
    dens = scene.mu * np.einsum("eij,eij->e", d, d)
    if state.Q is not None and scene.biphasic:
        dq = F - state.Q
        dens = dens + scene.mu_prime * np.einsum("eij,eij->e", dq, dq)
    return float(np.dot(scene.volume, dens))


def attachment_energy(scene: OScene, x):
    """solver.py:193-198."""
    e = 0.0
    for k in range(len(scene.att_nodes)):
        d = x[scene.att_nodes[k]] - scene.att_targets[k]
        e += 0.5 * scene.att_k[k] * float(d @ d)
    return e


def total_energy(scene: OScene, x, state: OState):
    """solver.py:216-231."""
    return (elastic_energy(scene, x, state) + attachment_energy(scene, x)
            + collision_energy(scene, x, state.active, state.target))


# ----------------------------------------------------------- substitutions


def forward_sub(sysm: OSystem, b1, b2):
    """linalg.py:385-398 (3 columns; _lsolve per column)."""
    l1 = sysm.l1
    y1 = np.ascontiguousarray(b1[sysm.fill_perm], dtype=np.float64)
    if sysm.n1:
        lib().or_lsolve3(sysm.n1, _p(l1.indptr.astype(np.int64)), _p(l1.indices.astype(np.int64)),
                         _p(np.ascontiguousarray(l1.data)), _p(y1))
    return y1, b2 - sysm.coupling @ y1


def backward_sub(sysm: OSystem, y1, x2):
    """linalg.py:401-414."""
    rhs = np.ascontiguousarray(y1 - sysm.coupling.T @ x2)
    l1 = sysm.l1
    if sysm.n1:
        lib().or_ltsolve3(sysm.n1, _p(l1.indptr.astype(np.int64)), _p(l1.indices.astype(np.int64)),
                          _p(np.ascontiguousarray(l1.data)), _p(rhs))
    x1 = np.empty_like(rhs)
    x1[sysm.fill_perm] = rhs
    return x1


def dense_factor(h):
    """linalg.py:432-440 (LAPACK dpotrf, lower)."""
    return scipy.linalg.cholesky(h, lower=True, check_finite=False)


def dense_solve(chol, g):
    """linalg.py:452-461 (two dtrtrs)."""
    y = scipy.linalg.solve_triangular(chol, g, lower=True, check_finite=False)
    return scipy.linalg.solve_triangular(chol, y, lower=True, trans="T", check_finite=False)


# -------------------------------------------------------------- the frame


def _beta_forces_local(scene, sysm, state):
    """solver.py:327-346."""
    out = np.zeros((sysm.n2, 3))
    eb = sysm.e_beta
    if len(eb) == 0:
        return out
    F = deformation_gradients(state.x, scene.tets[eb], scene.dm_inverse[eb])
    P = 2.0 * scene.mu * (F - state.R[eb])
    if scene.biphasic:
        P += 2.0 * scene.mu_prime * (F - state.Q[eb])
    G = -scene.volume[eb][:, None, None] * (P @ np.swapaxes(scene.dm_inverse[eb], 1, 2))
    tl = sysm.tets_beta_local
    np.add.at(out, tl[:, 0], -G.sum(axis=2))
    for a in range(3):
        np.add.at(out, tl[:, a + 1], G[:, :, a])
    return out


def _collision_forces_local(scene, sysm, state):
    """solver.py:349-364."""
    out = np.zeros((sysm.n2, 3))
    act = state.active
    if len(scene.prox_elem) == 0 or not act.any():
        return out
    nodes = scene.tets[scene.prox_elem]
    local = sysm.perm[nodes] - sysm.n1
    W = scene.prox_w
    pj = np.einsum("pa,pad->pd", W, state.x[nodes])
    coef = np.where(act, scene.prox_c, 0.0)
    f = -coef[:, None] * (pj - state.target)
    for a in range(4):
        np.add.at(out, local[:, a], W[:, a, None] * f)
    return out


@dataclass
class OMetrics:
    energy: float = 0.0
    active_proxies: int = 0
    max_penetration: float = 0.0
    residual: float = 0.0
    t_total_ms: float = 0.0


def solve_frame_schur(scene: OScene, sysm: OSystem, state: OState, outer_iters=1, inner_iters=1,
                      cadence="inner") -> OMetrics:
    """solver.py:387-455, with _finish_metrics (solver.py:373-384)."""
    t_frame = time.perf_counter()
    x1_ids, x2_ids = sysm.x1_ids, sysm.x2_ids
    first_detection_done = False
    residual = 0.0
    for _ in range(outer_iters):
        local_step(scene, state.x, sysm.e_alpha, state)
        f = elastic_forces(scene, state.x, state, sysm.e_alpha)
        attachment_forces(scene, state.x, f)
        y1, state.f_tilde2 = forward_sub(sysm, f[x1_ids], f[x2_ids])
        state.u2_accum = np.zeros_like(state.f_tilde2)
        for _ in range(inner_iters):
            fresh = cadence == "inner" or (cadence == "frame" and not first_detection_done)
            if fresh:
                state.active, state.target = detect(scene, state.x)
            first_detection_done = True
            local_step(scene, state.x, sysm.e_beta, state)
            c22 = c22_dense(scene, sysm, state.active)
            h = sysm.sigma0 + c22.toarray()
            chol = dense_factor(h) if sysm.n2 else h
            g = state.f_tilde2 + _beta_forces_local(scene, sysm, state)
            g += _collision_forces_local(scene, sysm, state)
            u2 = dense_solve(chol, g) if sysm.n2 else np.zeros_like(g)
            state.x[x2_ids] += u2
            state.f_tilde2 -= sysm.sigma0 @ u2 - sysm.k22_beta @ u2
            state.u2_accum += u2
            residual = float(np.linalg.norm(h @ u2 - g) / max(np.linalg.norm(g), np.finfo(float).tiny))
        u1 = backward_sub(sysm, y1, state.u2_accum)
        state.x[x1_ids] += u1
    met = OMetrics(residual=residual)
    met.active_proxies = int(state.active.sum())
    met.energy = total_energy(scene, state.x, state)
    met.max_penetration = float(np.max(penetration_depths(scene, state.x), initial=0.0))
    met.t_total_ms = 1e3 * (time.perf_counter() - t_frame)
    return met


def num_threads() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
