"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
`schurpd` package (read-only at /root/reference/pkg/src) in this container.

This script is the only place that imports the reference; it is run by hand
(never by the tests, never on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Fixtures (all small, np.savez_compressed):
  svd.npz        signed SVD / polar / bi-phasic projections on adversarial F
                 (material.py:116-290)
  detect.npz     detection against every collider kind under rigid transforms
                 (collision.py:57-203, 316-359)
  bar_*.npz      the reference test fixture `make_scene` (test_solver.py:16-32),
                 frame-by-frame pre/post SolverState for several (outer, inner,
                 cadence, biphasic) configurations (solver.py:387-455)
  cfg1.npz       BASELINE config 1 (beam 20x8x8, proxies on x in [0.7,1.3] of the
                 top face), 50 frames through Simulation.step()
  bar_pcg.npz    the PCG baseline (solver.py:542-603) on the bar fixture:
                 pre/post states and iteration counts
  hinge.npz      built-in hinge_fold scene (capsule collider, rotating
                 attachments, outer=2 inner=2), 24 frames
  setup hashes   sha256 of every setup array, so the product's own host-side
                 setup is pinned bit-for-bit without storing the arrays
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)

from schurpd import collision as col  # noqa: E402
from schurpd import harness  # noqa: E402
from schurpd import solver as sol  # noqa: E402
from schurpd.material import (  # noqa: E402
    MaterialParams,
    biphasic_projections,
    polar_rotations,
    signed_svd,
)
from schurpd.mesh import build_box_lattice, compute_rest_data  # noqa: E402
from schurpd.partition import classify  # noqa: E402


def h(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode()).hexdigest()


# ----------------------------------------------------------------------- svd


def gen_svd():
    rng = np.random.default_rng(7)
    F = [rng.normal(size=(600, 3, 3))]
    F.append(np.eye(3)[None] + 0.05 * rng.normal(size=(200, 3, 3)))  # near-rest
    inv = rng.normal(size=(100, 3, 3))
    inv[np.linalg.det(inv) > 0, 0] *= -1.0  # inverted
    F.append(inv)
    F.append(np.array([np.zeros((3, 3)), np.eye(3), np.diag([2.0, 1.0, 0.5]),
                       np.diag([1.0, 1.0, -1.0]), np.diag([3.0, 0.0, 0.0]),
                       np.diag([1e-200, 1e-200, 1e-200]), np.diag([1e6, 1e-6, 1.0])]))
    u = rng.normal(size=(50, 3)); v = rng.normal(size=(50, 3))
    F.append(np.einsum("ni,nj->nij", u, v))  # rank 1
    a = rng.normal(size=(50, 3, 2)); b = rng.normal(size=(50, 2, 3))
    F.append(a @ b)  # rank 2
    scale = 10.0 ** rng.uniform(-6, 6, size=(100, 1, 1))
    F.append(scale * rng.normal(size=(100, 3, 3)))
    F = np.concatenate(F).astype(np.float64)
    R = polar_rotations(F)
    params = MaterialParams(mu=1.0, mu_prime=1.0, sigma_min=0.7, sigma_max=1.3)
    Q = biphasic_projections(F, params)
    U = np.empty_like(F); S = np.empty((len(F), 3)); V = np.empty_like(F)
    for k in range(len(F)):
        U[k], S[k], V[k] = signed_svd(F[k])
    np.savez_compressed(OUT / "svd.npz", F=F, R=R, Q=Q, U=U, S=S, V=V,
                        sigma_min=0.7, sigma_max=1.3)
    print("svd", F.shape)


# -------------------------------------------------------------------- detect


def _rot(rng):
    q = rng.normal(size=4); q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def _small_rot(rng, deg=6.0):
    k = rng.normal(size=3); k /= np.linalg.norm(k)
    a = np.radians(deg)
    K = np.array([[0.0, -k[2], k[1]], [k[2], 0.0, -k[0]], [-k[1], k[0], 0.0]])
    return np.eye(3) + np.sin(a) * K + (1 - np.cos(a)) * (K @ K)


def gen_detect():
    """One small lattice, proxies on its whole surface, displaced positions,
    and collider sets of every kind; records flags, targets, depths."""
    rng = np.random.default_rng(3)
    mesh = build_box_lattice((1.0, 0.6, 0.4), (10, 6, 4))
    prox = col.scatter_proxies(mesh, lambda p: np.ones(len(p), bool), per_element=3, stiffness=5.0)
    x = mesh.rest_positions + 0.03 * rng.normal(size=mesh.rest_positions.shape)
    # level set: signed distance of a sphere sampled on a grid
    nx, ny, nz = 12, 9, 7
    sp_ = 0.1
    origin = np.array([-0.05, -0.1, -0.15])
    gi = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1)
    pts = origin + sp_ * gi
    vals = np.linalg.norm(pts - np.array([0.5, 0.3, 0.35]), axis=-1) - 0.3
    flat = vals.transpose(2, 1, 0).ravel()  # x-fastest
    sets = {
        "halfspace": [col.Collider(col.HalfSpace((0.0, 0.0, 0.3), (0.0, 0.0, -1.0)))],
        "halfspace_rot": [col.Collider(col.HalfSpace((0.1, 0.2, 0.25), (0.0, 0.6, -0.8)),
                                       col.RigidTransform(_small_rot(rng, 20.0), rng.normal(size=3) * 0.05))],
        "sphere": [col.Collider(col.Sphere((0.5, 0.3, 0.55), 0.25),
                                col.RigidTransform(_small_rot(rng), np.array([0.02, -0.01, 0.0])))],
        "capsule": [col.Collider(col.Capsule((0.2, -0.2, 0.45), (0.8, 0.8, 0.45), 0.12),
                                 col.RigidTransform(_small_rot(rng), np.array([0.0, 0.03, -0.02])))],
        "capsule_degenerate": [col.Collider(col.Capsule((0.5, 0.3, 0.45), (0.5, 0.3, 0.45), 0.2))],
        "levelset": [col.Collider(col.GridLevelset(origin, sp_, (nx, ny, nz), flat))],
        "levelset_rot": [col.Collider(col.GridLevelset(origin, sp_, (nx, ny, nz), flat),
                                      col.RigidTransform(_small_rot(rng), np.array([0.01, 0.0, 0.02])))],
        "multi": [col.Collider(col.HalfSpace((0.0, 0.0, 0.35), (0.0, 0.0, -1.0))),
                  col.Collider(col.Sphere((0.3, 0.3, 0.5), 0.2)),
                  col.Collider(col.Capsule((0.7, -0.2, 0.45), (0.7, 0.8, 0.45), 0.1),
                               col.RigidTransform(_small_rot(rng), np.zeros(3))),
                  col.Collider(col.GridLevelset(origin, sp_, (nx, ny, nz), flat))],
    }
    out = {"x": x, "ls_origin": origin, "ls_spacing": sp_, "ls_dims": np.array([nx, ny, nz]),
           "ls_values": flat, "prox_elem": np.array([p.element for p in prox]),
           "prox_w": np.array([p.weights for p in prox]), "tets": mesh.tets}
    for name, cols in sets.items():
        a = col.detect(prox, mesh, x, cols)
        pen = col.penetration_depths(prox, mesh, x, cols)
        out[f"{name}__active"] = a.active
        out[f"{name}__target"] = a.target
        out[f"{name}__pen"] = pen
        out[f"{name}__desc"] = json.dumps(_describe(cols))
    np.savez_compressed(OUT / "detect.npz", **out)
    print("detect", len(prox), "proxies")


def _describe(cols):
    d = []
    for c in cols:
        s = c.shape
        tf = c.transform
        if isinstance(s, col.HalfSpace):
            d.append(("half_space", s.point.tolist() + s.normal.tolist(), tf.rotation.tolist(), tf.translation.tolist()))
        elif isinstance(s, col.Sphere):
            d.append(("sphere", s.center.tolist() + [s.radius], tf.rotation.tolist(), tf.translation.tolist()))
        elif isinstance(s, col.Capsule):
            d.append(("capsule", s.p0.tolist() + s.p1.tolist() + [s.radius], tf.rotation.tolist(), tf.translation.tolist()))
        else:
            d.append(("levelset", [], tf.rotation.tolist(), tf.translation.tolist()))
    return d


# ------------------------------------------------------------- bar fixture


def make_scene(cells=(6, 2, 2), extent=(1.5, 0.4, 0.4), press_depth=0.05, biphasic=False):
    """Same construction as the reference fixture (test_solver.py:16-32)."""
    mesh = build_box_lattice(extent, cells)
    rest = compute_rest_data(mesh)
    params = MaterialParams(mu=1e4, mu_prime=5e3 if biphasic else 0.0, sigma_min=0.7, sigma_max=1.3)
    left = np.flatnonzero(mesh.rest_positions[:, 0] < 1e-9)
    atts = [sol.Attachment(int(i), mesh.rest_positions[i], 1e6) for i in left]
    stiff = sol.default_collision_stiffness(mesh, params)
    prox = col.scatter_proxies(mesh, lambda p: p[:, 0] > extent[0] - 1e-9, per_element=1, stiffness=stiff)
    part = classify(mesh, prox)
    system = sol.build_system(mesh, rest, params, atts, part)
    wall = col.Collider(col.HalfSpace((extent[0] - press_depth, 0, 0), (-1.0, 0, 0)))
    model = sol.Model(mesh, rest, params, atts, prox, [wall])
    state = sol.SolverState.at_rest(mesh, params, len(prox), part.n2)
    return model, system, state, part


def _state_dict(prefix, st, rotations=True):
    d = {f"{prefix}x": st.x.copy(),
         f"{prefix}active": st.active.active.copy(), f"{prefix}target": st.active.target.copy(),
         f"{prefix}f_tilde2": st.f_tilde2.copy(), f"{prefix}u2_accum": st.u2_accum.copy()}
    if rotations:
        d[f"{prefix}R"] = st.rotations.r.copy()
        if st.rotations.q is not None:
            d[f"{prefix}Q"] = st.rotations.q.copy()
    return d


def _metrics_vec(m):
    return np.array([m.energy, m.active_proxies, m.max_penetration, m.residual])


def gen_bar(name, biphasic, outer, inner, cadence, frames, press_depth=0.08, jitter=0.0):
    model, system, state, part = make_scene(press_depth=press_depth, biphasic=biphasic)
    if jitter:
        state.x += jitter * np.random.default_rng(1).normal(size=state.x.shape)
    cfg = sol.SolverConfig(outer_iters=outer, inner_iters=inner, detection_cadence=cadence)
    out = {"outer": outer, "inner": inner, "cadence": cadence, "biphasic": biphasic,
           "press_depth": press_depth, "frames": frames}
    out["sigma0"] = system.factor.sigma0
    out["perm"] = part.perm
    out["x0"] = state.x.copy()
    for f in range(frames):
        pre = state.copy()
        met = sol.solve_frame_schur(model, system, state, cfg)
        out.update(_state_dict(f"pre{f}_", pre))
        out.update(_state_dict(f"post{f}_", state))
        out[f"metrics{f}"] = _metrics_vec(met)
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(name, "m =", part.n2, "active", state.active.count)


def gen_bar_pcg(name, outer, inner, cadence, frames, press_depth=0.08, tol=1e-10):
    """The PCG baseline (solver.py:542-603) on the same bar: pre/post states
    and the worst per-pass iteration count of every frame."""
    model, system, state, part = make_scene(press_depth=press_depth)
    cfg = sol.SolverConfig(outer_iters=outer, inner_iters=inner, detection_cadence=cadence, solver_kind="pcg",
                           pcg_tol=tol)
    out = {"outer": outer, "inner": inner, "cadence": cadence, "press_depth": press_depth, "frames": frames,
           "tol": tol}
    for f in range(frames):
        pre = state.copy()
        met = sol.solve_frame_pcg(model, system, state, cfg)
        out.update(_state_dict(f"pre{f}_", pre, rotations=False))
        out.update(_state_dict(f"post{f}_", state, rotations=False))
        out[f"metrics{f}"] = _metrics_vec(met)
        out[f"iters{f}"] = met.pcg_iterations
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(name, "m =", part.n2, "iters", [int(out[f"iters{f}"]) for f in range(frames)])


# ----------------------------------------------------------------- scenes


CFG1 = """
name: cfg1_beam5pct
mesh: {lattice: {extent: [2.0, 0.8, 0.8], cells: [20, 8, 8]}}
material: {mu: 1.0e+4}
attachments:
  - name: base
    region: {box: {min: [-0.01, -0.01, -0.01], max: [2.01, 0.81, 0.005]}}
    stiffness: 1.0e+7
    motion: {kind: fixed}
proxies:
  region: {box: {min: [0.699, -0.01, 0.795], max: [1.301, 0.81, 0.81]}}
  per_element: 1
  stiffness: auto
colliders:
  - shape: {half_space: {point: [0.0, 0.0, 0.9], normal: [0.0, 0.0, -1.0]}}
    motion: {kind: translate, velocity: [0.0, 0.0, -0.004], stop_frame: 50}
solver: {kind: schur, outer_iters: 1, inner_iters: 1}
frames: 50
"""


def _setup_hashes(sim, prefix=""):
    m = sim.model
    return {
        f"{prefix}hash_rest_positions": h(sim.mesh.rest_positions),
        f"{prefix}hash_tets": h(sim.mesh.tets),
        f"{prefix}hash_surface_tris": h(sim.mesh.surface_tris),
        f"{prefix}hash_dm_inverse": h(sim.rest.dm_inverse),
        f"{prefix}hash_volume": h(sim.rest.volume),
        f"{prefix}hash_perm": h(sim.partition.perm),
        f"{prefix}hash_e_beta": h(sim.partition.e_beta),
        f"{prefix}hash_prox_elem": h(m.proxy_elements),
        f"{prefix}hash_prox_w": h(m.proxy_weights),
        f"{prefix}hash_prox_c": h(m.proxy_stiffness),
        f"{prefix}hash_att_nodes": h(np.array([a.node for a in m.attachments])),
    }


def gen_scene(name, text, frames, every=1):
    sc = harness.parse_scenario(text)
    sim = harness.Simulation(sc)
    out = {"yaml": text, "frames": frames, "n1": sim.partition.n1, "n2": sim.partition.n2}
    out.update(_setup_hashes(sim))
    out["sigma0_diag"] = np.diag(sim.system.factor.sigma0).copy()
    out["sigma0_rowsum"] = sim.system.factor.sigma0.sum(axis=1)
    for f in range(1, frames + 1):
        pre = sim.state.copy()
        met = sim.step()
        if f % every == 0:
            # R/Q at frame entry never reach the solve (alpha is re-projected
            # first, beta before each use: solver.py:403, :426)
            out.update(_state_dict(f"pre{f}_", pre, rotations=False))
            out.update(_state_dict(f"post{f}_", sim.state, rotations=False))
        out[f"metrics{f}"] = _metrics_vec(met)
        out[f"active{f}"] = sim.state.active.active.copy()
    out["final_x"] = sim.state.x.copy()
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(name, "n =", sim.mesh.num_nodes, "m =", sim.partition.n2, "P =", len(sim.model.proxies),
          "active", sim.state.active.count)


def gen_partial_factor():
    """Σ0 of a small permuted matrix (sigma0 is ordering independent)."""
    sc = harness.parse_scenario(CFG1)
    sim = harness.Simulation(sc)
    np.savez_compressed(OUT / "cfg1_sigma0.npz", sigma0=sim.system.factor.sigma0)


if __name__ == "__main__":
    if sys.argv[1:] == ["pcg"]:  # only the PCG-baseline fixture
        gen_bar_pcg("bar_pcg", 1, 2, "inner", 3)
        sys.exit(0)
    gen_svd()
    gen_detect()
    gen_bar("bar_plain", False, 1, 1, "inner", 5)
    gen_bar("bar_multi", False, 2, 3, "inner", 4)
    gen_bar("bar_biphasic", True, 1, 2, "frame", 4)
    gen_bar("bar_never", False, 1, 2, "never", 3, jitter=0.01)
    gen_scene("cfg1", CFG1, 50, every=10)
    hinge = harness.builtin_scene_path("hinge_fold").read_text()
    gen_scene("hinge", hinge, 24, every=6)
    gen_partial_factor()
    gen_bar_pcg("bar_pcg", 1, 2, "inner", 3)
