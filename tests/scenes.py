"""Scene builders shared by the tests and bench.py, plus converters to the
oracle's plain-array data model (oracle/oracle.py)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import paper_2008_01541_b200 as P  # noqa: E402
from paper_2008_01541_b200 import collision as col  # noqa: E402
from paper_2008_01541_b200 import solver as sol  # noqa: E402

GOLDEN = Path(__file__).resolve().parent / "golden"

from scene_yaml import CONFIGS, block_yaml  # noqa: E402,F401


def make_bar(cells=(6, 2, 2), extent=(1.5, 0.4, 0.4), press_depth=0.05, biphasic=False):
    """The reference test fixture (test_solver.py:16-32) with the product API."""
    mesh = P.build_box_lattice(extent, cells)
    rest = P.compute_rest_data(mesh)
    params = P.MaterialParams(mu=1e4, mu_prime=5e3 if biphasic else 0.0, sigma_min=0.7, sigma_max=1.3)
    left = np.flatnonzero(mesh.rest_positions[:, 0] < 1e-9)
    atts = [sol.Attachment(int(i), mesh.rest_positions[i], 1e6) for i in left]
    stiff = sol.default_collision_stiffness(mesh, params)
    prox = col.scatter_proxies(mesh, lambda p: p[:, 0] > extent[0] - 1e-9, per_element=1, stiffness=stiff)
    part = P.classify(mesh, prox)
    system = sol.build_system(mesh, rest, params, atts, part)
    wall = col.Collider(col.HalfSpace((extent[0] - press_depth, 0, 0), (-1.0, 0, 0)))
    model = sol.Model(mesh, rest, params, atts, prox, [wall])
    state = sol.SolverState.at_rest(mesh, params, len(prox), part.n2)
    return model, system, state, part


def config_yaml(name: str, **kw) -> str:
    if name == "cfg1":
        return str(np.load(GOLDEN / "cfg1.npz")["yaml"])
    return block_yaml(*CONFIGS[name], **kw)


# ------------------------------------------------------------ oracle views


def oracle_colliders(model):
    from oracle.oracle import OCollider

    out = []
    for c in model.colliders:
        s = c.shape
        if isinstance(s, col.HalfSpace):
            prm = {"point": s.point, "normal": s.normal}
        elif isinstance(s, col.Sphere):
            prm = {"center": s.center, "radius": s.radius}
        elif isinstance(s, col.Capsule):
            prm = {"p0": s.p0, "p1": s.p1, "radius": s.radius}
        else:
            prm = {"origin": s.origin, "spacing": s.spacing, "dims": s.dims, "values": s.flat_values}
        out.append(OCollider(s.KIND, prm, np.array(c.transform.rotation, dtype=float),
                             np.array(c.transform.translation, dtype=float)))
    return out


def oracle_scene(model):
    from oracle.oracle import OScene

    p = model.params
    return OScene(
        tets=model.mesh.tets, dm_inverse=model.rest.dm_inverse, volume=model.rest.volume, mu=p.mu,
        mu_prime=p.mu_prime, sigma_min=p.sigma_min, sigma_max=p.sigma_max,
        att_nodes=np.array([a.node for a in model.attachments], dtype=np.int64),
        att_k=np.array([a.stiffness for a in model.attachments]),
        att_targets=np.array([a.target for a in model.attachments]).reshape(-1, 3),
        prox_elem=model.proxy_elements, prox_w=model.proxy_weights.reshape(-1, 4), prox_c=model.proxy_stiffness,
        colliders=oracle_colliders(model), num_nodes=model.mesh.num_nodes,
    )


def oracle_system(model, system, use_product_factor=False):
    """OSystem with the oracle's own dense partial factor (small scenes), or
    with the product's exported L1 / C / sigma0 (large scenes)."""
    from oracle import oracle as O

    part = system.partition
    if not use_product_factor:
        return O.build_system(oracle_scene(model), part.perm, part.n1, part.e_alpha, part.e_beta)
    f = system.factor
    l1 = f.l1.to_scipy()
    return O.OSystem(part.n1, part.n2, part.perm, part.e_alpha, part.e_beta, l1, f.fill_perm, f.coupling,
                     f.sigma0, system.k22_beta, system.tets_beta_local)


def oracle_state(state):
    from oracle.oracle import OState

    q = state.rotations.q
    return OState(state.x.copy(), state.rotations.r.copy(), None if q is None else q.copy(),
                  state.active.active.copy(), state.active.target.copy(), state.f_tilde2.copy(),
                  state.u2_accum.copy())


def state_from_golden(g, prefix, state_like):
    """Overwrite a product SolverState with a golden (reference) state."""
    st = state_like.copy()
    st.x[...] = g[prefix + "x"]
    st.active = col.ActiveSet(g[prefix + "active"].copy(), g[prefix + "target"].copy())
    st.f_tilde2 = g[prefix + "f_tilde2"].copy()
    st.u2_accum = g[prefix + "u2_accum"].copy()
    if prefix + "R" in g:
        st.rotations.r[...] = g[prefix + "R"]
    if prefix + "Q" in g and st.rotations.q is not None:
        st.rotations.q[...] = g[prefix + "Q"]
    return st


def step_rel(x_new, x_ref, x_pre):
    """Step-relative difference (harness.py:747-752)."""
    return float(np.linalg.norm(x_new - x_ref) / max(np.linalg.norm(x_ref - x_pre), np.finfo(float).tiny))
