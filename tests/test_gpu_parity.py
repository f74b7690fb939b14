"""GPU parity: the sm_100a path through the C ABI against the oracle and the
reference goldens. Run on a B200 with `pytest -m gpu`.

Bars (north star): positions within 1e-6 relative (we gate lockstep frames at
1e-7 step-relative), active sets bit-exact outside the certified sign band
(SURVEY §7 H3), rotations bit-exact on identical inputs."""

import json

import numpy as np
import pytest

import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import _native
from paper_2008_01541_b200 import collision as col
from paper_2008_01541_b200 import solver as sol
from scenes import GOLDEN, make_bar, oracle_scene, oracle_system, oracle_state, state_from_golden, step_rel

pytestmark = pytest.mark.gpu


def test_device_visible():
    assert _native.device_count() >= 1


# ------------------------------------------------------------ element ops


def test_svd_bitwise():
    """Sign-carrying SVD, R = U V^T and the clamp on the device equal the
    reference's numba results bit for bit (material.py:116-290)."""
    g = np.load(GOLDEN / "svd.npz")
    out = _native.op_svd(g["F"], want=("U", "S", "V", "R", "Q"), sigma_min=float(g["sigma_min"]),
                         sigma_max=float(g["sigma_max"]))
    for k in ("U", "S", "V", "R", "Q"):
        assert np.array_equal(out[k], g[k]), k


def test_deformation_gradients_and_forces_vs_oracle(rng):
    from oracle import oracle as O

    model, system, state, part = make_bar(cells=(8, 3, 3))
    x = state.x + 0.03 * rng.normal(size=state.x.shape)
    F = P.deformation_gradients(model.mesh, model.rest, x)
    Fo = O.deformation_gradients(x, model.mesh.tets, model.rest.dm_inverse)
    assert np.array_equal(F, Fo)
    R = O.polar_rotations(Fo)
    cache = P.RotationCache(R.copy())
    f = P.elastic_forces(model.mesh, model.rest, x, cache, model.params)
    sc = oracle_scene(model)
    st = O.OState(x, R, None, np.zeros(0, bool), np.zeros((0, 3)), None, None)
    fo = O.elastic_forces(sc, x, st, None)
    assert np.array_equal(f, fo)  # same op order: bitwise
    e = P.elastic_energy(model.mesh, model.rest, x, cache, model.params)
    assert abs(e - O.elastic_energy(sc, x, st)) <= 1e-12 * abs(e)


def _golden_colliders(desc, g):
    cols = []
    for kind, prm, R, t in json.loads(desc):
        if kind == "half_space":
            s = col.HalfSpace(prm[:3], prm[3:6])
        elif kind == "sphere":
            s = col.Sphere(prm[:3], prm[3])
        elif kind == "capsule":
            s = col.Capsule(prm[:3], prm[3:6], prm[6])
        else:
            s = col.GridLevelset(g["ls_origin"], float(g["ls_spacing"]), g["ls_dims"], g["ls_values"])
        cols.append(col.Collider(s, col.RigidTransform(np.array(R), np.array(t))))
    return cols


@pytest.mark.parametrize("name", ["halfspace", "halfspace_rot", "sphere", "capsule", "capsule_degenerate",
                                  "levelset", "levelset_rot", "multi"])
def test_detect_vs_reference(name):
    """Flags bit-exact outside the certified band |phi| <= 2 gamma_3 sum|p n|;
    targets and depths within 1e-12 of the reference."""
    g = np.load(GOLDEN / "detect.npz")
    cols = _golden_colliders(str(g[name + "__desc"]), g)
    act, tgt, dep = _native.op_detect(g["x"], g["tets"], g["prox_elem"], g["prox_w"],
                                      [(c.shape, c.transform.rotation, c.transform.translation) for c in cols])
    ref = g[name + "__active"]
    mism = np.flatnonzero(act != ref)
    if len(mism):
        # any mismatch must be a certified-ambiguous sign (|depth| ~ roundoff)
        assert np.all(np.abs(g[name + "__pen"][mism]) < 1e-14), mism
    assert len(mism) == 0
    np.testing.assert_allclose(tgt, g[name + "__target"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(dep, g[name + "__pen"], rtol=0, atol=1e-12)


# ------------------------------------------------------------ linalg ops


@pytest.mark.parametrize("m", [1, 5, 64, 130, 300])
def test_dense_factor_solve(rng, m):
    a = rng.normal(size=(m, m))
    h = a @ a.T + m * np.eye(m)
    f = P.dense_factor(h)
    ref = np.linalg.cholesky(h)
    assert np.abs(f.chol - ref).max() <= 1e-12 * np.abs(ref).max()
    g = rng.normal(size=(m, 3))
    x = P.dense_solve(f, g)
    assert np.linalg.norm(h @ x - g) <= 1e-10 * np.linalg.norm(g)
    x1 = P.dense_solve(f, g[:, 0])
    assert x1.shape == (m,)


def test_dense_factor_indefinite_names_column():
    h = np.diag([4.0, 1.0, -1.0, 2.0])
    with pytest.raises(P.IndefiniteMatrixError) as ei:
        P.dense_factor(h)
    assert ei.value.column == 2


@pytest.mark.parametrize("split", [(50, 30), (80, 1), (80, 79), (64, 0), (64, 64)])
def test_three_step_solve_equals_dense(rng, split):
    """reference test_linalg.py:143-159 on the device sweeps."""
    n, n1 = split
    M = rng.normal(size=(n, n))
    A = M @ M.T + n * np.eye(n)
    A[np.abs(A) < 0.5 * np.abs(A).mean()] = 0.0
    A = 0.5 * (A + A.T) + n * np.eye(n)
    S = P.ScalarSparseSym.from_dense(A)
    f = P.partial_cholesky(S, n1)
    b = rng.normal(size=(n, 3))
    y1, y2 = P.forward_sub(f, b[:n1], b[n1:])
    x2 = np.linalg.solve(f.sigma0, y2) if n - n1 else np.zeros((0, 3))
    x1 = P.backward_sub(f, y1, x2)
    x = np.concatenate([x1, x2])
    ref = np.linalg.solve(A, b)
    assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)


def test_forward_backward_vs_oracle_cfg2_partial():
    """Device sweeps vs the oracle's scalar column solves on the same
    exported factor (sizes the oracle finishes in seconds)."""
    from oracle import oracle as O
    from scenes import block_yaml

    sim = P.Simulation(P.parse_scenario(block_yaml(20, 12, 10, 0.7)), diagnostics=False)
    f = sim.system.factor
    osys = oracle_system(sim.model, sim.system, use_product_factor=True)
    rng = np.random.default_rng(1)
    b1 = rng.normal(size=(f.n1, 3)); b2 = rng.normal(size=(f.n2, 3))
    y1, y2 = P.forward_sub(f, b1, b2)
    oy1, oy2 = O.forward_sub(osys, b1, b2)
    assert np.abs(y1 - oy1).max() <= 1e-11 * np.abs(oy1).max()
    assert np.abs(y2 - oy2).max() <= 1e-11 * np.abs(oy2).max()
    x2 = rng.normal(size=(f.n2, 3))
    x1 = P.backward_sub(f, y1, x2)
    ox1 = O.backward_sub(osys, oy1, x2)
    assert np.abs(x1 - ox1).max() <= 1e-11 * np.abs(ox1).max()


# ------------------------------------------------------------ whole frames


def _bar_golden(name):
    g = np.load(GOLDEN / f"{name}.npz")
    model, system, state, part = make_bar(press_depth=float(g["press_depth"]), biphasic=bool(g["biphasic"]))
    cfg = sol.SolverConfig(outer_iters=int(g["outer"]), inner_iters=int(g["inner"]),
                           detection_cadence=str(g["cadence"]))
    return g, model, system, state, cfg


@pytest.mark.parametrize("name", ["bar_plain", "bar_multi", "bar_biphasic", "bar_never"])
@pytest.mark.parametrize("graph", [True, False])
def test_frame_lockstep_vs_reference(name, graph):
    """Every frame starts from the REFERENCE's pre-state; the device frame
    must land on the reference's post-state."""
    g, model, system, state, cfg = _bar_golden(name)
    cfg.use_graph = graph
    for f in range(int(g["frames"])):
        st = state_from_golden(g, f"pre{f}_", state)
        met = sol.solve_frame_schur(model, system, st, cfg)
        assert step_rel(st.x, g[f"post{f}_x"], g[f"pre{f}_x"]) < 1e-7, f
        assert np.array_equal(st.active.active, g[f"post{f}_active"])
        np.testing.assert_allclose(st.active.target, g[f"post{f}_target"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(st.rotations.r, g[f"post{f}_R"], rtol=0, atol=1e-10)
        sc = np.abs(g[f"post{f}_f_tilde2"]).max()
        np.testing.assert_allclose(st.f_tilde2, g[f"post{f}_f_tilde2"], rtol=0, atol=1e-8 * sc)
        e, act, pen, res = g[f"metrics{f}"]
        assert met.active_proxies == int(act)
        assert abs(met.energy - e) <= 1e-8 * max(abs(e), 1e-30)
        assert abs(met.max_penetration - pen) <= 1e-12
        assert met.residual < 1e-10


@pytest.mark.parametrize("name", ["cfg1", "hinge"])
def test_scene_lockstep_vs_reference(name):
    g = np.load(GOLDEN / f"{name}.npz")
    sim = P.Simulation(P.parse_scenario(str(g["yaml"])), diagnostics=False)
    checked = 0
    for f in range(1, int(g["frames"]) + 1):
        if f"pre{f}_x" not in g:
            continue
        sim.pose(f)
        st = state_from_golden(g, f"pre{f}_", sim.state)
        met = sol.solve_frame(sim.model, sim.system, st, sim.config)
        assert step_rel(st.x, g[f"post{f}_x"], g[f"pre{f}_x"]) < 1e-7
        assert np.array_equal(st.active.active, g[f"post{f}_active"])
        assert met.active_proxies == int(g[f"metrics{f}"][1])
        checked += 1
    assert checked >= 2


def test_cfg1_free_running_vs_reference():
    """Config 1 through Simulation.step() for all 50 frames: active sets equal
    the reference's every frame; final x within 1e-8 of max|x|."""
    g = np.load(GOLDEN / "cfg1.npz")
    sim = P.Simulation(P.parse_scenario(str(g["yaml"])), diagnostics=False)
    for f in range(1, int(g["frames"]) + 1):
        met = sim.step()
        assert np.array_equal(sim.state.active.active, g[f"active{f}"]), f
        e, act, pen, res = g[f"metrics{f}"]
        assert abs(met.energy - e) <= 1e-7 * abs(e) + 1e-18, f
    assert np.abs(sim.state.x - g["final_x"]).max() <= 1e-8 * np.abs(g["final_x"]).max()


def test_hinge_free_running_vs_oracle():
    """Capsule collider + rotating attachments, outer=2 inner=2, 24 frames:
    device vs oracle free-running."""
    from oracle import oracle as O

    g = np.load(GOLDEN / "hinge.npz")
    sim = P.Simulation(P.parse_scenario(str(g["yaml"])), diagnostics=False)
    osys = oracle_system(sim.model, sim.system)
    ost = oracle_state(sim.state)
    for f in range(1, int(g["frames"]) + 1):
        sim.step()
        O.solve_frame_schur(oracle_scene(sim.model), osys, ost, 2, 2, "inner")
        assert np.array_equal(sim.state.active.active, ost.active), f
        assert np.array_equal(sim.state.active.active, g[f"active{f}"]), f
    assert np.abs(sim.state.x - ost.x).max() <= 1e-9 * np.abs(ost.x).max()


def test_determinism_bitwise():
    """reference test_solver.py:275-283 on the device path."""
    runs = []
    for _ in range(2):
        model, system, state, part = make_bar(press_depth=0.08)
        cfg = sol.SolverConfig(outer_iters=2, inner_iters=3)
        for _ in range(4):
            sol.solve_frame_schur(model, system, state, cfg)
        runs.append(state.x.copy())
    assert np.array_equal(runs[0], runs[1])


def test_no_collision_equals_monolithic(rng):
    """reference test_solver.py:101-110: one pass == dense monolithic solve."""
    model, system, state, part = make_bar()
    model.colliders = []
    state.x += 0.03 * rng.normal(size=state.x.shape)
    pre = state.copy()
    sol.solve_frame_schur(model, system, state, sol.SolverConfig())
    A = system.A.toarray()
    f = sol.compute_forces(model.mesh, model.rest, pre.x, state.rotations, model.params, None, model.attachments)
    dx_ref = np.linalg.solve(A, f[part.order])
    dx = (state.x - pre.x)[part.order]
    assert np.linalg.norm(dx - dx_ref) / np.linalg.norm(dx_ref) < 1e-10


def test_inner_keeps_x1_frozen_and_rhs_maintenance():
    """x1 bitwise frozen inside the inner loop and f~2 maintenance equals a
    scratch forward sweep (reference test_solver.py:198-217, :286-304)."""
    model, system, state, part = make_bar(press_depth=0.08)
    sol.solve_frame_schur(model, system, state, sol.SolverConfig())
    pre = state.copy()
    sol.solve_frame_schur(model, system, state, sol.SolverConfig(outer_iters=1, inner_iters=3))
    x_inner = state.x.copy()
    x_inner[system.x1_ids] = pre.x[system.x1_ids]
    f = sol.compute_forces(model.mesh, model.rest, x_inner, state.rotations, model.params, part.e_alpha,
                           model.attachments)
    _, scratch = P.forward_sub(system.factor, f[system.x1_ids], f[system.x2_ids])
    scale = max(np.abs(scratch).max(), np.abs(state.f_tilde2).max())
    assert np.abs(state.f_tilde2 - scratch).max() < 1e-9 * scale


@pytest.mark.parametrize("env", [{"SPB_SWEEP_FLOW": "1"}, {"SPB_SWEEP_FUSE": "0"}, {"SPB_SWEEP_FUSE": "99"}])
def test_sweep_variants_match(monkeypatch, env):
    """The sweep schedules (dataflow kernels, no fused subtrees, everything in
    subtrees) are alternative orders of the same per-supernode arithmetic:
    each must agree with the default level schedule to roundoff."""
    from scenes import block_yaml

    def sweep(extra):
        for k, v in extra.items():
            monkeypatch.setenv(k, v)
        sim = P.Simulation(P.parse_scenario(block_yaml(16, 10, 8, 0.75)), diagnostics=False)
        f = sim.system.factor
        rng = np.random.default_rng(7)
        b1 = rng.normal(size=(f.n1, 3)); b2 = rng.normal(size=(f.n2, 3)); x2 = rng.normal(size=(f.n2, 3))
        y1, y2 = P.forward_sub(f, b1, b2)
        x1 = P.backward_sub(f, y1, x2)
        for k in extra:
            monkeypatch.delenv(k)
        return y1, y2, x1

    ref = sweep({})
    alt = sweep(env)
    for a, b in zip(ref, alt):
        assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()


@pytest.mark.parametrize("graph", [True, False])
def test_frame_metrics_phase_split(graph):
    """FrameMetrics carries the reference's phase split every frame
    (solver.py:402-446: t_local, t_forward, t_detect, t_dense, t_backward),
    on the graph-replay path as well as eagerly: device times from event
    markers of the last outer pass (detection: around each launch)."""
    model, system, state, _ = make_bar(press_depth=0.08)
    cfg = sol.SolverConfig(outer_iters=1, inner_iters=2, use_graph=graph)
    for _ in range(3):
        met = sol.solve_frame_schur(model, system, state, cfg)
    for k in ("t_local_ms", "t_forward_ms", "t_detect_ms", "t_dense_ms", "t_backward_ms"):
        assert getattr(met, k) > 0.0, k
    parts = met.t_local_ms + met.t_forward_ms + met.t_dense_ms + met.t_backward_ms
    assert parts <= met.t_total_ms
    assert met.t_detect_ms <= met.t_total_ms
