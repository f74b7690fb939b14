"""Pin the ORACLE (oracle/oracle.py) against the golden vectors produced by the
reference itself (tests/golden/make_golden.py). CPU only.

Bars: rotations/SVD bit-exact (numba restated in C, same op order); detection
flags exact; frame solves within 1e-7 step-relative and 1e-12 of max|x| (the oracle's dense
partial factor differs from the reference's AMD sparse factor only by
roundoff)."""

import json

import numpy as np
import pytest

from oracle import oracle as O
from scenes import GOLDEN, make_bar, oracle_scene, oracle_system, step_rel

import paper_2008_01541_b200 as P


def test_oracle_svd_bitwise():
    g = np.load(GOLDEN / "svd.npz")
    U, S, V = O.signed_svd_batch(g["F"])
    assert np.array_equal(U, g["U"])
    assert np.array_equal(S, g["S"])
    assert np.array_equal(V, g["V"])
    assert np.array_equal(O.polar_rotations(g["F"]), g["R"])
    assert np.array_equal(O.biphasic_projections(g["F"], float(g["sigma_min"]), float(g["sigma_max"])), g["Q"])


def _golden_colliders(desc, g):
    cols = []
    for kind, prm, R, t in json.loads(desc):
        if kind == "half_space":
            p = {"point": prm[:3], "normal": prm[3:6]}
        elif kind == "sphere":
            p = {"center": prm[:3], "radius": prm[3]}
        elif kind == "capsule":
            p = {"p0": prm[:3], "p1": prm[3:6], "radius": prm[6]}
        else:
            p = {"origin": g["ls_origin"], "spacing": float(g["ls_spacing"]), "dims": g["ls_dims"],
                 "values": g["ls_values"]}
        cols.append(O.OCollider(kind, p, np.array(R), np.array(t)))
    return cols


@pytest.mark.parametrize("name", ["halfspace", "halfspace_rot", "sphere", "capsule", "capsule_degenerate",
                                  "levelset", "levelset_rot", "multi"])
def test_oracle_detect(name):
    g = np.load(GOLDEN / "detect.npz")
    sc = O.OScene(tets=g["tets"], dm_inverse=None, volume=None, mu=1.0, mu_prime=0.0, sigma_min=0.9,
                  sigma_max=1.1, att_nodes=np.zeros(0, np.int64), att_k=np.zeros(0), att_targets=np.zeros((0, 3)),
                  prox_elem=g["prox_elem"], prox_w=g["prox_w"], prox_c=np.ones(len(g["prox_elem"])),
                  colliders=_golden_colliders(str(g[name + "__desc"]), g), num_nodes=len(g["x"]))
    act, tgt = O.detect(sc, g["x"])
    assert np.array_equal(act, g[name + "__active"])
    np.testing.assert_allclose(tgt, g[name + "__target"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(O.penetration_depths(sc, g["x"]), g[name + "__pen"], rtol=0, atol=1e-13)


def _ostate(g, prefix, biphasic):
    q = g[prefix + "Q"].copy() if biphasic else None
    return O.OState(g[prefix + "x"].copy(), g[prefix + "R"].copy(), q, g[prefix + "active"].copy(),
                    g[prefix + "target"].copy(), g[prefix + "f_tilde2"].copy(), g[prefix + "u2_accum"].copy())


@pytest.mark.parametrize("name", ["bar_plain", "bar_multi", "bar_biphasic", "bar_never"])
def test_oracle_bar_frames(name):
    g = np.load(GOLDEN / f"{name}.npz")
    bip = bool(g["biphasic"])
    model, system, state, part = make_bar(press_depth=float(g["press_depth"]), biphasic=bip)
    assert np.array_equal(part.perm, g["perm"])
    sc = oracle_scene(model)
    osys = oracle_system(model, system)
    np.testing.assert_allclose(osys.sigma0, g["sigma0"], rtol=0, atol=1e-9 * np.abs(g["sigma0"]).max())
    for f in range(int(g["frames"])):
        st = _ostate(g, f"pre{f}_", bip)
        met = O.solve_frame_schur(sc, osys, st, int(g["outer"]), int(g["inner"]), str(g["cadence"]))
        ref_x, pre_x = g[f"post{f}_x"], g[f"pre{f}_x"]
        assert step_rel(st.x, ref_x, pre_x) < 1e-7
        assert np.abs(st.x - ref_x).max() <= 1e-12 * np.abs(ref_x).max()
        assert np.array_equal(st.active, g[f"post{f}_active"])
        np.testing.assert_allclose(st.R, g[f"post{f}_R"], rtol=0, atol=1e-9)
        np.testing.assert_allclose(st.f_tilde2, g[f"post{f}_f_tilde2"], rtol=1e-8,
                                   atol=1e-9 * np.abs(g[f"post{f}_f_tilde2"]).max())
        e, act, pen, res = g[f"metrics{f}"]
        assert met.active_proxies == int(act)
        assert abs(met.energy - e) <= 1e-8 * max(abs(e), 1e-30)
        assert abs(met.max_penetration - pen) <= 1e-10


def _sim_frames(name):
    g = np.load(GOLDEN / f"{name}.npz")
    sim = P.Simulation(P.parse_scenario(str(g["yaml"])), diagnostics=False)
    return g, sim


@pytest.mark.parametrize("name", ["cfg1", "hinge"])
def test_oracle_scene_lockstep(name):
    """Each stored frame: oracle one frame from the reference's pre-state
    (pose from the product's host scripting, pinned by the setup hashes)."""
    g, sim = _sim_frames(name)
    sc0 = oracle_scene(sim.model)
    osys = oracle_system(sim.model, sim.system)
    cfg = sim.config
    nframes = int(g["frames"])
    checked = 0
    for f in range(1, nframes + 1):
        if f"pre{f}_x" not in g:
            continue
        sim.pose(f)
        sc = oracle_scene(sim.model)
        st = O.OState(g[f"pre{f}_x"].copy(), np.broadcast_to(np.eye(3), (sim.mesh.num_elements, 3, 3)).copy(), None,
                      g[f"pre{f}_active"].copy(), g[f"pre{f}_target"].copy(), g[f"pre{f}_f_tilde2"].copy(),
                      g[f"pre{f}_u2_accum"].copy())
        met = O.solve_frame_schur(sc, osys, st, cfg.outer_iters, cfg.inner_iters, cfg.detection_cadence)
        assert step_rel(st.x, g[f"post{f}_x"], g[f"pre{f}_x"]) < 1e-7
        assert np.array_equal(st.active, g[f"post{f}_active"])
        e, act, pen, res = g[f"metrics{f}"]
        assert met.active_proxies == int(act)
        assert abs(met.energy - e) <= 1e-8 * max(abs(e), 1e-30)
        checked += 1
    assert checked >= 2
    del sc0


def test_oracle_cfg1_free_running():
    """All 50 frames of config 1 free-running: active sets equal the
    reference's every frame; final positions within 1e-8 of its max |x|."""
    g, sim = _sim_frames("cfg1")
    osys = oracle_system(sim.model, sim.system)
    ne = sim.mesh.num_elements
    st = O.OState(sim.state.x.copy(), np.broadcast_to(np.eye(3), (ne, 3, 3)).copy(), None,
                  np.zeros(len(sim.model.proxies), bool), np.zeros((len(sim.model.proxies), 3)),
                  np.zeros((osys.n2, 3)), np.zeros((osys.n2, 3)))
    for f in range(1, int(g["frames"]) + 1):
        sim.pose(f)
        O.solve_frame_schur(oracle_scene(sim.model), osys, st, 1, 1, "inner")
        assert np.array_equal(st.active, g[f"active{f}"]), f
    assert np.abs(st.x - g["final_x"]).max() <= 1e-8 * np.abs(g["final_x"]).max()
