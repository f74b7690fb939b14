"""Lockstep parity at BASELINE.json's sizes, pinned by the STOCK REFERENCE.

The fixtures `tests/golden/large_*.npz` were produced by running the
unmodified reference `schurpd` (`tests/golden/make_golden_large.py`, which
imports only the reference) on the BASELINE scenes built through the
reference's own scenario schema (`tests/scene_yaml.py`):

  cfg2_plane  100K tets (40x25x20), m = 1,131, half-space pressing 1 cm/frame
  cfg2_jaw    the same block, a capsule on a `rotate` motion (articulated
              contact, SURVEY §7 H6 / reference hinge_fold.yaml:17-32)
  cfg5_plane  one config-5 scene: 150K tets (50x30x20), m = 1,767
  cfg3_plane  600K tets (80x50x30), m = 6,197: the headline scene
  cfg3_jaw    the headline scene with the articulated capsule ("jaw")

Every recorded frame starts from the REFERENCE's own pre-state (lockstep,
SURVEY §8c protocol 1) and must land on the reference's post-state:
positions within 1e-7 step-relative (the `harness.compare` metric,
harness.py:747-752; north_star asks 1e-6), active sets bit-exact, targets,
f~2 and the frame metrics within stated tolerances. One extra frame runs at
(outer, inner) = (1, 5), the paper's 5-inner case. The host setup is pinned
too: sha256 of every setup array and Σ₀'s diagonal and row sums.
"""

from pathlib import Path

import numpy as np
import pytest

import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import collision as col
from paper_2008_01541_b200 import solver as sol
from scenes import step_rel

GOLDEN = Path(__file__).resolve().parent / "golden"
VARIANTS = ["cfg2_plane", "cfg2_jaw", "cfg5_plane", "cfg3_plane", "cfg3_jaw"]


def _load(name):
    p = GOLDEN / f"large_{name}.npz"
    if not p.exists():
        pytest.fail(f"missing golden {p.name} (tests/golden/make_golden_large.py)")
    return np.load(p)


_SIMS = {}


def _sim(name):
    """One product Simulation per golden (the cfg3 setup takes seconds)."""
    if name not in _SIMS:
        _SIMS.clear()
        g = _load(name)
        _SIMS[name] = (g, P.Simulation(P.parse_scenario(str(g["yaml"])), diagnostics=False))
    return _SIMS[name]


def _state(g, prefix, like):
    st = like.copy()
    st.x[...] = g[prefix + "x"]
    st.active = col.ActiveSet(g[prefix + "active"].copy(), g[prefix + "target"].copy())
    st.f_tilde2 = g[prefix + "f_tilde2"].copy()
    st.u2_accum = g[prefix + "u2_accum"].copy()
    return st


def _check(st, met, g, pre_prefix, post_prefix, metrics):
    rel = step_rel(st.x, g[post_prefix + "x"], g[pre_prefix + "x"])
    assert rel < 1e-7, rel
    assert np.array_equal(st.active.active, g[post_prefix + "active"])
    tscale = max(1.0, np.abs(g[post_prefix + "target"]).max())
    np.testing.assert_allclose(st.active.target, g[post_prefix + "target"], rtol=0, atol=1e-12 * tscale)
    fs = np.abs(g[post_prefix + "f_tilde2"]).max()
    np.testing.assert_allclose(st.f_tilde2, g[post_prefix + "f_tilde2"], rtol=0, atol=1e-8 * fs)
    e, act, pen, res = metrics
    assert met.active_proxies == int(act)
    assert abs(met.energy - e) <= 1e-8 * abs(e)
    assert abs(met.max_penetration - pen) <= 1e-10 * max(1.0, abs(pen))
    assert met.residual < 1e-10
    return rel


@pytest.mark.parametrize("name", VARIANTS)
def test_setup_matches_reference(name):
    """The product's host setup of the BASELINE scene is bit-identical to the
    reference's (mesh, rest data, partition, proxies, attachments), and its
    Σ₀ = A22 - C C^T (linalg.py:380) agrees with the reference's."""
    import hashlib

    g, sim = _sim(name)

    def h(a):
        a = np.ascontiguousarray(a)
        return hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode()).hexdigest()

    m = sim.model
    got = {"rest_positions": sim.mesh.rest_positions, "tets": sim.mesh.tets, "dm_inverse": sim.rest.dm_inverse,
           "volume": sim.rest.volume, "perm": sim.partition.perm, "e_beta": sim.partition.e_beta,
           "prox_elem": m.proxy_elements, "prox_w": m.proxy_weights, "prox_c": m.proxy_stiffness,
           "att_nodes": np.array([a.node for a in m.attachments])}
    for k, v in got.items():
        assert h(v) == str(g[f"hash_{k}"]), k
    assert (sim.partition.n1, sim.partition.n2) == (int(g["n1"]), int(g["n2"]))
    s0 = np.asarray(sim.system.factor.sigma0)
    np.testing.assert_allclose(np.diag(s0), g["sigma0_diag"], rtol=1e-10)
    np.testing.assert_allclose(s0.sum(axis=1), g["sigma0_rowsum"], rtol=0,
                               atol=1e-9 * np.abs(g["sigma0_diag"]).max())


@pytest.mark.gpu
@pytest.mark.parametrize("name", VARIANTS)
def test_lockstep_vs_reference(name):
    """Every recorded frame at the scene's (1, 1), with and without CUDA-graph
    replay, then one frame at (outer, inner) = (1, 5): the active set is
    re-detected on every inner pass at the updated x2 (solver.py:417-440)."""
    g, sim = _sim(name)
    first, lock = int(g["first"]), int(g["lock"])
    for graph in (True, False):
        cfg = sol.SolverConfig(outer_iters=sim.config.outer_iters, inner_iters=sim.config.inner_iters,
                               detection_cadence=sim.config.detection_cadence, use_graph=graph)
        worst = 0.0
        for k in range(lock):
            pre = "pre_" if k == 0 else f"post{k - 1}_"
            sim.pose(first + k)
            st = _state(g, pre, sim.state)
            met = sol.solve_frame_schur(sim.model, sim.system, st, cfg)
            worst = max(worst, _check(st, met, g, pre, f"post{k}_", g[f"metrics{k}"]))
        print(f"{name} graph={graph}: {lock} frames, worst step-relative {worst:.2e}")
    sim.pose(int(g["i5_frame"]))
    pre = f"post{lock - 1}_"
    st = _state(g, pre, sim.state)
    cfg = sol.SolverConfig(outer_iters=1, inner_iters=5, detection_cadence=sim.config.detection_cadence)
    met = sol.solve_frame_schur(sim.model, sim.system, st, cfg)
    rel = _check(st, met, g, pre, "i5_post_", g["i5_metrics"])
    print(f"{name} (1,5): step-relative {rel:.2e}, active {met.active_proxies}")
