"""Early exit and late-registered colliders on the device path.

* Early exit (reference solver.py:448-452, the invariant of the reference's
  test_solver.py::test_early_exit_skips_remaining_outer_passes, which spies on
  the Python-level collision.detect and so cannot run against a device
  frame): after every outer pass the RMS of the total nodal force
  (_equilibrium_residual, solver.py:468-471) is computed on the device; once
  it is <= the threshold the remaining passes are skipped.
* A collider that becomes active after CUDA graphs were captured (the
  built-in untangle scene: capsule active_from_frame 45) must reach the
  captured detection nodes: graph replay and eager enqueue agree bitwise, and
  both follow the reference's own run of the scene (tests/golden/untangle.npz).
"""

from pathlib import Path

import numpy as np
import pytest

import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import solver as sol
from scenes import make_bar

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def _passes(model, system, state, outer, inner, cadence="inner", early=None, graph=True):
    ds = sol.device_scene(model, system)
    met = ds.step(model, state, outer, inner, cadence, graph, early)
    return int(met.outer_passes)


def test_early_exit_skips_remaining_outer_passes():
    model, system, state, _ = make_bar(press_depth=0.08)
    one = state.copy()
    assert _passes(model, system, one, 1, 1) == 1
    st = state.copy()
    assert _passes(model, system, st, 6, 1, early=1e12) == 1  # exits after the first pass
    assert np.array_equal(st.x, one.x)
    assert np.array_equal(st.active.active, one.active.active)
    # a threshold never met runs every pass and equals the fused 6-pass frame
    six = state.copy()
    assert _passes(model, system, six, 6, 1) == 6
    st = state.copy()
    assert _passes(model, system, st, 6, 1, early=0.0) == 6
    assert np.array_equal(st.x, six.x)
    # through the public API (solver.py SolverConfig.early_exit_residual)
    st = state.copy()
    sol.solve_frame_schur(model, system, st, sol.SolverConfig(outer_iters=6, inner_iters=1, early_exit_residual=1e12))
    assert np.array_equal(st.x, one.x)


@pytest.mark.parametrize("cadence", ["frame", "inner", "never"])
def test_early_exit_per_pass_path_equals_fused_frame(cadence):
    """'frame' cadence detects only in the first outer pass even when the
    passes are issued one by one (first_detection_done, solver.py:417-421)."""
    model, system, state, _ = make_bar(press_depth=0.08)
    sol.solve_frame_schur(model, system, state, sol.SolverConfig())  # some contact in state.active
    a = state.copy()
    b = state.copy()
    assert _passes(model, system, a, 3, 2, cadence) == 3
    assert _passes(model, system, b, 3, 2, cadence, early=0.0) == 3
    assert np.array_equal(a.x, b.x)
    assert np.array_equal(a.active.active, b.active.active)
    assert np.array_equal(a.active.target, b.active.target)


def test_early_exit_threshold_matches_reference_residual():
    """The device RMS is the reference's _equilibrium_residual. After a pass
    the forces are evaluated with the rotations that pass solved with, so the
    residual is at roundoff level (~1e-13 here) and its last digits depend on
    summation order: a threshold 1e3x above the host-evaluated value stops
    after pass 1, one 1e3x below it does not."""
    model, system, state, _ = make_bar(press_depth=0.08)
    s1 = state.copy()
    _passes(model, system, s1, 1, 1)
    r1 = sol._equilibrium_residual(model, s1)  # host restatement of solver.py:468-471 (test-side check)
    assert 0.0 < r1 < 1e-6
    st = state.copy()
    assert _passes(model, system, st, 4, 1, early=r1 * 1e3) == 1
    st = state.copy()
    assert _passes(model, system, st, 4, 1, early=r1 * 1e-3) > 1


def test_early_exit_pcg():
    model, system, state, _ = make_bar(press_depth=0.08)
    cfg = sol.SolverConfig(outer_iters=4, inner_iters=1, solver_kind="pcg")
    one = state.copy()
    sol.solve_frame_pcg(model, system, one, sol.SolverConfig(outer_iters=1, inner_iters=1, solver_kind="pcg"))
    st = state.copy()
    cfg.early_exit_residual = 1e12
    sol.solve_frame_pcg(model, system, st, cfg)
    assert np.array_equal(st.x, one.x)


def test_collider_registered_after_graph_capture():
    """untangle.yaml: frames 1-44 run (graphs captured) with no collider; the
    capsule appears at frame 45. Graph replay == eager enqueue bitwise, and
    both follow the reference's per-frame active sets."""
    g = np.load(GOLDEN / "untangle.npz")
    runs = []
    for use_graph in (True, False):
        sim = P.Simulation(P.parse_scenario(str(g["yaml"])), diagnostics=False)
        sim.config.use_graph = use_graph
        for f in range(1, 50):
            met = sim.step()
            assert np.array_equal(sim.state.active.active, g[f"active{f}"]), (use_graph, f)
            e = g[f"metrics{f}"][0]
            assert abs(met.energy - e) <= 1e-7 * abs(e) + 1e-18, (use_graph, f)
            if f"x{f}" in g:
                ref = g[f"x{f}"]
                assert np.abs(sim.state.x - ref).max() <= 1e-8 * np.abs(ref).max(), (use_graph, f)
        assert sim.state.active.count > 0
        runs.append(sim.state.x.copy())
    assert np.array_equal(runs[0], runs[1])
