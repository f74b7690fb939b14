"""Parity at BASELINE.json's full size (config 3: 600K tets, 128,061 nodes,
m = 6,197 prone nodes, 8,000 proxies) on the GPU, through the C ABI.

At this size the reference's own precompute takes ~8 min. The oracle
therefore runs the reference algorithm (oracle/oracle.py, solver.py:387-455)
on the product's exported factor (L1, C, sigma0), and the exported factor is
checked on its own through size-independent properties:
  * three-step solve (forward sweep, dense Schur solve, backward sweep)
    against the monolithic A (reference test_linalg.py:143-159 semantics);
  * dense Cholesky of H = sigma0 + C22 (every proxy active) against LAPACK;
  * a lockstep frame against the oracle (positions 1e-7 step-relative,
    active set bit-exact);
  * bit-identical replays.
"""

import numpy as np
import pytest

import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import collision as col
from paper_2008_01541_b200 import solver as sol
from scenes import config_yaml, oracle_scene, oracle_state, oracle_system, step_rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg3():
    sim = P.Simulation(P.parse_scenario(config_yaml("cfg3")), diagnostics=False)
    assert sim.mesh.num_elements == 600_000 and sim.partition.n2 == 6_197
    for _ in range(4):  # the plane reaches the top face on frame 2
        met = sim.step()
    assert met.active_proxies > 0
    return sim


def test_cfg3_three_step_solve_equals_monolithic(cfg3):
    f = cfg3.system.factor
    rng = np.random.default_rng(3)
    b1 = rng.normal(size=(f.n1, 3))
    b2 = rng.normal(size=(f.n2, 3))
    y1, ft2 = P.forward_sub(f, b1, b2)
    x2 = P.dense_solve(P.dense_factor(np.asarray(f.sigma0)), ft2)
    x1 = P.backward_sub(f, y1, x2)
    A = cfg3.system.A.full()
    x = np.concatenate([x1, x2])
    b = np.concatenate([b1, b2])
    assert np.linalg.norm(A @ x - b) <= 1e-10 * np.linalg.norm(b)


def test_cfg3_dense_factor_vs_lapack(cfg3):
    """H = sigma0 + C22 with all 8,000 proxies active (the largest H of the
    scene): device tile Cholesky vs LAPACK dpotrf, and the solve residual."""
    sim = cfg3
    P_ = len(sim.model.proxies)
    act = col.ActiveSet(np.ones(P_, dtype=bool), np.zeros((P_, 3)))
    c22 = col.assemble_c22(sim.model.proxies, act, sim.partition, sim.mesh)
    h = np.asarray(sim.system.factor.sigma0) + c22.full().toarray()
    f = P.dense_factor(h)
    ref = np.linalg.cholesky(h)
    assert np.abs(f.chol - ref).max() <= 1e-12 * np.abs(ref).max()
    g = np.random.default_rng(5).normal(size=(h.shape[0], 3))
    u = P.dense_solve(f, g)
    assert np.linalg.norm(h @ u - g) <= 1e-10 * np.linalg.norm(g)


def test_cfg3_frame_lockstep_vs_oracle(cfg3):
    from oracle import oracle as O

    sim = cfg3
    pre = sim.state.copy()
    osys = oracle_system(sim.model, sim.system, use_product_factor=True)
    ost = oracle_state(pre)
    sim.frame += 1
    sim.pose(sim.frame)
    st = pre.copy()
    met = sol.solve_frame(sim.model, sim.system, st, sim.config)
    cfg = sim.config
    om = O.solve_frame_schur(oracle_scene(sim.model), osys, ost, cfg.outer_iters, cfg.inner_iters,
                             cfg.detection_cadence)
    assert step_rel(st.x, ost.x, pre.x) < 1e-7
    assert np.array_equal(st.active.active, ost.active)
    np.testing.assert_allclose(st.active.target, ost.target, rtol=0, atol=1e-12)
    assert met.active_proxies == om.active_proxies
    assert abs(met.energy - om.energy) <= 1e-8 * abs(om.energy)
    assert met.residual < 1e-10
    sim.state = st


def test_cfg3_replay_bit_identical(cfg3):
    sim = cfg3
    pre = sim.state.copy()
    runs = []
    for use_graph in (True, True, False):
        st = pre.copy()
        cfg = sol.SolverConfig(outer_iters=1, inner_iters=2, use_graph=use_graph)
        sol.solve_frame_schur(sim.model, sim.system, st, cfg)
        runs.append((st.x.copy(), st.active.active.copy(), st.f_tilde2.copy()))
    for r in runs[1:]:
        for a, b in zip(runs[0], r):
            assert np.array_equal(a, b)
