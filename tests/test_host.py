"""Host-side checks (CPU): setup bit-identity with the reference, native
precompute correctness, C-ABI exports, scenario schema."""

import ctypes
import hashlib
import re
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import _native
from scenes import GOLDEN, block_yaml, make_bar

ROOT = Path(__file__).resolve().parent.parent


def h(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode()).hexdigest()


@pytest.mark.parametrize("name", ["cfg1", "hinge"])
def test_setup_bit_identical_to_reference(name):
    g = np.load(GOLDEN / f"{name}.npz")
    sim = P.Simulation(P.parse_scenario(str(g["yaml"])), diagnostics=False)
    m = sim.model
    arrays = dict(rest_positions=sim.mesh.rest_positions, tets=sim.mesh.tets, surface_tris=sim.mesh.surface_tris,
                  dm_inverse=sim.rest.dm_inverse, volume=sim.rest.volume, perm=sim.partition.perm,
                  e_beta=sim.partition.e_beta, prox_elem=m.proxy_elements, prox_w=m.proxy_weights,
                  prox_c=m.proxy_stiffness, att_nodes=np.array([a.node for a in m.attachments]))
    for k, v in arrays.items():
        assert h(v) == str(g["hash_" + k]), k
    assert sim.partition.n2 == int(g["n2"])


def test_sigma0_matches_reference():
    ref = np.load(GOLDEN / "cfg1_sigma0.npz")["sigma0"]
    g = np.load(GOLDEN / "cfg1.npz")
    sim = P.Simulation(P.parse_scenario(str(g["yaml"])), diagnostics=False)
    assert np.abs(sim.system.factor.sigma0 - ref).max() <= 1e-12 * np.abs(ref).max()


def test_partial_cholesky_known_answer():
    """reference test_linalg.py:75-80: [[4,1],[1,3]] -> L1=2, C=0.5, sigma0=2.75."""
    f = P.partial_cholesky(P.ScalarSparseSym.from_dense(np.array([[4.0, 1.0], [1.0, 3.0]])), 1)
    assert f.l1.to_scipy().toarray()[0, 0] == 2.0
    assert f.coupling.toarray()[0, 0] == 0.5
    assert f.sigma0[0, 0] == 2.75


@pytest.mark.parametrize("cells,frac", [((20, 12, 10), 0.7), ((12, 8, 6), 1.0)])
def test_factor_identities(cells, frac):
    sim = P.Simulation(P.parse_scenario(block_yaml(*cells, frac)), diagnostics=False)
    f = sim.system.factor
    A = sim.system.A.full()
    n1 = f.n1
    a11 = A[:n1, :n1][f.fill_perm][:, f.fill_perm]
    L = f.l1.to_scipy()
    assert abs(L @ L.T - a11).max() <= 1e-12 * abs(a11).max()
    a21 = A[n1:, :n1][:, f.fill_perm]
    assert abs(f.coupling @ L.T - a21).max() <= 1e-12 * abs(a21).max()
    s0 = A[n1:, n1:].toarray() - (f.coupling @ f.coupling.T).toarray()
    assert np.abs(s0 - f.sigma0).max() <= 1e-12 * np.abs(s0).max()
    assert np.array_equal(f.sigma0, f.sigma0.T)
    # the nested-dissection tree is shallow (device chain length)
    assert f.native.levels <= 20


@pytest.mark.parametrize("split", [(50, 30), (80, 1), (80, 79), (64, 0), (64, 64)])
def test_partial_cholesky_splits(rng, split):
    n, n1 = split
    M = sp.random(n, n, density=0.08, random_state=np.random.RandomState(3))
    A = (M @ M.T + sp.diags(np.full(n, 2.0))).toarray()
    f = P.partial_cholesky(P.ScalarSparseSym.from_dense(A), n1)
    Ad = A
    if n1:
        L = f.l1.to_scipy().toarray()
        a11 = Ad[:n1, :n1][f.fill_perm][:, f.fill_perm]
        assert np.abs(L @ L.T - a11).max() <= 1e-12 * np.abs(a11).max()
    if n - n1:
        ref = Ad[n1:, n1:] - (Ad[n1:, :n1] @ np.linalg.solve(Ad[:n1, :n1], Ad[:n1, n1:]) if n1 else 0)
        assert np.abs(f.sigma0 - ref).max() <= 1e-10 * np.abs(ref).max()


def test_indefinite_leading_block_names_column():
    A = np.diag([4.0, 1.0, -2.0, 5.0])
    with pytest.raises(P.IndefiniteMatrixError) as ei:
        P.partial_cholesky(P.ScalarSparseSym.from_dense(A), 3, use_fill_ordering=False)
    assert ei.value.column == 2


def test_build_system_requires_anchoring():
    mesh = P.build_box_lattice((1, 1, 1), (2, 2, 2))
    rest = P.compute_rest_data(mesh)
    part = P.classify(mesh, [])
    with pytest.raises(P.SolverSetupError):
        P.build_system(mesh, rest, P.MaterialParams(mu=1e4), [], part)


def test_fill_ordering_beats_natural():
    sim = P.Simulation(P.parse_scenario(block_yaml(20, 12, 10, 0.7)), diagnostics=True)
    d = sim.diagnostics
    assert d.constrained_factor_nnz > 0 and d.free_factor_nnz > 0
    A = sim.system.A.full()
    nat = _native.symbolic_nnz(A.shape[0], sp.triu(A, format="csc"))
    assert d.free_factor_nnz < 0.5 * nat


def test_c_abi_exports_every_declared_symbol():
    """Every entry point declared in include/schurpd_b200.h is exported by the
    library and bound by the shim (no compute call needs a GPU here)."""
    header = (ROOT / "include" / "schurpd_b200.h").read_text()
    declared = set(re.findall(r"\b(spb_[a-z0-9_]+)\s*\(", header))
    L = ctypes.CDLL(str(_native.LIB_PATH))
    for name in declared:
        assert hasattr(L, name), name
    assert declared <= set(_native.EXPORTED)
    assert _native.lib().spb_version() >= 100


def test_scenario_schema_rejects_unknown_keys():
    g = np.load(GOLDEN / "cfg1.npz")
    text = str(g["yaml"]).replace("frames: 50", "frames: 50\nbogus: 1")
    with pytest.raises(P.ScenarioError) as ei:
        P.parse_scenario(text)
    assert "bogus" in str(ei.value)
    bad = str(g["yaml"]).replace("stiffness: 1.0e+7", "stiffness: 1.0e+7\n    extra: 2")
    with pytest.raises(P.ScenarioError) as ei:
        P.parse_scenario(bad)
    assert "attachments[0]" in str(ei.value)


def test_scenario_round_trip():
    sc = P.load_scenario(P.builtin_scene_path("hinge_fold"))
    assert P.parse_scenario(sc.to_yaml()) == sc


def test_motion_rates():
    sc = P.load_scenario(P.builtin_scene_path("hinge_fold"))
    tf = sc.attachments[1].motion.transform_at(1)
    ang = np.degrees(np.arccos((np.trace(tf.rotation) - 1) / 2))
    assert abs(ang - 2.5) < 1e-9
