"""Proxy setup on the device: collision.scatter_proxies
(reference collision.py:255-300) through spb_scatter_proxies.

* Bit-identical to the host path (the reference's owner map and append
  order) for node-set, mask and predicate regions and 1 / 4 / 16 points per
  triangle, on lattice meshes.
* At BASELINE size, the proxies of the reference's own setup: the product's
  Simulation (device path on a GPU box) reproduces the sha256 of the
  reference's proxy elements / weights / stiffness recorded in the golden
  fixtures (tests/golden/make_golden_large.py).
"""

import hashlib
from pathlib import Path

import numpy as np
import pytest

import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import _native
from paper_2008_01541_b200 import collision as col
from paper_2008_01541_b200 import mesh as pmesh

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def _host(monkeypatch, *args, **kw):
    monkeypatch.setenv("SPB_SETUP_DEVICE", "0")
    try:
        return col.scatter_proxies(*args, **kw)
    finally:
        monkeypatch.delenv("SPB_SETUP_DEVICE")


def _same(a, b):
    assert len(a) == len(b)
    assert [p.element for p in a] == [p.element for p in b]
    wa = np.array([p.weights for p in a])
    wb = np.array([p.weights for p in b])
    assert wa.tobytes() == wb.tobytes()
    assert all(p.stiffness == q.stiffness for p, q in zip(a, b))


@pytest.mark.parametrize("per", [1, 4, 16])
def test_scatter_device_equals_host(monkeypatch, per):
    mesh = pmesh.build_box_lattice((1.2, 0.5, 0.4), (12, 5, 4))
    assert _native.scatter_proxies(mesh.tets, mesh.num_nodes, mesh.surface_tris,
                                   np.ones(mesh.num_nodes, bool), 1, np.array([[1 / 3] * 3])) is not None
    z = mesh.rest_positions[:, 2]
    regions = [
        lambda X: X[:, 2] > 0.3,  # predicate (top face)
        np.flatnonzero(mesh.rest_positions[:, 0] < 0.25),  # node ids
        z < 0.05,  # boolean mask
        np.ones(mesh.num_nodes, dtype=bool),  # every surface triangle
    ]
    for reg in regions:
        dev = col.scatter_proxies(mesh, reg, per_element=per, stiffness=2.5e4)
        _same(dev, _host(monkeypatch, mesh, reg, per_element=per, stiffness=2.5e4))


def test_scatter_device_empty_region_raises():
    mesh = pmesh.build_box_lattice((1.0, 1.0, 1.0), (3, 3, 3))
    inner = np.zeros(mesh.num_nodes, dtype=bool)
    inner[np.argmin(np.abs(mesh.rest_positions - 0.5).sum(axis=1))] = True  # one interior node
    with pytest.raises(P.EmptyRegionError):
        col.scatter_proxies(mesh, inner)


@pytest.mark.parametrize("name", ["cfg2_plane", "cfg2_jaw", "cfg5_plane"])
def test_baseline_proxies_match_reference(name):
    g = np.load(GOLDEN / f"large_{name}.npz")
    sim = P.Simulation(P.parse_scenario(str(g["yaml"])), diagnostics=False)

    def h(a):
        a = np.ascontiguousarray(a)
        return hashlib.sha256(a.tobytes() + str(a.dtype).encode() + str(a.shape).encode()).hexdigest()

    m = sim.model
    for k, v in {"prox_elem": m.proxy_elements, "prox_w": m.proxy_weights, "prox_c": m.proxy_stiffness}.items():
        assert h(v) == str(g[f"hash_{k}"]), k
