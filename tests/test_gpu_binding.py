"""The reference-side ctypes binding (integration/schurpd_binding.py), driven
with this package's mirror types (same field names as the reference's), must
give the same frame as the package's own device path: bit-identical, since
both run the same kernels."""

import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2008_01541_b200 import solver as sol
from scenes import make_bar

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "integration"))

pytestmark = pytest.mark.gpu


def test_binding_matches_package_path(monkeypatch):
    import schurpd_binding as B

    model, system, state, part = make_bar(press_depth=0.08)
    cfg = sol.SolverConfig(outer_iters=2, inner_iters=2)
    a, b = state.copy(), state.copy()
    ma = sol.solve_frame_schur(model, system, a, cfg)
    monkeypatch.setitem(sol.SOLVE_FUNCTIONS, "schur", sol.SOLVE_FUNCTIONS["schur"])
    B.install(sol)
    mb = sol.solve_frame(model, system, b, cfg)
    assert np.array_equal(a.x, b.x)
    assert np.array_equal(a.active.active, b.active.active)
    assert np.array_equal(a.f_tilde2, b.f_tilde2)
    assert np.array_equal(a.rotations.r, b.rotations.r)
    assert ma.active_proxies == mb.active_proxies > 0
    assert ma.energy == mb.energy
    assert b.metrics[-1] is mb
