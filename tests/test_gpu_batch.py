"""Batch mode (BASELINE config 5): scenes sharing one factor stepped
concurrently on separate streams must give bit-identical states to the same
scenes stepped one at a time (per-context sweep workspaces, no shared
scratch), and the scenes must really differ (different collider speeds)."""

import ctypes

import numpy as np
import pytest

import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import _native
from paper_2008_01541_b200.solver import device_scene
from scenes import block_yaml

pytestmark = pytest.mark.gpu


def _scenes(k):
    sims = []
    for i in range(k):
        sim = P.Simulation(P.parse_scenario(block_yaml(16, 10, 8, 0.75, vel=-0.004 * (1 + i / 64.0) * 4)),
                           diagnostics=False)
        if sims:
            sim.system = sims[0].system
        sims.append(sim)
    for sim in sims:
        for _ in range(3):
            sim.step()
    return sims


def _x(ds, n):
    x = np.empty((n, 3))
    _native.check(_native.lib().spb_ctx_get_state(ds.handle, _native.ptr(x), None, None, None, None, None, None))
    return x


def test_concurrent_scenes_match_serial():
    lib = _native.lib()
    cfg = _native.StepConfig(1, 1, 0, 1, 0, -1.0)
    a = _scenes(3)
    hs = [device_scene(s.model, s.system) for s in a]
    assert len({id(h) for h in hs}) == 3 and a[1].system is a[0].system
    arr = (ctypes.c_void_p * 3)(*[h.handle for h in hs])
    ms = ctypes.c_double(0)
    _native.check(lib.spb_bench_batch(arr, 3, ctypes.byref(cfg), 4, ctypes.byref(ms)))
    xa = [_x(h, a[0].mesh.num_nodes) for h in hs]
    b = _scenes(3)
    xb = []
    for s in b:
        h = device_scene(s.model, s.system)
        _native.check(lib.spb_ctx_bench(h.handle, ctypes.byref(cfg), 4, ctypes.byref(ms), None))
        xb.append(_x(h, s.mesh.num_nodes))
    for u, v in zip(xa, xb):
        assert np.array_equal(u, v)
    assert not np.array_equal(xa[0], xa[2])


def test_concurrency_hint_is_bitwise_neutral():
    """spb_ctx_set_concurrency only resizes the tile-Cholesky grid (cfg2:
    36 -> 18 CTAs for 8 concurrent scenes): every tile is still computed in
    the same order, so the frames are bit-identical."""
    text = block_yaml(40, 25, 20, 0.7)
    a = P.Simulation(P.parse_scenario(text), diagnostics=False)
    b = P.Simulation(P.parse_scenario(text), diagnostics=False)
    device_scene(b.model, b.system).set_concurrency(8)
    for _ in range(3):
        a.step()
        b.step()
    assert a.state.active.count > 0
    assert np.array_equal(a.state.x, b.state.x)
    device_scene(b.model, b.system).set_concurrency(1)
    a.step()
    b.step()
    assert np.array_equal(a.state.x, b.state.x)


def test_step_batch_matches_sequential_steps():
    """harness.step_batch (one spb_frame_batch call: every scene's frame in
    flight before the host waits) leaves each scene exactly where step() would."""
    def sims():
        out = []
        for i in range(3):
            s = P.Simulation(P.parse_scenario(block_yaml(16, 10, 8, 0.75, vel=-0.004 * (1 + i / 64.0) * 4)),
                             diagnostics=False)
            if out:
                s.system = out[0].system
            out.append(s)
        return out

    a, b = sims(), sims()
    for _ in range(4):
        ma = P.step_batch(a)
        mb = [s.step() for s in b]
    for sa, sb, x, y in zip(a, b, ma, mb):
        assert np.array_equal(sa.state.x, sb.state.x)
        assert np.array_equal(sa.state.active.active, sb.state.active.active)
        assert np.array_equal(sa.state.f_tilde2, sb.state.f_tilde2)
        assert x.active_proxies == y.active_proxies and x.energy == y.energy
    assert a[0].state.active.count > 0
    assert not np.array_equal(a[0].state.x, a[2].state.x)
