"""Per-call host timing of the device path inside Simulation.step (diagnostics)."""
import ctypes, sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import _native, solver as S
from scenes import config_yaml
sim = P.Simulation(P.parse_scenario(config_yaml(sys.argv[1] if len(sys.argv) > 1 else "cfg3")), diagnostics=False)
for _ in range(5): sim.step()
ds = S.device_scene(sim.model, sim.system)
T = {k: 0.0 for k in ("harness.pose", "ds.pose", "set_state", "step(graph+sync)", "get_state", "glue")}
F = 50
lib = _native.lib()
t_all = time.perf_counter()
for f in range(F):
    t = time.perf_counter(); sim.frame += 1; sim.pose(sim.frame); T["harness.pose"] += time.perf_counter() - t
    st = sim.state
    t = time.perf_counter(); ds.pose(sim.model); T["ds.pose"] += time.perf_counter() - t
    t = time.perf_counter()
    x = _native.f64(st.x); act = np.ascontiguousarray(st.active.active, dtype=np.uint8); tgt = _native.f64(st.active.target)
    T["glue"] += time.perf_counter() - t
    t = time.perf_counter()
    _native.check(lib.spb_ctx_set_state(ds.handle, _native.ptr(x), None, None, _native.ptr(act), _native.ptr(tgt), None, None))
    T["set_state"] += time.perf_counter() - t
    t = time.perf_counter()
    cfg = _native.StepConfig(1, 1, 0, 1, 0, -1.0); met = _native.FrameMetricsC()
    _native.check(lib.spb_ctx_step(ds.handle, ctypes.byref(cfg), ctypes.byref(met)))
    T["step(graph+sync)"] += time.perf_counter() - t
    t = time.perf_counter()
    a = np.empty(ds.P, np.uint8); tg = np.empty((ds.P, 3)); f2 = np.empty((ds.m, 3)); u2 = np.empty((ds.m, 3))
    T["glue"] += time.perf_counter() - t
    t = time.perf_counter()
    _native.check(lib.spb_ctx_get_state(ds.handle, _native.ptr(x), None, None, _native.ptr(a), _native.ptr(tg), _native.ptr(f2), _native.ptr(u2)))
    T["get_state"] += time.perf_counter() - t
    t = time.perf_counter()
    st.active = P.ActiveSet(a.astype(bool), tg); st.f_tilde2 = f2; st.u2_accum = u2
    T["glue"] += time.perf_counter() - t
tot = time.perf_counter() - t_all
for k, v in T.items(): print(f"{k:18s} {v / F * 1e3:7.3f} ms")
print(f"{'total':18s} {tot / F * 1e3:7.3f} ms;  Simulation.step:", end=" ")
t = time.perf_counter()
for _ in range(F): sim.step()
print(f"{(time.perf_counter() - t) / F * 1e3:.3f} ms")
