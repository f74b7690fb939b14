"""Where the end-to-end frame time goes (Simulation.step vs the device frame).

    python tools/e2e_profile.py [cfg3] [frames]

Prints: device-resident ms/frame (spb_ctx_bench), Simulation.step() ms/frame,
the share spent in pose / the C call / the Python around it, and a cProfile
top list of one batch of steps."""
import cProfile
import ctypes
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2008_01541_b200 as P  # noqa: E402
from paper_2008_01541_b200 import _native  # noqa: E402
from paper_2008_01541_b200 import solver as sol  # noqa: E402
from scenes import config_yaml  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 40
sim = P.Simulation(P.parse_scenario(config_yaml(cfg)), diagnostics=False)
for _ in range(5):
    sim.step()
ds = sol.device_scene(sim.model, sim.system)
c = _native.StepConfig(1, 1, 0, 1, 0, -1.0)
ms = ctypes.c_double(0)
_native.check(_native.lib().spb_ctx_bench(ds.handle, ctypes.byref(c), frames, ctypes.byref(ms), None))
print(f"device frame        {ms.value:.3f} ms")
t0 = time.perf_counter()
for _ in range(frames):
    sim.step()
t_step = (time.perf_counter() - t0) / frames * 1e3
print(f"Simulation.step     {t_step:.3f} ms")
tp = tc = 0.0
orig = ds.step


def timed_step(*a, **k):
    global tc
    t = time.perf_counter()
    r = orig(*a, **k)
    tc += time.perf_counter() - t
    return r


ds.step = timed_step
tin = [0.0]
for _ in range(frames):
    sim.frame += 1
    t = time.perf_counter()
    sim.pose(sim.frame)
    tp += time.perf_counter() - t
    m = sol.solve_frame(sim.model, sim.system, sim.state, sim.config)
    tin[0] += sim.state.metrics[-1].t_total_ms
print(f"  pose              {tp / frames * 1e3:.3f} ms")
print(f"  DeviceScene.step  {tc / frames * 1e3:.3f} ms")
print(f"  solve_frame total {tin[0] / frames:.3f} ms (FrameMetrics.t_total_ms)")
# inside the C call: spb_ctx_frame's own wall clock (spb_frame_metrics.t_total_ms)
ds.step = orig
cm = []
for _ in range(frames):
    sim.frame += 1
    sim.pose(sim.frame)
    met = ds.step(sim.model, sim.state, 1, 1, sim.config.detection_cadence, True)
    cm.append(met.t_total_ms)
import numpy as np  # noqa: E402
print(f"  spb_ctx_frame wall {np.mean(cm):.3f} ms (median {np.median(cm):.3f})")
ds.step = timed_step
pr = cProfile.Profile()
pr.enable()
for _ in range(frames):
    sim.step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
