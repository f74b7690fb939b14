"""Where the batch (config 5, step_batch) end-to-end time goes (diagnostics):
device round (spb_bench_batch) vs step_batch wall time, and a cProfile of
step_batch rounds.  python tools/batch_profile.py [scenes] [rounds]"""
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
from paper_2008_01541_b200.solver import device_scene  # noqa: E402
from scene_yaml import CONFIGS, block_yaml  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
R = int(sys.argv[2]) if len(sys.argv) > 2 else 40
sims = []
for k in range(S):
    sim = P.Simulation(P.parse_scenario(block_yaml(*CONFIGS["cfg5"], vel=-0.004 * (1 + k / 64.0))), diagnostics=False)
    if sims:
        sim.system = sims[0].system
    sims.append(sim)
for _ in range(4):
    P.step_batch(sims)
handles = (ctypes.c_void_p * S)(*[device_scene(s.model, s.system).handle for s in sims])
cfg = _native.StepConfig(1, 1, _native.CADENCES[sims[0].config.detection_cadence], 1, 0, -1.0)
ms = ctypes.c_double(0)
_native.check(_native.lib().spb_bench_batch(handles, S, ctypes.byref(cfg), R, ctypes.byref(ms)))
print(f"device round {ms.value:.3f} ms ({S} scenes)")
t0 = time.perf_counter()
for _ in range(R):
    P.step_batch(sims)
print(f"step_batch round {(time.perf_counter() - t0) / R * 1e3:.3f} ms")
tc = 0.0
orig = _native.lib().spb_frame_batch
pr = cProfile.Profile()
pr.enable()
for _ in range(R):
    P.step_batch(sims)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
