"""Device-resident frame time and phase split of a config (diagnostics):
   python tools/phase_probe.py cfg3 [frames]"""
import ctypes, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import _native
from paper_2008_01541_b200.solver import device_scene
from scenes import config_yaml
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 50
sim = P.Simulation(P.parse_scenario(config_yaml(name)), diagnostics=False)
for _ in range(3): sim.step()
ds = device_scene(sim.model, sim.system)
cfg = _native.StepConfig(1, 1, _native.CADENCES[sim.config.detection_cadence], 1, 0, -1.0)
ms = ctypes.c_double(0); ph = (ctypes.c_double * 5)()
_native.check(_native.lib().spb_ctx_bench(ds.handle, ctypes.byref(cfg), frames, ctypes.byref(ms), ph))
print(f"{name}: {ms.value:.3f} ms/frame  local {ph[0]:.3f} fw {ph[1]:.3f} inner {ph[2]:.3f} bw {ph[3]:.3f} met {ph[4]:.3f}")
