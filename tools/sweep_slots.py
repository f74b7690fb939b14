"""Forward/backward sparse sweep times for the slot sizing knobs (one setting
per process: the level tables are built once per factor).
  SPB_FW_SLOTS=3 SPB_BW_SLOTS=4 python tools/sweep_slots.py [cfg]"""
import ctypes
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P  # noqa: E402
from paper_2008_01541_b200 import _native  # noqa: E402
from paper_2008_01541_b200.solver import device_scene  # noqa: E402
from scenes import config_yaml  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
sim = P.Simulation(P.parse_scenario(config_yaml(cfg)), diagnostics=False)
for _ in range(3):
    sim.step()
ds = device_scene(sim.model, sim.system)
out = []
for which in (3, 4):
    v = ctypes.c_double(0)
    _native.check(_native.lib().spb_ctx_bench_kernel(ds.handle, which, 50, ctypes.byref(v)))
    out.append(v.value)
print(f"FW_SLOTS={os.environ.get('SPB_FW_SLOTS', '4')} BW_SLOTS={os.environ.get('SPB_BW_SLOTS', '4')} "
      f"forward {1e3 * out[0]:.1f} us backward {1e3 * out[1]:.1f} us", flush=True)
