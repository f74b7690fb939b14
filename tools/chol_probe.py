"""Time the tile Cholesky alone on a config's H (diagnostics)."""
import ctypes, os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import _native
from paper_2008_01541_b200.solver import device_scene
from scenes import config_yaml
cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
sim = P.Simulation(P.parse_scenario(config_yaml(cfgname)), diagnostics=False)
for _ in range(3): sim.step()
ds = device_scene(sim.model, sim.system)
m = sim.partition.n2
ms = ctypes.c_double()
_native.check(_native.lib().spb_ctx_bench_cholesky(ds.handle, 5, ctypes.byref(ms)))
print(f"{cfgname}: {ms.value:.3f} ms  {m**3/3/ms.value/1e9:.2f} TF")
