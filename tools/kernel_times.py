"""Graph-replay times of the frame pieces on a config (diagnostics)."""
import ctypes, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import _native
from paper_2008_01541_b200.solver import device_scene
from scenes import config_yaml
sim = P.Simulation(P.parse_scenario(config_yaml(sys.argv[1] if len(sys.argv) > 1 else "cfg3")), diagnostics=False)
for _ in range(3): sim.step()
ds = device_scene(sim.model, sim.system)
out = []
for name, w in (("cholesky", 0), ("dense_backward", 1), ("sigma0_gemv", 2), ("sparse_forward", 3), ("sparse_backward", 4)):
    v = ctypes.c_double(0)
    _native.check(_native.lib().spb_ctx_bench_kernel(ds.handle, w, 20, ctypes.byref(v)))
    out.append(f"{name} {v.value * 1e3:.1f} us")
cfg = _native.StepConfig(1, 1, 0, 1, 0, -1.0); ms = ctypes.c_double(0)
_native.check(_native.lib().spb_ctx_bench(ds.handle, ctypes.byref(cfg), 200, ctypes.byref(ms), None))
print(" | ".join(out), f"| frame {ms.value:.3f} ms")
