"""Per-task cost model of the tile Cholesky from a traced launch (diagnostics):
duration = a + b * k_steps, fitted per task kind."""
import ctypes, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import _native
from paper_2008_01541_b200.solver import device_scene
from scenes import config_yaml
sim = P.Simulation(P.parse_scenario(config_yaml("cfg3")), diagnostics=False)
for _ in range(2): sim.step()
ds = device_scene(sim.model, sim.system)
n = ctypes.c_int32(0)
_native.check(_native.lib().spb_ctx_trace_cholesky(ds.handle, None, None, ctypes.byref(n)))
tr = np.zeros((n.value, 4), np.uint64); tk = np.zeros((n.value, 2), np.int32)
_native.check(_native.lib().spb_ctx_trace_cholesky(ds.handle, _native.ptr(tr), _native.ptr(tk), ctypes.byref(n)))
T = (tr.astype(np.int64) - int(tr[:, 0].min())) / 1e3
N = tk[:, 1].max() + 1
dur = T[:, 2] - T[:, 0]
i, j = tk[:, 0], tk[:, 1]
kinds = {"regular": (i != j) & (i != j + 1) & (i != N), "partial": (i == j + 1), "rhs": i == N, "diag": i == j}
print(f"total {T[:, 2].max():.1f} us, tasks {len(tk)}")
for name, sel in kinds.items():
    k = np.where(i == j, np.maximum(j - 1, 0), j)[sel].astype(float)
    d = dur[sel]
    A = np.vstack([np.ones_like(k), k]).T
    (a, b), *_ = np.linalg.lstsq(A, d, rcond=None)
    print(f"{name:8s} n={sel.sum():5d}  duration = {a:6.2f} us + {b:5.3f} us x k   (mean {d.mean():7.1f} us)")
busy = dur.sum() / 148
print(f"CTA busy {busy:.1f} us of {T[:, 2].max():.1f}; sum of fixed overheads per CTA ~"
      f"{sum((np.vstack([np.ones(s.sum()), np.zeros(s.sum())]).T @ np.linalg.lstsq(np.vstack([np.ones(s.sum()), np.where(i == j, np.maximum(j - 1, 0), j)[s].astype(float)]).T, dur[s], rcond=None)[0]).sum() for s in kinds.values()) / 148:.1f} us")
