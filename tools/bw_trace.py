"""Anatomy of one dense backward solve (u = L^-T y) per 64-row block (diagnostics)."""
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
_native.check(_native.lib().spb_ctx_trace_dense_backward(ds.handle, None, ctypes.byref(n)))
tr = np.zeros((n.value, 5), np.uint64)
_native.check(_native.lib().spb_ctx_trace_dense_backward(ds.handle, _native.ptr(tr), ctypes.byref(n)))
T = (tr.astype(np.int64) - int(tr[:, 0].min())) / 1e3
N = n.value
# block b handles j = N-1-b
j = N - 1 - np.arange(N)
order = np.argsort(-j)  # j descending = chain order
done = T[:, 4]
print(f"total {done.max():.1f} us, blocks {N}; kernel start spread {T[:,0].max():.1f} us")
rows = []
for b in range(1, N):
    # x_{j+1} stored by block b-1 at done[b-1]; block b receives it at T[b,3]
    comm = T[b, 3] - done[b - 1]
    comp = done[b] - T[b, 3]
    lag = T[b, 2] - done[b - 1]  # >0: c_j not ready when x_{j+1} was published
    rows.append((comm, comp, lag, done[b] - done[b - 1]))
r = np.array(rows)
print("mean per step: comm %.2f us, compute %.2f us, c_j-lag %.2f us (positive share %.0f%%), step %.2f us"
      % (r[:, 0].mean(), r[:, 1].mean(), np.maximum(r[:, 2], 0).mean(), 100 * (r[:, 2] > 0).mean(), r[:, 3].mean()))
for b in range(0, N, 12):
    print(f"b={b:3d} start {T[b,0]:7.1f} accdone {T[b,1]:7.1f} cj {T[b,2]:7.1f} recv {T[b,3]:7.1f} done {T[b,4]:7.1f}")
