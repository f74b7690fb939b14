"""Per-task anatomy of one traced tile-Cholesky launch (diagnostics):
k-loop phase (claim -> k-loop done), finalize phase (k-loop done -> finalize
done), by task kind, and the column chain (diagonal release times).

    python tools/chol_trace2.py [cfg3] [SPB_CHOL_INT8=0|1 via env]"""
import ctypes
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P  # noqa: E402
from paper_2008_01541_b200 import _native  # noqa: E402
from paper_2008_01541_b200.solver import device_scene  # noqa: E402
from scenes import config_yaml  # noqa: E402

sim = P.Simulation(P.parse_scenario(config_yaml(sys.argv[1] if len(sys.argv) > 1 else "cfg3")), diagnostics=False)
for _ in range(3):
    sim.step()
ds = device_scene(sim.model, sim.system)
n = ctypes.c_int32(0)
_native.check(_native.lib().spb_ctx_trace_cholesky(ds.handle, None, None, ctypes.byref(n)))
nt = n.value
best = None
for rep in range(3):
    tr = np.zeros((nt, 4), dtype=np.uint64)
    tk = np.zeros((nt, 2), dtype=np.int32)
    _native.check(_native.lib().spb_ctx_trace_cholesky(ds.handle, _native.ptr(tr), _native.ptr(tk), ctypes.byref(n)))
    span = (tr[:, 2].max() - tr[:, 0].min()) / 1e3
    if best is None or span < best[0]:
        best = (span, tr.copy(), tk.copy())
span, tr, tk = best
t0 = tr[:, 0].min()
T = (tr.astype(np.int64) - int(t0)) / 1e3  # claim, kdone, released, fin (us)
N = int(tk[:, 1].max()) + 1
kind = np.where(tk[:, 0] == N, "rhs", np.where(tk[:, 0] == tk[:, 1], "diag",
                np.where(tk[:, 0] == tk[:, 1] + 1, "partial", "regular")))
print(f"span {span:.1f} us, tasks {nt}, N {N}")
for k in ("regular", "partial", "diag", "rhs"):
    m = kind == k
    if not m.any():
        continue
    kl = T[m, 1] - T[m, 0]
    fz = T[m, 3] - T[m, 1]
    rel = T[m, 2] - T[m, 3]
    j = tk[m, 1].astype(float)
    print(f"{k:8s} n={m.sum():5d} k-loop phase {kl.mean():7.2f} us (per k-step {np.sum(kl) / max(np.sum(j), 1):.2f}) "
          f"finalize {fz.mean():6.2f} release {rel.mean():5.2f}")
busy = (T[:, 2] - T[:, 0]).sum() / 148
print(f"mean CTA busy {busy:.1f} us of {span:.1f} ({100 * busy / span:.0f}%)")
diag = {int(j): T[q] for q, (i, j) in enumerate(tk) if i == j}
rel = np.array([diag[j][3] for j in range(N)])  # factorization done (the diagonal flag is released inside it)
print("diagonal released at (us): " + " ".join(f"{j}:{rel[j]:.0f}" for j in range(0, N, max(1, N // 12))))
step = np.diff(rel)
print(f"chain step mean {step.mean():.2f} us; first 20 cols {step[:20].mean():.2f}, last 15 {step[-15:].mean():.2f}")
pre = np.array([diag[j][1] - diag[j - 1][3] for j in range(1, N)])
pot = np.array([diag[j][3] - diag[j][1] for j in range(N)])
print(f"diag j: kdone - fin(j-1) mean {pre.mean():.2f} us (LinvT hop + partial finalize), potrf (kdone -> fin) mean {pot.mean():.2f} us")
# the partial (j+1, j): when it finished relative to diag j's factorization
pj = {int(j): T[q] for q, (i, j) in enumerate(tk) if i == j + 1 and i != N}
lag = np.array([pj[j][2] - diag[j][3] for j in range(N - 1) if j in pj])
print(f"partial (j+1, j) released after fin(j): mean {lag.mean():.2f} us, max {lag.max():.2f}")
for j in list(range(0, 4)) + list(range(N - 4, N)):
    c, kd, r, f = diag[j]
    print(f"  diag {j:3d}: claim {c:8.1f} kdone {kd:8.1f} fin {f:8.1f} rel {r:8.1f}")
print(" j | partial(j+1,j): claim  kdone  fin  rel | diag j fin | diag j+1 kdone")
for j in list(range(1, 6)) + list(range(40, 46)) + list(range(N - 6, N - 1)):
    if j not in pj or (j + 1) not in diag:
        continue
    c, kd, r, f = pj[j]
    print(f"{j:3d} | {c:8.1f} {kd:8.1f} {f:8.1f} {r:8.1f} | {diag[j][3]:8.1f} | {diag[j + 1][1]:8.1f}")
allt = {(int(i), int(j)): T[q] for q, (i, j) in enumerate(tk)}
print(" j | reg (j+1,j-1): claim kdone fin rel | diag j kdone | partial(j+1,j) claim kdone rel | fin(j-1)")
for j in list(range(2, 7)) + list(range(40, 44)):
    r = allt.get((j + 1, j - 1))
    p_ = allt.get((j + 1, j))
    if r is None or p_ is None:
        continue
    print(f"{j:3d} | {r[0]:7.1f} {r[1]:7.1f} {r[3]:7.1f} {r[2]:7.1f} | {diag[j][1]:7.1f} | {p_[0]:7.1f} {p_[1]:7.1f} "
          f"{p_[2]:7.1f} | {diag[j - 1][3]:7.1f}")
