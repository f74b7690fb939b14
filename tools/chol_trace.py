"""Trace one tile-Cholesky launch of a config's H and print the critical-path
anatomy per column (diagnostics)."""
import ctypes, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import _native
from paper_2008_01541_b200.solver import device_scene
from scenes import config_yaml
sim = P.Simulation(P.parse_scenario(config_yaml(sys.argv[1] if len(sys.argv) > 1 else "cfg3")), diagnostics=False)
for _ in range(2): sim.step()
ds = device_scene(sim.model, sim.system)
n = ctypes.c_int32(0)
_native.check(_native.lib().spb_ctx_trace_cholesky(ds.handle, None, None, ctypes.byref(n)))
nt = n.value
tr = np.zeros((nt, 4), dtype=np.uint64); tk = np.zeros((nt, 2), dtype=np.int32)
_native.check(_native.lib().spb_ctx_trace_cholesky(ds.handle, _native.ptr(tr), _native.ptr(tk), ctypes.byref(n)))
t0 = tr[:, 0].min()
T = (tr[:, :4].astype(np.int64) - int(t0)) / 1e3  # us
N = tk[:, 1].max() + 1
done = {}; kd = {}; cl = {}
for (i, j), row in zip(tk, T):
    done[(i, j)] = row[2]; kd[(i, j)] = row[1]; cl[(i, j)] = row[0]
print(f"total {T[:, 2].max():.1f} us, tasks {nt}, N {N}")
fin = {(i, j): row[3] for (i, j), row in zip(tk, T)}
pc = [fin[(j, j)] - kd[(j, j)] for j in range(N)]
tail = [done[(j, j)] - fin[(j, j)] for j in range(N)]
print("diag: compute (kdone->fin) mean %.2f us, tail (fin->released) mean %.2f us" % (np.mean(pc), np.mean(tail)))
offt = [row[2] - row[3] for (i, j), row in zip(tk, T) if i != j]
print("offdiag tail mean %.2f us" % np.mean(offt))
print(" j  claim  kdone  fdone | potrf  gap(diag j -> potrf j+1)  kdone-after-partial")
rows = []
for j in range(N):
    pot = done[(j, j)] - kd[(j, j)]
    # gap: diag j-1 released -> diag j starts its factorization (includes the
    # sub-diagonal finalize + rank-64 update done inside diag task j)
    trsm = kd[(j + 1, j + 1)] - done[(j, j)] if (j + 1, j + 1) in kd else float("nan")
    wait = kd[(j, j)] - done.get((j, j - 1), float("nan")) if j > 0 else float("nan")
    rows.append((pot, trsm, wait))
    if j % 8 == 0 or j == N - 1:
        print(f"{j:3d} {cl[(j,j)]:7.1f} {kd[(j,j)]:7.1f} {done[(j,j)]:7.1f} | {pot:6.2f} {trsm:8.2f} {wait:10.2f}")
r = np.array(rows)
print("mean potrf %.2f  trsm-after-diag %.2f  diag-lastk-after-(j,j-1) %.2f us" % tuple(np.nanmean(r, axis=0)))
busy = (T[:, 2] - T[:, 0]).sum() / 148
print(f"mean CTA busy (claim->done) {busy:.1f} us of {T[:,2].max():.1f}")
