"""Factor a config's sigma0 with the device tile kernel (dense op) repeatedly and
compare tile-by-tile with numpy (diagnostics for the tile Cholesky)."""
import os, sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P
from scenes import config_yaml
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sim = P.Simulation(P.parse_scenario(config_yaml(cfg)), diagnostics=False)
H = sim.system.factor.sigma0
t = time.time(); ref = np.linalg.cholesky(H); print("numpy chol", time.time() - t)
m = H.shape[0]; N = (m + 63) // 64
for rep in range(reps):
    try:
        L = P.dense_factor(H).chol
    except Exception as e:
        print("rep", rep, "ERROR", e); continue
    err = np.abs(L - ref)
    bad = []
    for i in range(N):
        for j in range(i + 1):
            e = err[i*64:(i+1)*64, j*64:(j+1)*64].max()
            if e > 1e-8 * np.abs(ref).max():
                bad.append((i, j, float(e)))
    print("rep", rep, "max err", err.max() / np.abs(ref).max(), "bad tiles", len(bad), bad[:8])
