"""Per elimination-tree level statistics of the supernodal panels (diagnostics, CPU)."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P
from scenes import config_yaml
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
sim = P.Simulation(P.parse_scenario(config_yaml(name)), diagnostics=False)
f = sim.system.factor.native
first, rowptr, rows, parent, level = f.supernodes()
nc = np.diff(first); nr = np.diff(rowptr)
ent = nc.astype(np.int64) * nr
print(f"n1={f.n1} n2={f.n2} supernodes={len(nc)} levels={level.max()+1} panel MB={ent.sum()*8/1e6:.1f}")
print("lvl  nsn   maxnc  max_nr   sum_rows      MB   ctaTasks(32r)  top: nc x nr")
for L in range(level.max() + 1):
    s = np.flatnonzero(level == L)
    k = s[np.argmax(ent[s])]
    print(f"{L:3d} {len(s):5d} {nc[s].max():6d} {nr[s].max():7d} {nr[s].sum():10d} {ent[s].sum()*8/1e6:8.1f} "
          f"{int(np.ceil(nr[s]/32).sum()):8d}     {nc[k]} x {nr[k]}")
