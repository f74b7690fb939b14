"""Short programs for `ncu --set full` captures of the non-frame kernels:
  pcg   one device-PCG frame at cfg3 (k_pcg)
  emu   the tile-cyclic factorization of 4 emulated ranks, m = 4096 (k_cholesky_ranks)
  big   one config-4 factorization, m = 12288 (k_cholesky_tiles)"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

what = sys.argv[1]
if what == "pcg":
    import paper_2008_01541_b200 as P
    from paper_2008_01541_b200 import solver as sol
    from scenes import config_yaml

    sim = P.Simulation(P.parse_scenario(config_yaml("cfg3")), diagnostics=False)
    sim.step()
    cfg = sol.SolverConfig(solver_kind="pcg")
    m = sol.solve_frame(sim.model, sim.system, sim.state.copy(), cfg)
    print("pcg iterations", m.pcg_iterations)
else:
    from paper_2008_01541_b200.dense import DenseCholesky

    d = DenseCholesky(4096, nranks=4, emulate=True) if what == "emu" else DenseCholesky(12288)
    d.synthetic()
    print("ms", d.factor(1))
