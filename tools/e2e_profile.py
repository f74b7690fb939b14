"""Host-side profile of Simulation.step() at a config (diagnostics)."""
import cProfile, pstats, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P
from scenes import config_yaml
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
sim = P.Simulation(P.parse_scenario(config_yaml(name)), diagnostics=False)
for _ in range(5): sim.step()
t = time.perf_counter()
for _ in range(50): sim.step()
print(f"e2e {(time.perf_counter() - t) / 50 * 1e3:.3f} ms/frame")
pr = cProfile.Profile(); pr.enable()
for _ in range(50): sim.step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
