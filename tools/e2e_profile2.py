"""cProfile of Simulation.step at one config (host overhead around the one
C-ABI frame call): python tools/e2e_profile2.py [cfg3] [frames]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P  # noqa: E402
from scenes import config_yaml  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
F = int(sys.argv[2]) if len(sys.argv) > 2 else 100
sim = P.Simulation(P.parse_scenario(config_yaml(cfg)), diagnostics=False)
for _ in range(5):
    sim.step()
t = time.perf_counter()
for _ in range(F):
    sim.step()
print(f"Simulation.step {1e3 * (time.perf_counter() - t) / F:.3f} ms/frame")
pr = cProfile.Profile()
pr.enable()
for _ in range(F):
    sim.step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
