"""Host-side split of Simulation.step at one config: the C frame call
(spb_ctx_frame) against the Python around it (diagnostics)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2008_01541_b200 as P  # noqa: E402
from paper_2008_01541_b200 import _native  # noqa: E402
from scenes import config_yaml  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
sim = P.Simulation(P.parse_scenario(config_yaml(cfg)), diagnostics=False)
for _ in range(5):
    sim.step()
lib = _native.lib()
orig = lib.spb_ctx_frame
acc = {"c": 0.0}


def timed(*a):
    t0 = time.perf_counter()
    r = orig(*a)
    acc["c"] += time.perf_counter() - t0
    return r


lib.spb_ctx_frame = timed
F = 200
tp = 0.0
t = time.perf_counter()
for _ in range(F):
    t1 = time.perf_counter()
    sim.frame += 1
    sim.pose(sim.frame)
    tp += time.perf_counter() - t1
    P.solve_frame(sim.model, sim.system, sim.state, sim.config)
tot = time.perf_counter() - t
print(f"{cfg}: step {1e3 * tot / F:.3f} ms = pose {1e3 * tp / F:.3f} + C frame call {1e3 * acc['c'] / F:.3f} "
      f"+ other Python {1e3 * (tot - tp - acc['c']) / F:.3f}")
