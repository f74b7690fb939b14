"""Run a few frames of a config through the device context (for ncu / launch lists)."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))

import paper_2008_01541_b200 as P  # noqa: E402
from scenes import config_yaml  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--frames", type=int, default=4)
ap.add_argument("--graph", type=int, default=0)
a = ap.parse_args()
sim = P.Simulation(P.parse_scenario(config_yaml(a.config)), diagnostics=False)
sim.config.use_graph = bool(a.graph)
for _ in range(a.frames):
    m = sim.step()
print("ok", m.active_proxies, m.residual)
