"""Time the device PCG baseline against the Schur path on one config:
python tools/pcg_probe.py [cfg2|cfg3] [frames]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))

import paper_2008_01541_b200 as P  # noqa: E402
from scenes import config_yaml  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4
text = config_yaml(cfg)
for kind in ("schur", "pcg"):
    sim = P.Simulation(P.parse_scenario(text.replace("kind: schur", f"kind: {kind}")), diagnostics=False)
    sim.step()
    t = []
    for _ in range(frames):
        t0 = time.perf_counter()
        m = sim.step()
        t.append(time.perf_counter() - t0)
    print(f"{cfg} {kind}: {1e3 * min(t):.2f} ms/frame (min of {frames}), pcg_iterations={m.pcg_iterations}, "
          f"active={m.active_proxies}, residual={m.residual:.3e}", flush=True)
