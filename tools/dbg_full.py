import faulthandler, sys, time
faulthandler.dump_traceback_later(150, exit=True)
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import paper_2008_01541_b200 as P
from scenes import config_yaml
t=time.time()
def log(*a): print(f"[{time.time()-t:7.1f}]", *a, flush=True)
sim = P.Simulation(P.parse_scenario(config_yaml("cfg3")), diagnostics=False); log("sim")
for _ in range(4): met = sim.step()
log("steps", met.active_proxies)
f = sim.system.factor
rng = np.random.default_rng(3)
b1 = rng.normal(size=(f.n1, 3)); b2 = rng.normal(size=(f.n2, 3))
y1, ft2 = P.forward_sub(f, b1, b2); log("fw")
s0 = np.asarray(f.sigma0); log("sigma0")
df = P.dense_factor(s0); log("dense_factor")
x2 = P.dense_solve(df, ft2); log("dense_solve")
x1 = P.backward_sub(f, y1, x2); log("bw")
A = sim.system.A.full(); x = np.concatenate([x1, x2]); b = np.concatenate([b1, b2])
log("resid", np.linalg.norm(A @ x - b) / np.linalg.norm(b))
