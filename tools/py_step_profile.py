import cProfile, pstats, sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_2008_01541_b200 as P
from scenes import config_yaml
sim = P.Simulation(P.parse_scenario(config_yaml("cfg2")), diagnostics=False)
for _ in range(10): sim.step()
pr = cProfile.Profile()
pr.enable()
for _ in range(300): sim.step()
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(25)
