import sys, time
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import paper_2008_01541_b200 as P
from paper_2008_01541_b200 import linalg, solver
from scenes import config_yaml
import cProfile, pstats
sc=P.parse_scenario(config_yaml("cfg3"))
pr=cProfile.Profile(); pr.enable()
t=time.perf_counter()
sim=P.Simulation(sc, diagnostics=False)
print("setup", time.perf_counter()-t)
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(12)
