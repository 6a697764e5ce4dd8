import cProfile, pstats, time, sys, os
sys.path.insert(0, os.getcwd())
import bench
from paper_2603_08797_b200 import planner as P
from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace
app, table = bench.xr_inputs()
reqs = [PlanRequest(d, 28, SearchSpace(True, True, True)) for d in bench.demand_points(64, 0, 1)]
P.set_strategy("exhaustive", 1 << 40, device=0)
for _ in range(6): P.plan_batch(app, table, reqs, device=0)
pr = cProfile.Profile()
pr.enable()
for _ in range(50): P.plan_batch(app, table, reqs, device=0)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
