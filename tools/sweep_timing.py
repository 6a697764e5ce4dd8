import os, sys, time
sys.path.insert(0, '/root/repo')
from paper_2603_08797_b200 import planner as P, workloads
from paper_2603_08797_b200.plan_types import SearchSpace
app, table = workloads.xr(); grid = workloads.c3_grid(app); sp = SearchSpace(True, True, True)
P.set_strategy(sys.argv[1])
P.max_demand_grid(grid, table, 28, sp)
print("=====MARK", file=sys.stderr, flush=True)
t0 = time.perf_counter()
P.max_demand_grid(grid, table, 28, sp)
print("wall", (time.perf_counter() - t0) * 1e3, file=sys.stderr)
