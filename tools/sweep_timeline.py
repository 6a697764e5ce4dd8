"""Scratch: configs[2] sweep round structure (JSV_TIMING=1 host timeline on stderr)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_2603_08797_b200 import planner as P
from paper_2603_08797_b200.plan_types import SearchSpace
app, table = bench.xr_inputs()
grid = bench.c3_apps(app)
space = SearchSpace(True, True, True)
P.max_demand_grid(grid, table, 28, space)
for _ in range(2):
    t0 = time.perf_counter()
    r = P.max_demand_grid(grid, table, 28, space)
    print("sweep ms", (time.perf_counter() - t0) * 1e3, "probes", sum(x.probes for x in r), file=sys.stderr)
