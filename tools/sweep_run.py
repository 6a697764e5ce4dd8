"""configs[2] sweep for the launch list (tools/profile_round.sh): the 64-point XR SLO grid
through max_demand_grid (one warm-up, three timed passes, one pass with per-kernel
events); prints wall time, points/s, probe counts and the per-kernel device split."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
from paper_2603_08797_b200 import _native as N  # noqa: E402
from paper_2603_08797_b200 import planner as P  # noqa: E402
from paper_2603_08797_b200.plan_types import SearchSpace  # noqa: E402

app, table = bench.xr_inputs()
sp = SearchSpace(True, True, True)
grid = bench.c3_apps(app)
P.max_demand_grid(grid, table, 28, sp)
w = []
for _ in range(3):
    t0 = time.perf_counter()
    res = P.max_demand_grid(grid, table, 28, sp)
    w.append((time.perf_counter() - t0) * 1e3)
print("wall ms", min(w), "points/s", 64 / (min(w) / 1e3), "probes", sum(r.probes for r in res),
      P.last_demand_stats())
ctx = N.context(None)
N.profile(ctx, True)
N.kernel_times(ctx)
P.max_demand_grid(grid, table, 28, sp)
print({k: v for k, v in N.kernel_times(ctx).items() if v[1]})
N.profile(ctx, False)
