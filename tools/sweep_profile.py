"""Scratch: where the configs[2] sweep (64 max_demand points) spends its time."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_08797_b200 import _native as N, planner as P, workloads
from paper_2603_08797_b200.plan_types import SearchSpace
import ctypes as C

app, table = workloads.xr()
grid = workloads.c3_grid(app)
sp = SearchSpace(True, True, True)
P.max_demand_grid(grid, table, 28, sp)
ctx = N.context()
for strat in ("auto", "search"):
    P.set_strategy(strat)
    N.profile(ctx, True)
    t0 = time.perf_counter()
    res = P.max_demand_grid(grid, table, 28, sp)
    wall = (time.perf_counter() - t0) * 1e3
    kt = {k: round(v[0], 2) for k, v in N.kernel_times(ctx).items() if v[1]}
    cnt = {k: v[1] for k, v in N.kernel_times(ctx).items() if v[1]}
    N.profile(ctx, False)
    print(strat, f"wall {wall:.1f} ms", "stats", P.last_stats())
    print("  kernel ms", kt)
    print("  launches", cnt)
P.set_strategy("auto")
