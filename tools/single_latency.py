"""Single-solve latency: one XR plan() at 240 / 480 / 700 rps, 28 slices,
A+S+T, under the auto and exhaustive strategies; median wall (perf_counter around the
public call) and libjsv's device times (total, Stage 1, Stage 2) over 15 calls."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
from paper_2603_08797_b200 import planner as P  # noqa: E402
from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace  # noqa: E402

app, table = bench.xr_inputs()
sp = SearchSpace(True, True, True)
for strat in ("auto", "exhaustive"):
    P.set_strategy(strat, 1 << 40)
    for dem in (240.0, 480.0, 700.0):
        one = PlanRequest(dem, 28, sp)
        for _ in range(5):
            P.plan(app, table, one)
        w, d, s1, s2 = [], [], [], []
        for _ in range(15):
            t0 = time.perf_counter()
            P.plan(app, table, one)
            w.append((time.perf_counter() - t0) * 1e3)
            st = P.last_stats()
            d.append(st["ms_total"])
            s1.append(st["ms_stage1"])
            s2.append(st["ms_stage2"])
        m = statistics.median
        print(strat, dem, "wall %.3f dev %.3f s1 %.3f s2 %.3f" % (m(w), m(d), m(s1), m(s2)), flush=True)
P.set_strategy("auto")
