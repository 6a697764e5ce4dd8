"""Scratch: where the host time of plan_batch goes (64 XR solves)."""
import cProfile, os, pstats, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_08797_b200 import planner as P, workloads
from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace
app, table = workloads.xr()
reqs = [PlanRequest(240.0 + 7.5 * k, 28, SearchSpace(True, True, True)) for k in range(64)]
for _ in range(3):
    P.plan_batch(app, table, reqs)
t0 = time.perf_counter()
for _ in range(10):
    P.plan_batch(app, table, reqs)
print("wall ms per batch", (time.perf_counter() - t0) * 100, "device", P.last_stats()["ms_total"])
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    P.plan_batch(app, table, reqs)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
