import sys, time
sys.path.insert(0, "/root/repo")
from paper_2603_08797_b200 import planner as P, workloads, _native as N
from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace
app, table = workloads.star(12)
req = PlanRequest(200.0, 84, SearchSpace(True, True, True))
for _ in range(3): P.plan(app, table, req)
ctx = N.context(None)
N.profile(ctx, True)
for _ in range(5): P.plan(app, table, req)
kt = N.kernel_times(ctx); N.profile(ctx, False)
print("ms_total", P.last_stats()["ms_total"])
for k, (ms, c) in sorted(kt.items(), key=lambda kv: -kv[1][0]):
    if c: print(f"{k:12s} {ms/5:8.3f} ms/solve  launches {c/5:.0f}")
