"""Scratch: feasibility of plan(feasible_only) around a max_demand disagreement."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_io import load, profile_of
from paper_2603_08797_b200 import planner as P
from paper_2603_08797_b200.model import app_from_dict
from paper_2603_08797_b200.plan_types import PlannerOptions, PlanRequest, SearchSpace

doc = [d for d in load("max_demand.json") if d["name"] == sys.argv[1]][0]
app = app_from_dict(doc["app"]); table = profile_of(doc)
sp = SearchSpace.from_label(doc["space"])
opt = PlannerOptions(feasible_only=True)
dems = [600 + 2 * k for k in range(30)]
for strat in ("search", "exhaustive"):
    P.set_strategy(strat, 1 << 32)
    res = P.plan_batch(app, table, [PlanRequest(d, doc["budget"], sp, doc["slack"]) for d in dems], opt)
    print(strat, "".join("1" if r.feasible else "0" for r in res))
    res1 = [P.plan(app, table, PlanRequest(d, doc["budget"], sp, doc["slack"]), opt) for d in dems]
    print(strat, "".join("1" if r.feasible else "0" for r in res1), "(single)")
    print(P.last_stats())
P.set_strategy("exhaustive", 1 << 32)
res = P.plan_batch(app, table, [PlanRequest(d, doc["budget"], sp, doc["slack"]) for d in dems], opt)
print([r.stats.pool_sizes for r in res][::6])
for sub in (dems[6:9], dems[7:], [dems[0], dems[10]], [dems[10], dems[0]]):
    res = P.plan_batch(app, table, [PlanRequest(d, doc["budget"], sp, doc["slack"]) for d in sub], opt)
    print(sub, "".join("1" if r.feasible else "0" for r in res))
