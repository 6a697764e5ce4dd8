"""Scratch: a few exhaustive XR batch solves (ncu target)."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_08797_b200 import planner as P  # noqa: E402
from paper_2603_08797_b200.model import app_from_dict  # noqa: E402
from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace  # noqa: E402
from paper_2603_08797_b200.profiles import profile_from_rows  # noqa: E402

d = json.load(open(os.path.join(ROOT, "tests", "golden", "apps.json")))["ar-assistant"]
app, table = app_from_dict(d["app"]), profile_from_rows(d["profile"])
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reqs = [PlanRequest(240.0 + 7.5 * k, 28, SearchSpace(True, True, True)) for k in range(n)]
P.set_strategy(os.environ.get("JSV_STRATEGY", "exhaustive"), 1 << 40)
for _ in range(int(os.environ.get("REPS", "3"))):
    res = P.plan_batch(app, table, reqs)
print(P.last_stats())
