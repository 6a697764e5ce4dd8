"""Run one bundled plan and print the raw native result (debug helper)."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_08797_b200 import planner as P  # noqa: E402
from paper_2603_08797_b200.model import app_from_dict  # noqa: E402
from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace  # noqa: E402
from paper_2603_08797_b200.profiles import profile_from_rows  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ar-assistant"
dem = float(sys.argv[2]) if len(sys.argv) > 2 else 480.0
bud = int(sys.argv[3]) if len(sys.argv) > 3 else 28
d = json.load(open(os.path.join(ROOT, "tests", "golden", "apps.json")))[name]
app, table = app_from_dict(d["app"]), profile_from_rows(d["profile"])
r = P.plan(app, table, PlanRequest(dem, bud, SearchSpace(True, True, True)))
print(r.feasible, r.objective, r.binding_constraint, r.stats)
print(P.last_stats())
