"""Scratch timing of the GPU planner on the bundled configs (not the bench contract)."""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_08797_b200 import planner as P  # noqa: E402
from paper_2603_08797_b200.model import app_from_dict  # noqa: E402
from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace  # noqa: E402
from paper_2603_08797_b200.profiles import profile_from_rows  # noqa: E402

apps = json.load(open(os.path.join(ROOT, "tests", "golden", "apps.json")))


def load(name):
    d = apps[name]
    return app_from_dict(d["app"]), profile_from_rows(d["profile"])


FULL = SearchSpace(True, True, True)
for name, dem, bud in (("ar-assistant", 480.0, 28), ("social-media", 600.0, 28),
                       ("traffic-analysis", 400.0, 28), ("traffic-analysis", 9000.0, 840)):
    app, table = load(name)
    req = PlanRequest(dem, bud, FULL)
    for i in range(6):
        t0 = time.perf_counter()
        r = P.plan(app, table, req)
        ms = (time.perf_counter() - t0) * 1e3
        print(name, dem, bud, f"{ms:.2f} ms", r.objective, P.last_stats(), flush=True)

app, table = load("ar-assistant")
for i in range(2):
    t0 = time.perf_counter()
    r = P.max_demand(app, table, 28, FULL)
    print("max_demand xr", r.demand_rps, r.probes, f"{(time.perf_counter() - t0) * 1e3:.1f} ms",
          P.last_stats(), flush=True)
