"""Scratch: device time of search vs exhaustive Stage 2 on the bench workloads."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_08797_b200 import _native as N  # noqa: E402
from paper_2603_08797_b200 import planner as P  # noqa: E402
from paper_2603_08797_b200.model import app_from_dict  # noqa: E402
from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace  # noqa: E402
from paper_2603_08797_b200.profiles import profile_from_rows  # noqa: E402

apps = json.load(open(os.path.join(ROOT, "tests", "golden", "apps.json")))
FULL = SearchSpace(True, True, True)


def load(name):
    d = apps[name]
    return app_from_dict(d["app"]), profile_from_rows(d["profile"])


ctx = N.context()
for name, dems, bud in (("ar-assistant", [480.0], 28),
                        ("ar-assistant", [240.0 + 7.5 * k for k in range(64)], 28),
                        ("social-media", [600.0], 28),
                        ("traffic-analysis", [400.0], 28),
                        ("traffic-analysis", [9000.0], 840)):
    app, table = load(name)
    reqs = [PlanRequest(d, bud, FULL) for d in dems]
    ref = None
    for strat in ("search", "exhaustive"):
        P.set_strategy(strat, 1 << 40)
        for _ in range(3):
            res = P.plan_batch(app, table, reqs)
        N.profile(ctx, True)
        ms = []
        for _ in range(5):
            res = P.plan_batch(app, table, reqs)
            ms.append(P.last_stats()["ms_total"])
        kt = {k: round(v[0] / 5, 4) for k, v in N.kernel_times(ctx).items() if v[1]}
        N.profile(ctx, False)
        st = P.last_stats()
        key = [(r.feasible, r.objective, r.config.m if r.config else None) for r in res]
        if ref is None:
            ref = key
        same = key == ref
        print(f"{name} n={len(dems)} S={bud} {strat:10s} ms={min(ms):.3f} s1={st['ms_stage1']:.3f} "
              f"s2={st['ms_stage2']:.3f} exh_cand={st['exh_candidates']} leaves={st['leaves']} "
              f"same={same} kt={kt}", flush=True)
P.set_strategy("search")
