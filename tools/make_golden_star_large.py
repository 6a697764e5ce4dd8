"""configs[3] goldens beyond the reference's reach, by the independent exact star solver.

    python tools/make_golden_star_large.py

The reference's depth-first search does not finish the 12-task star (SURVEY.md
a12), so the 8-, 10- and 12-task stars of workloads.star are solved by
oracle/star_oracle.py (restated reference Stage 1 + per-entry-bundle knapsack DP
+ exact derive/validate of every near-optimal class vector; the oracle itself
is pinned to the reference on the 3..7-task ladder by tests/test_oracle_golden.py).
Writes tests/golden/plans_star_large.json (serialised like the other goldens).
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import star_oracle as SO  # noqa: E402
from paper_2603_08797_b200 import workloads  # noqa: E402
from paper_2603_08797_b200.plan_types import (  # noqa: E402
    PlannerOptions, PlanRequest, SearchSpace, plan_result_to_dict,
)


def main() -> None:
    out = []
    for n in (8, 10, 12):
        app, table = workloads.star(n)
        req = PlanRequest(200.0, 84, SearchSpace(True, True, True))
        t0 = time.perf_counter()
        res = SO.star_plan(app, table, req)
        d = plan_result_to_dict(res)
        d["stats"].pop("nodes")
        out.append({"name": f"star_{n}", "n_tasks": n, "request": {"demand": 200.0, "budget": 84,
                    "space": "A+S+T", "slack": 0.05, "overrides": None},
                    "options": {"pareto_width": 512, "exhaustive_limit": 2000, "eps": 1e-9,
                                "mix_fractions": [0.25, 0.5, 0.75], "feasible_only": False},
                    "result": d, "oracle_s": time.perf_counter() - t0})
        print(n, res.objective, res.config.total_slices, f"{out[-1]['oracle_s']:.1f}s", flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "plans_star_large.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
