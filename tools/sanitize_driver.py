"""One pass over every libjsv kernel family, checked against the reference goldens,
for compute-sanitizer (memcheck / racecheck / synccheck; tools/sanitize.sh).

Kernel families exercised: fused and legacy Stage 1 (k_s1_job; k_generate ..
k_truncate), the exhaustive Stage 2 (k_x_rank, k_m_rank, k_x_live, k_x_sched,
k_s2_exh register and looped sweeps, the float evaluator, k_s2_xreduce), the
level-synchronous branch-and-bound (k_s2_prefix/level/leaf/reduce/blocked), the
fan-out solver (k_fo_*), plan_uninformed (k_uni_pick), finalize, derive/validate,
brute_force_plan, max_demand's feasibility probes, the bench batch (the Stage-1 LPT
job map) and the best-first split of branch-and-bound frontiers.  Small cases only: the
sanitizers slow kernels down 10-100x.  Exit status 1 on any golden mismatch."""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from golden_io import app_from_dict, case_inputs, load, profile_of, result_dict  # noqa: E402


def main() -> int:
    from paper_2603_08797_b200 import planner as P
    from paper_2603_08797_b200.plan_types import SearchSpace

    bad = 0
    docs = load("plans_bundled.json")[::12] + load("plans_tiny.json")[:3] + load("plans_star.json")[:2]
    for strat in ("exhaustive", "search", "auto"):
        P.set_strategy(strat, 1 << 32)
        for doc in docs:
            app, table, req, opt = case_inputs(doc)
            if result_dict(P.plan(app, table, req, opt)) != doc["result"]:
                print("MISMATCH", strat, doc["name"])
                bad += 1
    # the bench batch (64 XR solves = 192 Stage-1 jobs: the LPT job map) and the
    # branch-and-bound with split frontiers (best-first sorts of the halves)
    from paper_2603_08797_b200 import workloads
    from paper_2603_08797_b200.plan_types import PlanRequest

    P.set_strategy("exhaustive", 1 << 32)
    app, table = workloads.xr()
    rows = load("bench_xr64.json")["solves"]
    got = P.plan_batch(app, table, [PlanRequest(r["demand"], 28, SearchSpace(True, True, True))
                                    for r in rows])
    for r, res in zip(rows, got):
        if result_dict(res) != r["result"]:
            print("MISMATCH bench", r["demand"])
            bad += 1
    P.set_strategy("search")
    os.environ["JSV_BB_MAX_SLOTS"] = "64"
    for doc in docs[:4]:
        app, table, req, opt = case_inputs(doc)
        if result_dict(P.plan(app, table, req, opt)) != doc["result"]:
            print("MISMATCH split", doc["name"])
            bad += 1
    del os.environ["JSV_BB_MAX_SLOTS"]
    P.set_strategy("auto")
    for doc in load("max_demand.json")[:2]:
        app = app_from_dict(doc["app"])
        r = P.max_demand(app, profile_of(doc), doc["budget"], SearchSpace.from_label(doc["space"]),
                         doc["slack"], None, doc["rel_tol"])
        if r.demand_rps != doc["demand"]:
            print("MISMATCH max_demand", doc["name"])
            bad += 1
    print("sanitize driver:", "ok" if not bad else f"{bad} mismatches",
          "env", {k: v for k, v in os.environ.items() if k.startswith("JSV_")})
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
