"""Full-size golden vectors by the REFERENCE, for every workload bench.py reports.

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_full.py [bench|md840|day]

* ``bench``: the 64 XR single solves of one bench step (configs[1]; demands
  ``bench.demand_points(64, 0, 1)`` = 240, 247.5, ..., 712.5 rps; 28 slices,
  A+S+T) -> tests/golden/bench_xr64.json;
* ``md840``: configs[4](i), ``max_demand`` of traffic-analysis at 840 slices in
  all 8 spaces -> tests/golden/max_demand_840.json;
* ``day``: configs[4](ii), run_day's planning decisions for EVERY bin of the
  288-bin trace in A+S+T and the three ablations (1,152 plans: plan() at the
  predictor's demand, the memoised max_demand plan when infeasible)
  -> tests/golden/day_traffic_840_full.json.gz.

Independent reference calls run in a process pool over this container's cores
(the reference functions are pure).
"""

from __future__ import annotations

import gzip
import json
import os
import sys
import time
from multiprocessing import Pool
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import make_golden as MG  # noqa: E402

P = MG.P
from sliceserve import workload as RW  # noqa: E402

DAY_SPACES = ("A+S+T", "S+T", "A+T", "A+S")
_state = {}


def _bench_one(demand):
    app, _k, table = _state.setdefault("xr", MG.bundled("ar-assistant"))
    t0 = time.perf_counter()
    r = P.plan(app, table, P.PlanRequest(demand, 28, P.SearchSpace(True, True, True)))
    return {"demand": demand, "result": MG.result_doc(r), "ref_ms": (time.perf_counter() - t0) * 1e3}


def _md840(label):
    app, _k, table = _state.setdefault("traffic", MG.bundled("traffic-analysis"))
    t0 = time.perf_counter()
    r = P.max_demand(app, table, 840, P.SearchSpace.from_label(label))
    return {"name": f"traffic-analysis_840_{label}", "profile_ref": "traffic-analysis",
            "app": MG.app_doc(app), "budget": 840, "space": label, "slack": 0.05, "rel_tol": 1e-3,
            "demand": r.demand_rps, "probes": r.probes, "plan": MG.result_doc(r.plan),
            "ref_ms": (time.perf_counter() - t0) * 1e3}


def _day_one(job):
    label, b, demand = job
    app, _k, table = _state.setdefault("traffic", MG.bundled("traffic-analysis"))
    r = P.plan(app, table, P.PlanRequest(demand, 840, P.SearchSpace.from_label(label), 0.05))
    return label, b, r.feasible, MG.result_doc(r)


def bench() -> None:
    import bench as B

    dem = B.demand_points(64, 0, 1)
    with Pool(os.cpu_count()) as pool:
        rows = pool.map(_bench_one, dem)
    doc = {"app": "ar-assistant", "budget": 28, "space": "A+S+T", "slack": 0.05, "solves": rows}
    (MG.OUT / "bench_xr64.json").write_text(json.dumps(doc))
    print("bench", len(rows), sum(r["ref_ms"] for r in rows) / 1e3, "s of reference CPU")


def md840() -> None:
    with Pool(8) as pool:
        rows = pool.map(_md840, [sp.label for sp in P.ALL_SPACES])
    (MG.OUT / "max_demand_840.json").write_text(json.dumps(rows))
    for r in rows:
        print(r["space"], r["demand"], r["probes"], f"{r['ref_ms'] / 1e3:.1f}s")


def day() -> None:
    t0 = time.perf_counter()
    md = json.loads((MG.OUT / "max_demand_840.json").read_text())
    by = {r["space"]: r for r in md}
    scale = by["A+S+T"]["demand"]
    trace = RW.gen_trace(RW.TraceShape(0.35, 0.65, 0.03, 288), scale, 21)
    preds = []
    st = RW.PredictorState(slack=0.05)
    for _, actual in trace.bins:
        preds.append(RW.predict(st) if st.window else actual * 1.05)
        st.observe(actual)
    jobs = [(label, b, preds[b]) for label in DAY_SPACES for b in range(len(preds))]
    with Pool(os.cpu_count()) as pool:
        rows = pool.map(_day_one, jobs, chunksize=4)
    out = {"app": "traffic-analysis", "budget": 840, "slack": 0.05,
           "shape": [0.35, 0.65, 0.03, 288], "seed": 21, "scale": scale,
           "demands": list(trace.demands), "predicted": preds, "plans": {}}
    for label in DAY_SPACES:
        out["plans"][label] = []
    for label, b, feasible, doc in rows:
        # run_day's memoised fallback = max_demand's final plan (workload.py:268-275),
        # which is exactly md840's plan for that space
        used = not feasible
        out["plans"][label].append({"bin": b, "used_fallback": used,
                                    "plan": by[label]["plan"] if used else doc})
    with gzip.open(MG.OUT / "day_traffic_840_full.json.gz", "wt") as fh:
        json.dump(out, fh)
    print("day", len(rows), f"{time.perf_counter() - t0:.1f}s")


if __name__ == "__main__":
    what = sys.argv[1:] or ["bench", "md840", "day"]
    for w in what:
        {"bench": bench, "md840": md840, "day": day}[w]()
