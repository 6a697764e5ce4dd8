"""Golden vectors for configs[4] (traffic-analysis, 840 slices) by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_day.py

* the demand trace: gen_trace(TraceShape(0.35, 0.65, 0.03, 288), scale = the
  A+S+T max-serviceable demand at 840 slices, seed 21) -- all 288 bins;
* run_day's planning decisions without the simulator (no measured fan-out
  history): plan() at the reference predictor's demand for a subset of bins,
  falling back to max_demand()'s plan when infeasible, for A+S+T and the three
  ablations S+T (no accuracy scaling), A+T (no partitioning), A+S (no task-graph
  budgeting -> plan_uninformed).
Writes tests/golden/day_traffic_840.json.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as MG  # noqa: E402

P = MG.P
from sliceserve import workload as RW  # noqa: E402

BINS = list(range(0, 24)) + list(range(136, 148))
SPACES = ("A+S+T", "S+T", "A+T", "A+S")


def main() -> None:
    app, _knobs, table = MG.bundled("traffic-analysis")
    t0 = time.perf_counter()
    md = P.max_demand(app, table, 840, P.SearchSpace(True, True, True))
    print("max_demand", md.demand_rps, f"{time.perf_counter() - t0:.1f}s", flush=True)
    shape = RW.TraceShape(0.35, 0.65, 0.03, 288)
    trace = RW.gen_trace(shape, md.demand_rps, 21)
    preds = []
    st = RW.PredictorState(slack=0.05)
    for _, actual in trace.bins:
        preds.append(RW.predict(st) if st.window else actual * 1.05)
        st.observe(actual)
    out = {"app": "traffic-analysis", "budget": 840, "slack": 0.05,
           "shape": [0.35, 0.65, 0.03, 288], "seed": 21, "scale": md.demand_rps,
           "demands": list(trace.demands), "predicted": preds, "bins": BINS, "plans": {}}
    for label in SPACES:
        sp = P.SearchSpace.from_label(label)
        fallback = None
        rows = []
        for b in BINS:
            t1 = time.perf_counter()
            r = P.plan(app, table, P.PlanRequest(preds[b], 840, sp, 0.05))
            used = False
            if not r.feasible:
                if fallback is None:
                    fallback = P.max_demand(app, table, 840, sp, 0.05).plan
                r, used = fallback, True
            rows.append({"bin": b, "used_fallback": used, "plan": MG.result_doc(r),
                         "ref_ms": (time.perf_counter() - t1) * 1e3})
        out["plans"][label] = rows
        print(label, f"{time.perf_counter() - t0:.1f}s", flush=True)
        (MG.OUT / "day_traffic_840.json").write_text(json.dumps(out))


if __name__ == "__main__":
    main()
