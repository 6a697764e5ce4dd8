"""Scratch: the configs[3] star DAG at growing task counts through the GPU search."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_08797_b200 import planner as P, workloads
from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace

for n in [int(x) for x in sys.argv[1:]] or range(3, 13):
    app, table = workloads.star(n)
    req = PlanRequest(200.0, 84, SearchSpace(True, True, True))
    t0 = time.perf_counter()
    try:
        r = P.plan(app, table, req)
        st = P.last_stats()
        print(n, f"{(time.perf_counter() - t0) * 1e3:.1f} ms", r.feasible, r.objective,
              r.config.total_slices if r.config else None, {k: st[k] for k in ("ms_stage1", "ms_stage2", "nodes", "leaves", "leaf_work", "exh_probes")}, flush=True)
    except Exception as e:  # noqa: BLE001
        print(n, "ERROR", type(e).__name__, str(e)[:200], flush=True)
