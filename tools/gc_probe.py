"""Scratch: plan_batch wall time with the cyclic GC enabled vs disabled (64 XR solves)."""
import gc, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2603_08797_b200 import planner as P
from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace
app, table = bench.xr_inputs()
reqs = [PlanRequest(d, 28, SearchSpace(True, True, True)) for d in bench.demand_points(64, 0, 1)]
P.set_strategy("exhaustive", 1 << 40, device=0)
for _ in range(6):
    P.plan_batch(app, table, reqs, device=0)
for label in ("gc on", "gc off", "gc on", "gc off", "gc on discard", "gc off discard", "gc on discard", "gc off discard"):
    (gc.disable if label.startswith("gc off") else gc.enable)()
    keep = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        r = P.plan_batch(app, table, reqs, device=0)
        if "discard" not in label:
            keep.append(r)
    dt = (time.perf_counter() - t0) / 50 * 1e3
    print(label, round(dt, 4), "ms per batch")
gc.enable()
