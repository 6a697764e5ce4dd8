"""Scratch: where bench.py's e2e step time goes (profiling on/off, decode share)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes as C
import torch
import bench
from paper_2603_08797_b200 import _native as N, planner as P, _lower as LW
from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace, PlannerOptions

app, table = bench.xr_inputs()
reqs = [PlanRequest(d, 28, SearchSpace(True, True, True)) for d in bench.demand_points(64, 0, 1)]
ctx = N.context(0)
P.set_strategy("exhaustive", 1 << 40, device=0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    P.plan_batch(app, table, reqs, device=0)


def run(prof, steps=20, do_flush=True):
    N.profile(ctx, prof)
    tot = 0.0
    for _ in range(steps):
        if do_flush:
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.plan_batch(app, table, reqs, device=0)
        tot += time.perf_counter() - t0
    N.profile(ctx, False)
    return tot / steps * 1e3


print("e2e ms prof on  flush", run(True))
print("e2e ms prof off flush", run(False))
print("e2e ms prof off noflush", run(False, do_flush=False))
# decode alone
lw, _ = P._prepare(app, table, reqs[0], PlannerOptions(), 0)
probes = (N.Probe * len(reqs))()
for i, r in enumerate(reqs):
    probes[i] = LW.probe_struct(app, lw, r.demand_rps, None)
req, keep = LW.request_struct(lw, reqs[0], PlannerOptions())
outs = (N.PlanOut * len(reqs))()
t0 = time.perf_counter()
for _ in range(20):
    N.check(N.load_library().jsv_plan_batch(lw.ctx, lw.handle, C.byref(req), len(reqs), probes, outs))
t1 = time.perf_counter()
for _ in range(20):
    P._results_from(outs, [app] * len(reqs), lw, reqs, 0.0)
t2 = time.perf_counter()
print("native call ms", (t1 - t0) / 20 * 1e3, "decode ms", (t2 - t1) / 20 * 1e3,
      "device ms", P.last_stats(0)["ms_total"])

# phase split inside plan_batch with the flush, profiling off
import paper_2603_08797_b200.planner as PP
orig_results = PP._results_from
orig_lib = N.load_library()
phase = {"decode": 0.0}


def timed_results(*a, **k):
    t = time.perf_counter()
    r = orig_results(*a, **k)
    phase["decode"] += time.perf_counter() - t
    return r


PP._results_from = timed_results
for label, fl, slp in (("flush", True, 0.0), ("flush+sleep2ms", True, 0.002), ("flush+sleep0.2ms", True, 0.0002), ("noflush", False, 0.0)):
    phase["decode"] = 0.0
    tot = 0.0
    for _ in range(20):
        if fl:
            flush.zero_()
        torch.cuda.synchronize()
        if slp:
            time.sleep(slp)
        t0 = time.perf_counter()
        P.plan_batch(app, table, reqs, device=0)
        tot += time.perf_counter() - t0
    print(label, "e2e ms", tot / 20 * 1e3, "decode ms", phase["decode"] / 20 * 1e3,
          "device ms", P.last_stats(0)["ms_total"])
