#!/usr/bin/env python
"""Benchmark of the sm_100a allocation planner (one JSON line on rank 0).

Workload (BASELINE.json configs[1]): the paper's XR compound DAG
(ar-assistant: detect -> describe -> speak, 2 variants per task x 24 MIG/MPS
segments x 8 batch sizes, synthetic profile seed 13), 28-slice budget,
A+S+T space.  One step = one batch of B independent XR single solves
(plan() at B demand points spread over [240, 720) rps, all feasible), solved
in one plan_batch() call.  Inputs are regenerated from the bundled knobs
(synthetic data; no reference code is read at run time).

metric  candidate allocations evaluated/sec: every allocation of the solve's
        cross-product (prod of Stage-1 pool sizes, + the empty choice for
        could-be-idle tasks) is decided exactly per solve -- by a full
        derive/validate or by one of the reference's admissible filters --
        the same count for the GPU arm and the CPU reference arm.  Also
        reported: planner solve ms and candidates fully evaluated.
value   whole-job covered candidates / max-over-ranks device time (CUDA events
        recorded by libjsv on its launching stream).
e2e     same metric through the public API (planner.plan_batch) timed with
        torch CUDA events around the call: includes lowering lookup, the
        host->device request/probe copies, all kernels and the device->host
        results + Python decode.

--impl reference runs the CPU oracle port (oracle/planner_oracle.py, a
restatement of the reference planner, pinned to reference goldens) over a
bounded sample of the same workload on all host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLUSH_BYTES = 512 << 20  # > 126 MB L2
SLICE_BUDGET = 28
NOMINAL_DEMAND = 480.0


def xr_inputs():
    from paper_2603_08797_b200.model import app_from_dict
    from paper_2603_08797_b200.profiles import knobs_from_dict, synth_profile

    with open(os.path.join(ROOT, "tests", "golden", "apps.json")) as fh:
        doc = json.load(fh)["ar-assistant"]
    app = app_from_dict(doc["app"])
    return app, synth_profile(app.graph, knobs_from_dict(doc["knobs"]))


def demand_points(batch: int, rank: int, world: int) -> list[float]:
    # B points per rank, disjoint across ranks, all within the feasible range
    step = 480.0 / (batch * world)
    return [240.0 + step * (k * world + rank) for k in range(batch)]


def covered(app, res, demand) -> int:
    """|cross-product| the solve decided: prod over tasks of pool size (+1 if may be idle)."""
    from paper_2603_08797_b200.model import propagate_demand

    g = app.graph
    mins = {}
    for t in g.task_ids:
        for s in g.successors[t]:
            mins[(t, s)] = min(v.factors[s] for v in g.task(t).variants)
    low = propagate_demand(g, demand, mins)
    n = 1
    for t in g.task_ids:
        n *= res.stats.pool_sizes.get(t, 0) + (1 if low[t] == 0.0 else 0)
    return n


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = set()
        sm = []
        smax = None
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                smax = float(s[1])
            except ValueError:
                continue
            for n, v in zip(names, s[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return {}


def roofline(kt: dict, st_total: dict, steps: int, clocks: dict) -> dict:
    """Dominant kernel against its binding roof (SM issue / FP64 pipe).

    pairs_a does D order-preserving <= and == FP64 compares per candidate pair
    (2*D DSETP-class FP64 ops, the algorithmic minimum of a weak-dominance
    test); s2_leaf's algorithmic work is its (prefix, bundle) items times the
    filter chain.  Peak FP64 (no FMA, every compare counted as one op):
    148 SMs x 64 lanes x f_clk.
    """
    dom = max(kt.items(), key=lambda kv: kv[1][0])
    name, (ms, cnt) = dom
    per_launch_ms = ms / max(1, cnt)
    f_clk = 1.965e9
    peak = 148 * 64 * f_clk / 1e12  # TFLOP/s (FP64 ops, no FMA)
    if name == "pairs_a":
        ops = st_total["pair_tests_a"] * 2 * st_total["dims"] / max(1, cnt)
    elif name == "pairs_b":
        ops = st_total["pair_tests_b"] * st_total["dims"] / max(1, cnt)
    elif name == "s2_leaf":
        ops = st_total["leaf_work"] * 12 / max(1, cnt)
    else:
        ops = 0.0
    achieved = ops / (per_launch_ms / 1e3) / 1e12 if per_launch_ms > 0 else 0.0
    return {"bound": "fp64", "kernel": name, "achieved": achieved, "peak": peak,
            "unit": "TFLOP/s", "frac": achieved / peak if peak else None, "traffic": None,
            "per_launch_ms": per_launch_ms, "share_of_step": ms / max(1e-9, st_total["ms_total"]),
            "peak_source": "derived: 148 SM x 64 FP64 lanes x 1.965 GHz (not in MEASURED_PEAKS)"}


def cpu_sample(args) -> dict:
    """Oracle port (pure CPython restatement of the reference planner) on the host."""
    from multiprocessing import Pool

    n = args.cpu_sample
    dem = demand_points(n, 0, 1)
    cores = min(os.cpu_count() or 1, n) if args.impl == "reference" else 1
    if cores > 1:
        global _POOL
        if _POOL is None:
            _POOL = Pool(cores)
            _POOL.map(_cpu_one, dem[:cores])  # import + input generation outside the timing
        t0 = time.perf_counter()
        outs = _POOL.map(_cpu_one, dem, chunksize=1)
        wall = time.perf_counter() - t0
    else:
        _cpu_one(dem[0])
        t0 = time.perf_counter()
        outs = [_cpu_one(d) for d in dem]
        wall = time.perf_counter() - t0
    cov = sum(o[0] for o in outs)
    return {"value": cov / wall, "unit": "candidates/s", "cores": cores, "kind": "port",
            "sample": f"{n} XR single solves (plan, A+S+T, 28 slices, demand {dem[0]:.0f}..{dem[-1]:.0f})"
                      f" by oracle/planner_oracle.py in {wall:.1f}s",
            "solve_ms": wall * 1e3 * cores / n, "evaluated": sum(o[1] for o in outs)}


_POOL = None
_INPUTS = None


def _cpu_one(demand):
    global _INPUTS
    from oracle import planner_oracle as O
    from paper_2603_08797_b200.plan_types import PlannerOptions, PlanRequest, SearchSpace

    if _INPUTS is None:
        _INPUTS = xr_inputs()
    app, table = _INPUTS
    req = PlanRequest(demand, SLICE_BUDGET, SearchSpace(True, True, True))
    s = O.BranchAndBound(app, table, req, PlannerOptions())
    s.visit(0, 0)
    g = app.graph
    n = 1
    for t in g.task_ids:
        n *= len(s.pools[t]) + (1 if s.zero_ok[t] else 0)
    return n, s.nodes + getattr(s, "leaves", 0)


def run_reference(args, rank, world) -> None:
    if rank != 0:
        return
    vals = []
    for _ in range(args.steps):
        vals.append(cpu_sample(args))
    v = statistics.median(x["value"] for x in vals)
    cb = dict(vals[-1])
    cb["value"] = v
    line = {
        "impl": "reference", "metric": "candidate allocations evaluated/sec", "value": v,
        "unit": "candidates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "XR DAG single solves (configs[1]) - CPU oracle port sample",
                   "slice_budget": SLICE_BUDGET, "space": "A+S+T"},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": v, "unit": "candidates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "solve_ms": cb["solve_ms"],
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--impl", default="gpu", choices=("gpu", "reference"))
    ap.add_argument("--cpu-sample", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    os.environ["JSV_DEVICE"] = str(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2603_08797_b200 import _native as N
    from paper_2603_08797_b200 import planner as P
    from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace

    app, table = xr_inputs()
    space = SearchSpace(True, True, True)
    dem = demand_points(args.batch, rank, world)
    reqs = [PlanRequest(d, SLICE_BUDGET, space) for d in dem]
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    ctx = N.context(local)

    for _ in range(args.warmup):
        P.plan_batch(app, table, reqs)
    # covered candidates per step (fixed by the pools; identical every step)
    res = P.plan_batch(app, table, reqs)
    cov_step = sum(covered(app, r, d) for r, d in zip(res, dem))
    assert all(r.feasible for r in res)
    # single-solve latency (one plan() call at the nominal demand)
    one = PlanRequest(NOMINAL_DEMAND, SLICE_BUDGET, space)
    lat = []
    for _ in range(max(5, args.steps // 2)):
        flush.zero_()
        torch.cuda.synchronize()
        P.plan(app, table, one)
        lat.append(P.last_stats()["ms_total"])
    solve_ms = statistics.median(lat)

    N.profile(ctx, True)
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    dev_ms = 0.0
    e2e_ms = 0.0
    launches = 0
    tot = {"pair_tests_a": 0, "pair_tests_b": 0, "leaf_work": 0, "dims": 0, "ms_total": 0.0,
           "leaves": 0, "nodes": 0}
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        P.plan_batch(app, table, reqs)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms += e0.elapsed_time(e1)
        st = P.last_stats()
        dev_ms += st["ms_total"]
        launches += st["kernel_launches"]
        for k in ("pair_tests_a", "pair_tests_b", "leaf_work", "leaves", "nodes"):
            tot[k] += st[k]
        tot["dims"] = st["dims"]
        tot["ms_total"] += st["ms_total"]
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    kt = N.kernel_times(ctx)
    N.profile(ctx, False)

    t = torch.tensor([dev_ms, e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms_max, e2e_ms_max = t.tolist()
    total_cov = cov_step * args.steps * world
    value = total_cov / (dev_ms_max / 1e3)
    e2e_value = total_cov / (e2e_ms_max / 1e3)
    h2d = args.batch * __import__("ctypes").sizeof(N.Probe) + __import__("ctypes").sizeof(N.Request)
    d2h = args.batch * __import__("ctypes").sizeof(N.PlanOut)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": "candidate allocations evaluated/sec",
        "value": value,
        "unit": "candidates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_ms_max / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": "XR compound DAG single solves (BASELINE configs[1]): ar-assistant, "
                        "2 variants x 24 MIG/MPS segments x 8 batches per task, 28 slices, A+S+T",
            "solves_per_step_per_gpu": args.batch,
            "demand_rps": [round(dem[0], 3), round(dem[-1], 3)],
            "candidates_per_step_per_gpu": cov_step,
            "l2": "flushed between timed steps (512 MiB write)",
            "parallelism": f"independent solves sharded over {world} GPU(s)",
        },
        "solve_ms": solve_ms,
        "solves_per_s": args.batch * world * args.steps / (dev_ms_max / 1e3),
        "candidates_fully_evaluated_per_step": tot["leaves"] // args.steps,
        "search_nodes_per_step": tot["nodes"] // args.steps,
        "e2e": {"value": e2e_value, "unit": "candidates/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms_max / args.steps},
        "gpu_launches": launches,
        "clocks": clk,
        "roofline": roofline(kt, tot, args.steps, clk),
        "kernel_ms": {k: round(v[0], 4) for k, v in kt.items() if v[1]},
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = {k: v for k, v in cpu_sample(args).items()
                                if k in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
