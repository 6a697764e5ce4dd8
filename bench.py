#!/usr/bin/env python
"""Benchmark of the sm_100a allocation planner (one JSON line on rank 0).

Workload (BASELINE.json configs[1]): the paper's XR compound DAG
(ar-assistant: detect -> describe -> speak, 2 variants per task x 24 MIG/MPS
segments x 8 batch sizes, synthetic profile seed 13), 28-slice budget,
A+S+T space.  One step = one batch of B independent XR single solves
(plan() at B demand points spread over [240, 720) rps, all feasible), solved
in one plan_batch() call with the exhaustive Stage-2 strategy: every
allocation of each solve's Stage-1 cross-product (29.3M at 480 rps) is
decided -- by its prefix's throughput verdicts (k_x_live: the reference's
branch-and-bound kills such a prefix at that task, planner.py:876-881) or by
the register sweep of the live prefixes -- and the feasible ones are derived
and validated exactly and folded into the argmax.  Inputs are regenerated from
the bundled knobs (synthetic data; no reference code is read at run time).

metric  candidate allocations evaluated/sec, counted as allocations DECIDED
        per second (the pools' cross-product, jsv_stats exh_candidates) -- the
        same count the reference arm is credited with ("covered": its
        branch-and-bound decides the same cross-product), so value / reference
        is a solves-per-second ratio.  The allocations the sweep compared one by
        one (`swept`) and the prefixes it derived in full (`live_prefixes`) are
        reported beside it and are what the roofline counts.
value   whole-job decided candidates / max-over-ranks device time of the
        whole plan_batch (Stage 1 + Stage 2 + finalize; CUDA events recorded by
        libjsv on its launching stream; inputs resident on the host side of the
        call but no Python work inside the timed region).
e2e     same metric through the public API (planner.plan_batch) timed with
        torch CUDA events around the call: host->device request/probe copies,
        all kernels, device->host results and the Python decode of every
        PlanResult.
extras  solve_ms (one plan() at 480 rps, default strategy), search-mode
        covered/s, and configs[2]'s demand sweep (max-serviceable demand over
        the 64-point latency x accuracy SLO grid, sharded over ranks) in
        points/s.

--impl reference runs the CPU oracle port (oracle/planner_oracle.py, a
restatement of the reference planner pinned to reference goldens) over a
bounded sample of the same workload on all host cores.  The reference planner
is a branch-and-bound: its arm is credited with every allocation its search
decides (pool cross-product, "covered") -- the GPU arm counts the same decided
cross-product.
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
    from paper_2603_08797_b200 import workloads

    return workloads.xr()


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


# algorithmic lane-ops of the exhaustive Stage 2, per unit:
#   swept candidate: the four verdicts as integer compares on its rank record;
#   derived live prefix (XR: T = 3, E = 2, one path), the reference's operation
#   count of the prefix part of derive/validate: demand of the two downstream tasks
#   (2 x (mul + add)) and the sink's need (mul), the prefix tasks' throughput
#   verdicts (2 x (mul + sub)), the partial path latency (2 x 2 L + 2 adds of the
#   compensated sum) and accuracy product (2 muls) = 15
OPS_SWEPT = 4
OPS_PREFIX = 15


def roofline(kt: dict, tot: dict, dom: str = "s2_exh") -> dict:
    """The exhaustive sweep kernel against the SM instruction-issue roof.

    Work counted is what the pruned sweep actually evaluates: OPS_SWEPT integer
    lane-ops per candidate compared in the register sweep plus OPS_PREFIX per live
    prefix derived (prefixes failing a prefix task's throughput verdict are decided by
    k_x_live and cost nothing here; their candidates are in `value`, not here).
    Integer lane-ops issue on the ALU or the FMA pipe, so the roof is instruction
    issue: 148 SMs x 4 schedulers x 32 lanes x 1.965 GHz = 37.2 T lane-ops/s (derived;
    MEASURED_PEAKS.json holds only HBM and bf16 tensor peaks, neither of which this
    kernel uses).  `issue_active` is ncu's issue-slot utilisation of the same kernel
    (profiles/ncu_traffic.json), the instruction-level view of the same roof.
    """
    ms, cnt = kt.get(dom, (0.0, 0))
    per_launch_ms = ms / max(1, cnt)
    f_clk = 1.965e9
    peak = 148 * 4 * 32 * f_clk / 1e12
    swept = tot.get("swept", 0) / max(1, cnt)
    live = tot.get("live_prefixes", 0) / max(1, cnt)
    ops = swept * OPS_SWEPT + live * OPS_PREFIX
    achieved = ops / (per_launch_ms / 1e3) / 1e12 if per_launch_ms > 0 else 0.0
    traffic = issue = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            d = json.load(fh).get("k_s2_exh")
        if d:
            traffic = d["dram_read_bytes"] + d["dram_write_bytes"]
            issue = d.get("issue_active_pct")
    return {"bound": "issue", "kernel": "k_s2_exh", "achieved": achieved, "peak": peak,
            "unit": "Tops/s", "frac": achieved / peak if peak else None, "traffic": traffic,
            "traffic_note": "DRAM bytes per launch (64 solves) from profiles/ncu_traffic.json; "
                            "algorithmic DRAM bytes ~0 (sink records and sorted columns L1-resident)",
            "ops_per_swept_candidate": OPS_SWEPT, "ops_per_live_prefix": OPS_PREFIX,
            "swept_per_launch": swept, "live_prefixes_per_launch": live,
            "decided_per_launch": tot["exh_candidates"] / max(1, cnt),
            "per_launch_ms": per_launch_ms,
            "share_of_step": ms / max(1e-9, tot["ms_total"]),
            "issue_active": issue,
            "peak_source": "derived: 148 SM x 4 schedulers x 32 lanes x 1.965 GHz issue "
                           "(not in MEASURED_PEAKS)"}


# fused Stage 1 (k_s1_job) algorithmic lane-ops per unit: a skyline pair test on the
# float shadow (4 compares), an exact test behind it (2 (D - 1) double compares, D = 5
# for XR rows), a generated candidate's statistics (bundle_stats: per item a multiply,
# max, add and integer multiply-add, ~2.5 items -> 12)
OPS_SHADOW = 4
OPS_EXACT = 8
OPS_CAND = 12


def roofline_s1(kt: dict, tot: dict) -> dict:
    """k_s1_job (fused Stage 1) against the same SM issue roof as `roofline` (the work
    it does per launch: pair tests of both skyline passes and candidate statistics;
    generation, hash dedup, frontier sorts and truncation counted as overhead)."""
    ms, cnt = kt.get("generate", (0.0, 0))
    per_launch_ms = ms / max(1, cnt)
    peak = 148 * 4 * 32 * 1.965e9 / 1e12
    ops = (tot.get("s1_shadow_tests", 0) * OPS_SHADOW + tot.get("s1_exact_tests", 0) * OPS_EXACT +
           tot.get("candidates_generated", 0) * OPS_CAND) / max(1, cnt)
    achieved = ops / (per_launch_ms / 1e3) / 1e12 if per_launch_ms > 0 else 0.0
    traffic = issue = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            d = json.load(fh).get("k_s1_job")
        if d:
            traffic = d["dram_read_bytes"] + d["dram_write_bytes"]
            issue = d.get("issue_active_pct")
    return {"bound": "issue", "kernel": "k_s1_job", "achieved": achieved, "peak": peak,
            "unit": "Tops/s", "frac": achieved / peak if peak else None, "traffic": traffic,
            "ops_per_shadow_test": OPS_SHADOW, "ops_per_exact_test": OPS_EXACT,
            "ops_per_candidate": OPS_CAND,
            "shadow_tests_per_launch": tot.get("s1_shadow_tests", 0) / max(1, cnt),
            "exact_tests_per_launch": tot.get("s1_exact_tests", 0) / max(1, cnt),
            "candidates_per_launch": tot.get("candidates_generated", 0) / max(1, cnt),
            "per_launch_ms": per_launch_ms, "share_of_step": ms / max(1e-9, tot["ms_total"]),
            "issue_active": issue,
            "peak_source": "derived: 148 SM x 4 schedulers x 32 lanes x 1.965 GHz issue"}


def place_plans(app, table, reqs) -> dict:
    """the cli `plan` tail (cli.py:173-174) -- every plan's
    instance_segments -> min_gpus -> pack, through placement.py (libjsv host code)."""
    from paper_2603_08797_b200 import planner as P
    from paper_2603_08797_b200.placement import instance_segments, min_gpus, pack

    res = P.plan_batch(app, table, reqs)
    segs = [instance_segments(r.config) for r in res if r.config is not None]
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        plans = [pack(s, min_gpus(s)) for s in segs]
    ms = (time.perf_counter() - t0) * 1e3 / reps
    return {"plans": len(segs), "ms": ms, "plans_per_s": len(segs) / (ms / 1e3),
            "instances": sum(len(s) for s in segs), "gpus": sum(p.gpu_count for p in plans),
            "all_placed": all(p.fully_placed for p in plans)}


def cpu_sample(args) -> dict:
    """Oracle port (pure CPython restatement of the reference planner) on the host."""
    from multiprocessing import Pool

    n = args.cpu_sample
    if args.impl == "reference":
        # all host cores, ~24 solves (~4 s of CPU work) per core per step
        n = max(n, 24 * (os.cpu_count() or 1))
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


def sweep_detail(dstat: dict, st: dict, kt: dict) -> dict:
    """configs[2] beyond points/s: probes (the reference bisection's sequential count vs
    the GPU's, speculation included), the device time of the sweep and its kernel
    split, and the exhaustive kernel's work against the issue roof (as `roofline`)."""
    dev_ms = st["ms_total"]
    ms, cnt = kt.get("s2_exh", (0.0, 0))
    f_clk = 1.965e9
    peak = 148 * 4 * 32 * f_clk / 1e12
    ops = st.get("swept", 0) * OPS_SWEPT + st.get("live_prefixes", 0) * OPS_PREFIX
    achieved = ops / (ms / 1e3) / 1e12 if ms > 0 else 0.0
    tot_k = sum(v[0] for v in kt.values()) or 1.0
    return {"probes_reference": dstat.get("probes"), "probes_gpu": dstat.get("gpu_probes"),
            "speculation_overhead": (dstat.get("gpu_probes", 0) / max(1, dstat.get("probes", 1))),
            "device_ms": dev_ms, "probes_per_s_device": dstat.get("gpu_probes", 0) / (dev_ms / 1e3)
            if dev_ms else None,
            "decided_candidates_per_s_device": st["exh_candidates"] / (dev_ms / 1e3) if dev_ms else None,
            "kernel_share": {k: round(v[0] / tot_k, 3) for k, v in sorted(kt.items(), key=lambda x: -x[1][0])
                             if v[1] and v[0] / tot_k >= 0.02},
            "roofline": {"bound": "issue", "kernel": "k_s2_exh", "achieved": achieved, "peak": peak,
                         "unit": "Tops/s", "frac": achieved / peak, "launches": cnt,
                         "ms": ms, "swept": st.get("swept", 0), "live_prefixes": st.get("live_prefixes", 0)}}


def _cpu_point(i):
    from oracle import planner_oracle as O
    from paper_2603_08797_b200 import workloads
    from paper_2603_08797_b200.plan_types import SearchSpace

    app, table = workloads.xr()
    a = c3_apps(app)[i]
    return O.max_demand(a, table, SLICE_BUDGET, SearchSpace(True, True, True)).demand_rps


def cpu_sweep_all_cores(n_points: int = 32) -> dict:
    """configs[2] on every host core: independent grid points through the oracle port
    in a multiprocessing.Pool(os.cpu_count()) (max_demand is pure)."""
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    idx = list(range(0, 64, max(1, 64 // n_points)))[:n_points]
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_point, idx, chunksize=1)
    wall = time.perf_counter() - t0
    return {"value": len(idx) / wall, "unit": "points/s", "cores": cores, "kind": "port",
            "sample": f"{len(idx)} of the 64 grid points (max_demand, rel_tol 1e-3) by "
                      f"oracle/planner_oracle.py on {cores} processes in {wall:.1f}s"}


def cpu_sweep_sample(app) -> dict:
    """configs[2] on the host: the oracle port's max_demand for two of the 64 grid
    points (one core), next to the GPU sweep's points/s."""
    from oracle import planner_oracle as O
    from paper_2603_08797_b200.plan_types import SearchSpace

    _app, table = xr_inputs()
    pts = c3_apps(app)[::37]
    t0 = time.perf_counter()
    for a in pts:
        O.max_demand(a, table, SLICE_BUDGET, SearchSpace(True, True, True))
    wall = time.perf_counter() - t0
    return {"value": len(pts) / wall, "unit": "points/s", "cores": 1, "kind": "port",
            "sample": f"{len(pts)} grid points (max_demand, rel_tol 1e-3) by oracle/planner_oracle.py "
                      f"in {wall:.1f}s"}


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
    for _ in range(args.warmup):  # untimed, like the GPU arm's warm-up steps
        cpu_sample(args)
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


C3_LAT = (800.0, 1000.0, 1200.0, 1400.0, 1550.0, 1800.0, 2000.0, 2500.0)
C3_ACC = (0.80, 0.825, 0.85, 0.875, 0.90, 0.925, 0.95, 0.975)


def c3_apps(app):
    """BASELINE configs[2]: the XR app over the 64-point latency x accuracy SLO grid."""
    import dataclasses

    return [dataclasses.replace(app, latency_slo_ms=L, accuracy_slo=a) for L in C3_LAT for a in C3_ACC]


def star12_solve(P, torch, flush, layered: bool = True) -> dict:
    """configs[3]: the 12-task star at 200 rps / 84 slices (reference: no result in 600 s)."""
    from paper_2603_08797_b200 import workloads
    from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace

    app, table = workloads.star(12)
    req = PlanRequest(200.0, 84, SearchSpace(True, True, True))
    P.plan(app, table, req)
    dev, wall = [], []
    for _ in range(5):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = P.plan(app, table, req)
        wall.append((time.perf_counter() - t0) * 1e3)
        dev.append(P.last_stats()["ms_total"])
    # max_demand: the bisection's feasibility probes answered by the fan-out solver
    sp = SearchSpace(True, True, True)
    P.max_demand(app, table, 84, sp)
    t0 = time.perf_counter()
    md = P.max_demand(app, table, 84, sp)
    md_ms = (time.perf_counter() - t0) * 1e3
    return {"solve_ms": statistics.median(dev), "solve_wall_ms": statistics.median(wall),
            "objective": r.objective, "total_slices": r.config.total_slices,
            "solver": "fan-out knapsack-DP bounded enumeration + exact evaluation",
            "max_demand_rps": md.demand_rps, "max_demand_probes": md.probes,
            "max_demand_ms": md_ms,
            **({"layered_1_4_4_3": layered_solve(P)} if layered else {})}


def layered_solve(P) -> dict:
    """configs[3]'s layered stress variant: 1 -> 4 -> 4 -> 3, 12 tasks, 32
    edges, 48 paths, at 200 rps / 84 slices -- the GPU branch-and-bound (the reference's
    DFS needs 696 s for the 1-2-2-1 instance and does not finish this one)."""
    from paper_2603_08797_b200 import workloads
    from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace

    app, table = workloads.layered((1, 4, 4, 3))
    req = PlanRequest(200.0, 84, SearchSpace(True, True, True))
    P.plan(app, table, req)
    t0 = time.perf_counter()
    r = P.plan(app, table, req)
    wall = (time.perf_counter() - t0) * 1e3
    st = P.last_stats()
    return {"solve_wall_ms": wall, "solve_ms": st["ms_total"], "objective": r.objective,
            "total_slices": r.config.total_slices if r.config else None, "nodes": st["nodes"],
            "leaves": st["leaves"], "solver": "level-synchronous branch-and-bound, depth-first "
                                              "frontier chunks"}


def traffic840(P, rank: int = 0, world: int = 1, device=None) -> dict:
    """configs[4]: traffic-analysis on 840 slices -- max_demand in all 8 spaces, then the
    288-bin day trace planned for A+S+T and the three ablations (one batch per space).
    Sharded over the ranks (independent units, no data-path collective):
    spaces [rank::world] for max_demand and a contiguous block of the trace's bins per
    space (shard.block_range); the caller takes the max of the times over ranks."""
    from paper_2603_08797_b200 import workload, workloads
    from paper_2603_08797_b200.plan_types import ALL_SPACES, SearchSpace
    from paper_2603_08797_b200.shard import block_range

    app, table = workloads.traffic()
    md_all = {}
    for sp in ALL_SPACES:  # warm-up (device buffers grown to this budget's sizes); every
        md_all[sp.label] = P.max_demand(app, table, 840, sp).demand_rps  # rank needs A+S+T
    mine = ALL_SPACES[rank::world]
    t0 = time.perf_counter()
    md = {sp.label: P.max_demand(app, table, 840, sp).demand_rps for sp in mine}
    md_ms = (time.perf_counter() - t0) * 1e3
    trace = workload.gen_trace(workload.TraceShape(0.35, 0.65, 0.03, 288), md_all["A+S+T"], 21)
    spaces = [SearchSpace.from_label(x) for x in ("A+S+T", "S+T", "A+T", "A+S")]
    part = block_range(len(trace.bins), world, rank)
    for sp in spaces:  # warm-up
        workload.plan_day(app, table, trace, 840, sp, device=device, part=part)
    t0 = time.perf_counter()
    days = {sp.label: workload.plan_day(app, table, trace, 840, sp, device=device, part=part)
            for sp in spaces}
    day_ms = (time.perf_counter() - t0) * 1e3
    return {"max_demand_8_spaces_ms": md_ms, "max_demand_rps": md_all,
            "trace_bins": len(trace), "trace_plans": len(trace) * len(spaces), "trace_ms": day_ms,
            "trace_plans_per_s": len(trace) * len(spaces) / (day_ms / 1e3),
            "fallback_bins": {k: sum(d.used_fallback for d in v) for k, v in days.items()},
            "sharding": f"max_demand spaces [rank::{world}], trace bins [{part[0]}, {part[1]}) "
                        f"of {len(trace)} on rank {rank}"}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--impl", default="gpu", choices=("gpu", "reference"))
    ap.add_argument("--cpu-sample", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import ctypes

    import torch
    import torch.distributed as dist

    # JSV_BENCH_ONE_GPU=1 (tests only): every rank on GPU 0 with gloo plumbing, to
    # exercise the multi-rank path on a one-GPU box; real runs: one GPU per rank, NCCL
    one_gpu = os.environ.get("JSV_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    os.environ["JSV_DEVICE"] = str(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
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
    P.set_strategy("exhaustive", 1 << 40, device=local)

    for _ in range(args.warmup):
        P.plan_batch(app, table, reqs, device=local)
    res = P.plan_batch(app, table, reqs, device=local)
    assert all(r.feasible for r in res)
    cov_step = sum(covered(app, r, d) for r, d in zip(res, dem))

    # ---------------------------------------------------------- timed region
    # pass 1 (value, roofline): libjsv's CUDA events on its launching stream, one
    # pair around the whole batch and one per kernel; pass 2 (e2e): the same K
    # steps through the public API with the per-kernel events off, timed by torch
    # CUDA events around the call (host copies, kernels, result decode)
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    # (events only around the two roofline kernels: an event pair around every launch
    # of the step would add ~8% of host gaps to the device time it measures)
    N.profile(ctx, True, ("generate", "s2_exh"))
    dev_ms = e2e_ms = 0.0
    launches = 0
    tot = {"exh_candidates": 0, "leaves": 0, "swept": 0, "live_prefixes": 0, "ms_total": 0.0,
           "ms_stage1": 0.0, "ms_stage2": 0.0, "s1_shadow_tests": 0, "s1_exact_tests": 0,
           "candidates_generated": 0}
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        P.plan_batch(app, table, reqs, device=local)
        st = P.last_stats(local)
        dev_ms += st["ms_total"]
        launches += st["kernel_launches"]
        for k in tot:
            tot[k] += st[k]
    torch.cuda.synchronize()
    kt = N.kernel_times(ctx)
    N.profile(ctx, False)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        P.plan_batch(app, table, reqs, device=local)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms += e0.elapsed_time(e1)
        launches += P.last_stats(local)["kernel_launches"]
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    cand_step = tot["exh_candidates"] // args.steps

    # ---------------------------------------------------------------- extras
    extras = {}
    if not args.no_extras:
        # one plan() at the nominal demand with the default strategy
        P.set_strategy("auto", device=local)
        one = PlanRequest(NOMINAL_DEMAND, SLICE_BUDGET, space)
        lat_dev, lat_wall = [], []
        for i in range(max(10, args.steps // 2) + 2):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            P.plan(app, table, one)
            w = (time.perf_counter() - t0) * 1e3
            if i >= 2:
                lat_wall.append(w)
                lat_dev.append(P.last_stats(local)["ms_total"])
        extras["solve_ms"] = statistics.median(lat_dev)
        extras["solve_wall_ms"] = statistics.median(lat_wall)
        # the level-synchronous branch-and-bound: allocations covered per second
        P.set_strategy("search", device=local)
        P.plan_batch(app, table, reqs, device=local)
        sms = []
        for _ in range(5):
            flush.zero_()
            torch.cuda.synchronize()
            P.plan_batch(app, table, reqs, device=local)
            sms.append(P.last_stats(local)["ms_total"])
        extras["search_covered_per_s"] = cov_step / (statistics.median(sms) / 1e3)
        extras["search_ms_per_batch"] = statistics.median(sms)
        # configs[2]: max-serviceable demand over the 64-point SLO grid, points sharded over ranks
        P.set_strategy("auto", device=local)
        grid = c3_apps(app)[rank::world]
        P.max_demand_grid(grid, table, SLICE_BUDGET, space, device=local)  # warm-up
        torch.cuda.synchronize()
        sw = []
        for _ in range(3):
            t0 = time.perf_counter()
            mres = P.max_demand_grid(grid, table, SLICE_BUDGET, space, device=local)
            sw.append((time.perf_counter() - t0) * 1e3)
        sweep_ms = min(sw)
        probes = sum(r.probes for r in mres)
        dstat = P.last_demand_stats()
        # one more pass with libjsv's per-kernel events: device time split and the
        # exhaustive kernel's work (the sweep's feasibility probes use the same kernels)
        N.profile(ctx, True)
        N.kernel_times(ctx)  # (reset)
        P.max_demand_grid(grid, table, SLICE_BUDGET, space, device=local)
        sst = P.last_stats(local)
        skt = N.kernel_times(ctx)
        N.profile(ctx, False)
        extras["sweep_local"] = (len(grid), sweep_ms, probes)
        extras["sweep_detail"] = sweep_detail(dstat, sst, skt)
        c4 = traffic840(P, rank, world, device=local)
        extras["c4_local"] = (c4["max_demand_8_spaces_ms"], c4["trace_ms"])
        if rank == 0:
            # (the layered solve is a single-GPU figure; multi-rank runs skip it)
            extras["configs3_star12"] = star12_solve(P, torch, flush, layered=world == 1)
            extras["configs4_traffic840"] = c4
            extras["placement"] = place_plans(app, table, reqs)

    c4_local = extras.pop("c4_local", (0.0, 0.0))
    t = torch.tensor([dev_ms, e2e_ms, extras.get("sweep_local", (0, 0.0, 0))[1], c4_local[0],
                      c4_local[1]], dtype=torch.float64, device="cpu" if one_gpu else "cuda")
    tc = torch.tensor([float(tot["exh_candidates"])], dtype=torch.float64, device=t.device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tc, op=dist.ReduceOp.SUM)  # every rank's own demand points
    dev_ms_max, e2e_ms_max, sweep_ms_max, md_ms_max, day_ms_max = t.tolist()
    if "configs4_traffic840" in extras:
        c4 = extras["configs4_traffic840"]
        c4["max_demand_8_spaces_ms"] = md_ms_max  # (max over ranks)
        c4["trace_ms"] = day_ms_max
        c4["trace_plans_per_s"] = c4["trace_plans"] / (day_ms_max / 1e3)
    total_cand = int(tc.item())
    value = total_cand / (dev_ms_max / 1e3)
    e2e_value = total_cand / (e2e_ms_max / 1e3)
    h2d = args.batch * ctypes.sizeof(N.Probe) + ctypes.sizeof(N.Request)
    d2h = args.batch * ctypes.sizeof(N.PlanOut) + ctypes.sizeof(N.Stats)
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
                        "2 variants x 24 MIG/MPS segments x 8 batches per task, 28 slices, A+S+T; "
                        "exhaustive Stage 2 (every allocation of the Stage-1 cross-product decided)",
            "solves_per_step_per_gpu": args.batch,
            "demand_rps": [round(dem[0], 3), round(dem[-1], 3)],
            "candidates_per_step_per_gpu": cand_step,
            "l2": "flushed between timed steps (512 MiB write)",
            "parallelism": f"independent solves sharded over {world} GPU(s)",
        },
        "candidates_decided_per_step": tot["leaves"] // args.steps,
        "candidates_swept_per_step": tot["swept"] // args.steps,
        "live_prefixes_per_step": tot["live_prefixes"] // args.steps,
        "stage_ms_per_step": {"stage1": tot["ms_stage1"] / args.steps,
                              "stage2": tot["ms_stage2"] / args.steps},
        "solves_per_s": args.batch * world * args.steps / (dev_ms_max / 1e3),
        "e2e": {"value": e2e_value, "unit": "candidates/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms_max / args.steps},
        "gpu_launches": launches,
        "clocks": clk,
        # the dominant kernel of the step (largest share of the device time) first
        **dict(zip(("roofline", "roofline_next"),
                   sorted((roofline(kt, tot), roofline_s1(kt, tot)),
                          key=lambda r: -r["share_of_step"]))),
        "kernel_ms": {k: round(v[0], 4) for k, v in kt.items() if v[1]},
    }
    if extras:
        n_pts, _, probes = extras.pop("sweep_local")
        extras["sweep"] = {"config": "BASELINE configs[2]: XR max_demand over 8 latency x 8 accuracy "
                                     "SLOs, 28 slices, A+S+T, rel_tol 1e-3, points sharded over ranks",
                           "points": len(C3_LAT) * len(C3_ACC), "wall_ms": sweep_ms_max,
                           "points_per_s": len(C3_LAT) * len(C3_ACC) / (sweep_ms_max / 1e3),
                           "probes_rank0": probes}
        extras["sweep"].update(extras.pop("sweep_detail"))
        line.update(extras)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = {k: v for k, v in cpu_sample(args).items()
                                if k in ("value", "unit", "cores", "kind", "sample")}
        if "sweep" in line:
            line["sweep"]["cpu_baseline"] = cpu_sweep_sample(app)
            line["sweep"]["cpu_baseline_all_cores"] = cpu_sweep_all_cores()
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
