"""Drop-in replacement for ``sliceserve.planner`` backed by the sm_100a library.

Same public names, signatures and result types as the reference module
(reference pkg/src/sliceserve/planner.py:36-54).  Every candidate is
enumerated, evaluated, filtered and reduced on the GPU by libjsv.so:

    plan()            -> jsv_plan_batch        (planner.py:915-957 / 973-1110)
    plan_uninformed() -> jsv_plan_batch, T off (planner.py:973-1110)
    max_demand()      -> jsv_max_demand_batch  (planner.py:1125-1175)
    derive_configuration()   -> jsv_derive     (planner.py:243-315)
    validate_configuration() -> jsv_validate   (planner.py:329-361)

Host Python only validates inputs, lowers them to flat arrays once per
(graph, profile), and rebuilds the frozen result dataclasses.  If the CUDA
library or a GPU is missing, calls raise ``NativeError``; there is no CPU
fallback.
"""

from __future__ import annotations

import ctypes as C
import time
from collections import OrderedDict
from typing import Mapping, Sequence

import numpy as np

from . import _lower as LW
from . import _native as N
from .errors import ConfigError
from .plan_types import (
    ALL_SPACES,
    Configuration,
    ConstraintVerdict,
    MaxDemandResult,
    OracleCaps,
    PlannerOptions,
    PlanRequest,
    PlanResult,
    SearchSpace,
    SolverStats,
    plan_result_to_dict,
)

__all__ = [
    "SearchSpace",
    "ALL_SPACES",
    "PlanRequest",
    "PlannerOptions",
    "Configuration",
    "derive_configuration",
    "ConstraintVerdict",
    "validate_configuration",
    "SolverStats",
    "PlanResult",
    "plan",
    "plan_uninformed",
    "plan_batch",
    "MaxDemandResult",
    "max_demand",
    "max_demand_grid",
    "OracleCaps",
    "brute_force_plan",
    "plan_result_to_dict",
    "last_stats",
    "last_demand_stats",
    "set_strategy",
]

# ------------------------------------------------------------ problem cache

_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()
_CACHE_MAX = 32


def _problem(app, profile, device=None) -> LW.Lowered:
    ctx = N.context(device)
    key = (id(app.graph), id(profile), ctx.value)
    hit = _CACHE.get(key)
    if hit is not None and hit[0] is app.graph and hit[1] is profile:
        _CACHE.move_to_end(key)
        return hit[2]
    lw = LW.attach(LW.lower(app, profile), ctx)
    _CACHE[key] = (app.graph, profile, lw)  # strong refs keep ids unique while cached
    while len(_CACHE) > _CACHE_MAX:
        _CACHE.popitem(last=False)
    return lw


def set_strategy(strategy: str, max_candidates: int = 1 << 31, device=None) -> None:
    """Choose the Stage-2 strategy of this process's planner context.

    "search" (level-synchronous branch-and-bound with the reference's filters),
    "exhaustive" (every allocation of the Stage-1 cross-product derived and
    validated, for solves with at most `max_candidates` allocations) or "auto".
    All strategies return the reference's exact result; this is a performance
    knob with no reference counterpart.
    """
    N.set_strategy(N.context(device), strategy, max_candidates)


def last_stats(device=None) -> dict:
    s = N.last_stats(N.context(device))
    return {k: getattr(s, k) for k, _ in s._fields_}


# ------------------------------------------------------------ result decode

def _binding(code: int) -> str | None:
    return None if code < 0 else N.BINDING_NAMES[code]


def _config_from(out: N.PlanOut, app, lw: LW.Lowered, demand: float) -> Configuration:
    g = app.graph
    m = []
    hput = {}
    for ti, t in enumerate(lw.ids):
        for k in range(out.n_items[ti]):
            w = out.items[ti][k]
            vid, seg, batch = lw.keys[ti][w >> 16]
            m.append(((t, vid, seg, batch), int(w & 0xFFFF)))
    for t in g.topological_order:
        ti = lw.index[t]
        for k in range(out.n_items[ti]):
            w = out.items[ti][k]
            vid, seg, batch = lw.keys[ti][w >> 16]
            hput[(t, vid, seg, batch)] = out.hput[ti][k]
    idx = lw.index
    fan = {}
    for t in g.task_ids:
        for d in g.successors[t]:
            fan[(t, d)] = out.fanout[lw.edge_index[(t, d)]]
    return Configuration(
        m=tuple(m),
        entry_demand_rps=float(demand),
        latency_ms={t: out.latency[idx[t]] for t in g.task_ids},
        capacity_rps={t: out.capacity[idx[t]] for t in g.task_ids},
        demand_rps={t: out.demand[idx[t]] for t in g.topological_order},
        slices={t: int(out.slices[idx[t]]) for t in g.task_ids},
        accuracy={t: out.accuracy[idx[t]] for t in g.task_ids},
        fanout=fan,
        hput=hput,
        path_accuracy={p: out.path_acc[i] for i, p in enumerate(lw.paths)},
        total_slices=int(out.total_slices),
        a_obj=out.a_obj,
        a_max=lw.a_max,
        objective=out.objective,
        structurally_infeasible=tuple(
            t for t in g.topological_order if (out.uncovered_mask >> idx[t]) & 1
        ),
    )


def _verdicts_from(out: N.PlanOut, app, lw: LW.Lowered) -> tuple[ConstraintVerdict, ...]:
    g = app.graph
    vs = []
    for i, p in enumerate(lw.paths):
        mg = out.lat_margin[i]
        vs.append(ConstraintVerdict("latency", "->".join(p), mg >= 0, mg))
    for t in g.topological_order:
        mg = out.thr_margin[lw.index[t]]
        vs.append(ConstraintVerdict("throughput", t, mg >= 0, mg))
    mg = out.res_margin
    vs.append(ConstraintVerdict("resources", "", mg >= 0, mg))
    mg = out.acc_margin
    vs.append(ConstraintVerdict("accuracy", "", mg >= 0, mg))
    bad = tuple(t for t in g.topological_order if (out.uncovered_mask >> lw.index[t]) & 1)
    vs.append(ConstraintVerdict("coverage", ",".join(bad), not bad,
                                0.0 if not bad else -float(len(bad))))
    return tuple(vs)


_PLAN_DTYPE = None
_PROBE_DTYPE = None
_new = object.__new__


def _mk(cls, **fields):
    # frozen-dataclass instance without the per-field object.__setattr__ of its
    # __init__ (same __dict__, so ==, repr and dataclasses.* behave identically)
    o = _new(cls)
    o.__dict__.update(fields)
    return o


def _result_from(out: N.PlanOut, app, lw: LW.Lowered, request, wall_ms: float) -> PlanResult:
    return _results_from((N.PlanOut * 1).from_buffer_copy(out), [app], lw, [request], wall_ms)[0]


try:  # C decoder (csrc/jsv_decode.c); the Python decoder below is its reference
    from . import _jsvdecode as _DEC
except ImportError:  # pragma: no cover - built by __graft_entry__.build()
    _DEC = None
_DEC_LAYOUT = None


def _dec_meta(app, lw: LW.Lowered) -> tuple:
    """Per-(graph, lowering) tables of the C decoder, cached on the lowering."""
    g = app.graph
    hit = lw.arrays.get("_dec_meta")
    if hit is not None and hit[0] is g:
        return hit[1]
    idx = lw.index
    topo_t = tuple(g.topological_order)
    task_t = tuple(g.task_ids)
    edges = [((t, d), lw.edge_index[(t, d)]) for t in task_t for d in g.successors[t]]
    keys_full = tuple(tuple((t,) + k for k in lw.keys[ti]) for ti, t in enumerate(lw.ids))
    meta = (tuple(lw.ids), keys_full, topo_t, tuple(idx[t] for t in topo_t), task_t,
            tuple(idx[t] for t in task_t), tuple(e for e, _ in edges), tuple(k for _, k in edges),
            tuple(lw.paths), tuple("->".join(p) for p in lw.paths), float(lw.a_max),
            tuple(N.BINDING_NAMES[k] for k in range(len(N.BINDING_NAMES))),
            PlanResult, Configuration, ConstraintVerdict, SolverStats,
            # the keys' hashes (hput dict inserts skip the dataclass __hash__)
            tuple(tuple(hash(k) for k in ks) for ks in keys_full))
    lw.arrays["_dec_meta"] = (g, meta)
    return meta


def _results_from(outs, apps, lw: LW.Lowered, requests, wall_ms: float) -> list[PlanResult]:
    """jsv_plan_out records -> PlanResults (C decoder when built, else _results_py)."""
    global _DEC_LAYOUT
    if _DEC is None:
        return _results_py(outs, apps, lw, requests, wall_ms)
    if _DEC_LAYOUT is None:
        lay = {name: getattr(N.PlanOut, name).offset for name, _ in N.PlanOut._fields_}
        lay["size"] = C.sizeof(N.PlanOut)
        lay["max_items"] = N.MAX_ITEMS
        _DEC_LAYOUT = lay
    return _DEC.decode(outs, len(requests), _DEC_LAYOUT, _dec_meta(apps[0], lw),
                       [r.demand_rps for r in requests], float(wall_ms))


def _results_py(outs, apps, lw: LW.Lowered, requests, wall_ms: float) -> list[PlanResult]:
    """Decode a ctypes array of jsv_plan_out records into PlanResults.

    Every field is pulled out of the records once, batch-wide, through a numpy
    view (field access on ctypes structures costs microseconds each); the
    dataclasses are then built from plain Python lists.  Same values as the
    per-field decode: ints and IEEE doubles are copied bit-for-bit.
    """
    global _PLAN_DTYPE
    if _PLAN_DTYPE is None:
        _PLAN_DTYPE = np.dtype(N.PlanOut)
    arr = np.frombuffer(outs, dtype=_PLAN_DTYPE)
    T, P = len(lw.ids), len(lw.paths)
    E = len(lw.edges)
    g = apps[0].graph
    idx = lw.index
    ids = lw.ids
    topo_t = list(g.topological_order)
    topo_i = [idx[t] for t in topo_t]
    task_t = list(g.task_ids)
    task_i = [idx[t] for t in task_t]
    edge_k = [((t, d), lw.edge_index[(t, d)]) for t in task_t for d in g.successors[t]]
    edge_names = [e for e, _ in edge_k]
    col = {}
    for name in ("feasible", "has_config", "binding", "objective", "a_obj", "nodes",
                 "total_slices", "uncovered_mask", "res_margin", "acc_margin"):
        col[name] = arr[name].tolist()
    # per-task columns in the order the result dicts list them
    for name in ("latency", "capacity", "accuracy", "slices"):
        col[name] = arr[name][:, task_i].tolist()
    for name in ("demand", "thr_margin", "pool_size", "pool_present", "truncated"):
        col[name] = arr[name][:, topo_i].tolist()
    col["n_items"] = arr["n_items"][:, :T].tolist()
    col["items"] = arr["items"][:, :T].tolist()
    col["hput"] = arr["hput"][:, :T].tolist()
    col["fanout"] = arr["fanout"][:, [k for _, k in edge_k]].tolist()
    col["path_acc"] = arr["path_acc"][:, :P].tolist()
    col["lat_margin"] = arr["lat_margin"][:, :P].tolist()
    path_names = ["->".join(p) for p in lw.paths]
    paths = list(lw.paths)
    topo_pos = list(enumerate(topo_i))
    keys = lw.keys
    a_max = lw.a_max
    res = []
    for i, request in enumerate(requests):
        sizes = {}
        cut = []
        present, psize, trunc = col["pool_present"][i], col["pool_size"][i], col["truncated"][i]
        for k, t in enumerate(topo_t):
            if present[k]:
                sizes[t] = psize[k]
                if trunc[k]:
                    cut.append(t)
        stats = _mk(SolverStats, nodes=col["nodes"][i], wall_ms=wall_ms, pool_sizes=sizes,
                    truncated_tasks=tuple(cut))
        if not col["has_config"][i]:
            res.append(_mk(PlanResult, feasible=False, config=None, objective=None, a_max=a_max,
                           binding_constraint=_binding(col["binding"][i]), verdicts=(),
                           stats=stats))
            continue
        n_items, items, hp = col["n_items"][i], col["items"][i], col["hput"][i]
        m = []
        for ti, t in enumerate(ids):
            row, kt = items[ti], keys[ti]
            for k in range(n_items[ti]):
                w = row[k]
                m.append(((t,) + kt[w >> 16], w & 0xFFFF))
        hput = {}
        for t, ti in zip(topo_t, topo_i):
            row, kt, hrow = items[ti], keys[ti], hp[ti]
            for k in range(n_items[ti]):
                hput[(t,) + kt[row[k] >> 16]] = hrow[k]
        unc = col["uncovered_mask"][i]
        bad = tuple(t for t, ti in zip(topo_t, topo_i) if (unc >> ti) & 1) if unc else ()
        cfg = _mk(
            Configuration,
            m=tuple(m),
            entry_demand_rps=float(request.demand_rps),
            latency_ms=dict(zip(task_t, col["latency"][i])),
            capacity_rps=dict(zip(task_t, col["capacity"][i])),
            demand_rps=dict(zip(topo_t, col["demand"][i])),
            slices=dict(zip(task_t, col["slices"][i])),
            accuracy=dict(zip(task_t, col["accuracy"][i])),
            fanout=dict(zip(edge_names, col["fanout"][i])),
            hput=hput,
            path_accuracy=dict(zip(paths, col["path_acc"][i])),
            total_slices=col["total_slices"][i],
            a_obj=col["a_obj"][i],
            a_max=a_max,
            objective=col["objective"][i],
            structurally_infeasible=bad,
        )
        vs = []
        lm, tm = col["lat_margin"][i], col["thr_margin"][i]
        for name, mg in zip(path_names, lm):
            vs.append(_mk(ConstraintVerdict, name="latency", subject=name, passed=mg >= 0, margin=mg))
        for t, mg in zip(topo_t, tm):
            vs.append(_mk(ConstraintVerdict, name="throughput", subject=t, passed=mg >= 0, margin=mg))
        mg = col["res_margin"][i]
        vs.append(_mk(ConstraintVerdict, name="resources", subject="", passed=mg >= 0, margin=mg))
        mg = col["acc_margin"][i]
        vs.append(_mk(ConstraintVerdict, name="accuracy", subject="", passed=mg >= 0, margin=mg))
        vs.append(_mk(ConstraintVerdict, name="coverage", subject=",".join(bad), passed=not bad,
                      margin=0.0 if not bad else -float(len(bad))))
        vs = tuple(vs)
        if col["feasible"][i]:
            res.append(_mk(PlanResult, feasible=True, config=cfg, objective=cfg.objective,
                           a_max=lw.a_max, binding_constraint=None, verdicts=vs, stats=stats))
        else:
            res.append(_mk(PlanResult, feasible=False, config=cfg, objective=None, a_max=lw.a_max,
                           binding_constraint=_binding(col["binding"][i]), verdicts=vs,
                           stats=stats))
    return res


# ------------------------------------------------------------------ solves

def _prepare(app, profile, request: PlanRequest, options: PlannerOptions, device=None):
    lw = _problem(app, profile, device)
    statics = None
    if request.space.task_graph_informed:
        LW.check_usable(app, profile, lw, request)
    else:
        statics = LW.uninformed_statics(app, profile, lw, request)
    return lw, statics


def plan_batch(
    app,
    profile,
    requests: Sequence[PlanRequest],
    options: PlannerOptions | None = None,
    apps: Sequence | None = None,
    device: int | None = None,
) -> list[PlanResult]:
    """Many plan() calls in one GPU batch.

    All requests must share slice budget, space, slack and overrides; demand
    (and, through ``apps``, the SLO/objective scalars) may differ per probe.
    Results equal ``[plan(a, profile, r, options) for a, r in ...]``.
    """
    if not requests:
        return []
    t0 = time.perf_counter()
    w = int((options or PlannerOptions()).pareto_width)
    if w == 0 and requests[0].space.task_graph_informed:
        return [_zero_width_result(a, profile, r, device)
                for a, r in zip(list(apps) if apps is not None else [app] * len(requests), requests)]
    if not 1 <= w <= 32766:
        raise ConfigError(f"pareto_width {w} is outside the supported range 1..32766 "
                          "(0 only with a task-graph-informed space)")
    outs, lw, apps = solve_records(app, profile, requests, options, apps, device, transient=True)
    wall = (time.perf_counter() - t0) * 1000.0
    return _results_from(outs, apps, lw, requests, wall)


def _zero_width_result(app, profile, request: PlanRequest, device=None) -> PlanResult:
    """pareto_width = 0: _pareto_filter keeps no bundle of any (non-empty) frontier
    (planner.py:574-583), so every pool is empty and truncated and the first task is
    dead -- plan() returns its "resources" result (planner.py:930-938)."""
    t0 = time.perf_counter()
    lw, _ = _prepare(app, profile, request, PlannerOptions(), device)
    order = tuple(app.graph.topological_order)
    stats = SolverStats(nodes=0, wall_ms=(time.perf_counter() - t0) * 1000.0,
                        pool_sizes={t: 0 for t in order}, truncated_tasks=order)
    return PlanResult(False, None, None, lw.a_max, "resources", (), stats)


def solve_records(app, profile, requests: Sequence[PlanRequest], options=None, apps=None,
                  device=None, shard: tuple[int, int] | None = None, transient: bool = False):
    """plan_batch without the decode: (jsv_plan_out array, lowering, apps).

    ``shard=(rank, world)`` sweeps only that block of every exhaustive
    candidate space (jsv_plan_batch_shard; shard.plan_sharded combines).
    ``transient``: the records land in this thread's page-locked buffer, valid
    until the thread's next transient call (plan_batch decodes them at once).
    """
    options = options or PlannerOptions()
    same_app = apps is None
    apps = list(apps) if apps is not None else [app] * len(requests)
    r0 = requests[0]
    ov0 = dict(r0.factor_overrides or {})
    sp0 = r0.space
    for r in requests[1:]:
        sp = r.space
        if (r.slice_budget != r0.slice_budget or r.slack != r0.slack
                or (sp is not sp0 and (sp.__class__ is not sp0.__class__
                                       or sp.accuracy_scaling != sp0.accuracy_scaling
                                       or sp.spatial_partitioning != sp0.spatial_partitioning
                                       or sp.task_graph_informed != sp0.task_graph_informed))
                or (r.factor_overrides is not r0.factor_overrides
                    and dict(r.factor_overrides or {}) != ov0)):
            raise ConfigError("plan_batch requests must share budget, space, slack and overrides")
    lw, _ = _prepare(app, profile, r0, options, device)
    probes = (N.Probe * len(requests))()
    if same_app and r0.space.task_graph_informed:
        # one app: the probes differ only in demand (a numpy view fills them)
        global _PROBE_DTYPE
        if _PROBE_DTYPE is None:
            _PROBE_DTYPE = np.dtype(N.Probe)
        proto = LW.probe_struct(app, lw, 0.0, None)
        view = np.frombuffer(probes, dtype=_PROBE_DTYPE)
        view[:] = np.frombuffer(proto, dtype=_PROBE_DTYPE)[0]
        view["demand"] = [float(r.demand_rps) for r in requests]
    else:
        # plan_uninformed's static budgets depend on the app and the space, not on the
        # demand: one computation per distinct app object (a day trace of 288 bins paid
        # 288 Python passes over the profile otherwise)
        statics = {}
        for i, (a, r) in enumerate(zip(apps, requests)):
            if a.graph is not app.graph and a.graph != app.graph:
                raise ConfigError("plan_batch apps must share one task graph")
            st = None
            if not r.space.task_graph_informed:
                key = (id(a), r.space.accuracy_scaling, r.space.spatial_partitioning)
                st = statics.get(key)
                if st is None:
                    st = statics[key] = LW.uninformed_statics(a, profile, lw, r)
            probes[i] = LW.probe_struct(a, lw, r.demand_rps, st)
    req, keep = LW.request_struct(lw, r0, options)
    outs = N.pinned_outs(len(requests)) if transient else None
    if outs is None:
        outs = (N.PlanOut * len(requests))()
    lib = N.load_library()
    if shard is None:
        N.check(lib.jsv_plan_batch(lw.ctx, lw.handle, C.byref(req), len(requests), probes, outs))
    else:
        N.check(lib.jsv_plan_batch_shard(lw.ctx, lw.handle, C.byref(req), len(requests), probes,
                                         int(shard[0]), int(shard[1]), outs))
    return outs, lw, apps


def derive_record(app, profile, lw: LW.Lowered, request: PlanRequest, n_items, items) -> N.PlanOut:
    """derive + validate of one assignment given as per-task packed items (jsv_derive)."""
    ni = np.ascontiguousarray(n_items, dtype=np.int32)
    it = np.ascontiguousarray(items, dtype=np.uint32)
    req, keep = LW.request_struct(lw, request, PlannerOptions())
    probe = LW.probe_struct(app, lw, float(request.demand_rps))
    out = N.PlanOut()
    N.check(N.load_library().jsv_derive(
        lw.ctx, lw.handle, C.byref(req), C.byref(probe),
        ni.ctypes.data_as(C.POINTER(C.c_int32)), it.ctypes.data_as(C.POINTER(C.c_uint32)),
        C.byref(out)))
    return out


def decode_records(outs, app, lw: LW.Lowered, requests, wall_ms: float = 0.0) -> list[PlanResult]:
    """jsv_plan_out records -> PlanResults (the decoder plan_batch uses)."""
    return _results_from(outs, [app] * len(requests), lw, requests, wall_ms)


def plan(
    app,
    profile,
    request: PlanRequest,
    options: PlannerOptions | None = None,
) -> PlanResult:
    """Best instance-count assignment in the requested search space (planner.py:915-957)."""
    return plan_batch(app, profile, [request], options)[0]


def plan_uninformed(
    app,
    profile,
    request: PlanRequest,
    options: PlannerOptions | None = None,
) -> PlanResult:
    """Statically budgeted baseline (planner.py:973-1110)."""
    if request.space.task_graph_informed:
        raise ConfigError("plan_uninformed requires a space with task_graph_informed=False")
    return plan_batch(app, profile, [request], options)[0]


def max_demand_grid(
    apps: Sequence,
    profile,
    slice_budget: int,
    space: SearchSpace,
    slack: float = 0.05,
    options: PlannerOptions | None = None,
    rel_tol: float = 1e-3,
    device: int | None = None,
) -> list[MaxDemandResult]:
    """max_demand() for several SLO variants of one app graph, solved together.

    Each point replays the reference doubling + bisection exactly
    (planner.py:1152-1175); the GPU evaluates many speculative probes per launch.
    """
    if slice_budget <= 0:
        raise ConfigError(f"slice budget must be positive, got {slice_budget}")
    options = options or PlannerOptions()
    apps = list(apps)
    if not apps:
        return []
    t0 = time.perf_counter()
    base_req = PlanRequest(1e-6, slice_budget, space, slack)
    lw, _ = _prepare(apps[0], profile, base_req, options, device)
    points = (N.Probe * len(apps))()
    for i, a in enumerate(apps):
        if a.graph is not apps[0].graph and a.graph != apps[0].graph:
            raise ConfigError("max_demand_grid apps must share one task graph")
        st = None if space.task_graph_informed else LW.uninformed_statics(a, profile, lw, base_req)
        points[i] = LW.probe_struct(a, lw, 0.0, st)
    req, keep = LW.request_struct(lw, base_req, options)
    outs = (N.DemandOut * len(apps))()
    plans = (N.PlanOut * len(apps))()
    N.check(N.load_library().jsv_max_demand_batch(lw.ctx, lw.handle, C.byref(req), len(apps),
                                                  points, float(rel_tol), outs, plans))
    wall = (time.perf_counter() - t0) * 1000.0
    global _LAST_DEMAND
    _LAST_DEMAND = {"points": len(apps), "probes": sum(int(o.probes) for o in outs),
                    "gpu_probes": sum(int(o.gpu_probes) for o in outs), "wall_ms": wall}
    res = []
    for i, a in enumerate(apps):
        o = outs[i]
        dem = 0.0 if o.status == 1 else o.demand
        plan_dem = 1e-6 if o.status == 1 else o.demand
        pr = _result_from(plans[i], a, lw, PlanRequest(plan_dem, slice_budget, space, slack), wall)
        res.append(MaxDemandResult(dem, pr, int(o.probes)))
    return res


_LAST_DEMAND: dict = {}


def last_demand_stats() -> dict:
    """Probe counts of the last max_demand / max_demand_grid call: `probes` is the
    reference bisection's sequential count (MaxDemandResult.probes), `gpu_probes` the
    probes the GPU evaluated, speculation included."""
    return dict(_LAST_DEMAND)


def max_demand(
    app,
    profile,
    slice_budget: int,
    space: SearchSpace,
    slack: float = 0.05,
    options: PlannerOptions | None = None,
    rel_tol: float = 1e-3,
) -> MaxDemandResult:
    """Largest serviceable demand for a space, by doubling then bisection (1125-1175)."""
    return max_demand_grid([app], profile, slice_budget, space, slack, options, rel_tol)[0]


# -------------------------------------------------------- derive / validate

def _scalar_request(app, profile, request=None):
    lw = _problem(app, profile)
    request = request or PlanRequest(0.0, 0)
    req, keep = LW.request_struct(lw, request, PlannerOptions())
    return lw, req, keep


def derive_configuration(
    m: Mapping,
    app,
    profile,
    demand_rps: float,
    factor_overrides: Mapping[tuple[str, str], float] | None = None,
) -> Configuration:
    """Every quantity implied by an instance-count map, computed on the GPU (243-315)."""
    lw = _problem(app, profile)
    n_items, items, _ = LW.encode_assignment(app, profile, lw, m)
    request = PlanRequest(0.0, 0, SearchSpace(True, True, True), 0.0, factor_overrides)
    req, keep = LW.request_struct(lw, request, PlannerOptions())
    probe = LW.probe_struct(app, lw, float(demand_rps))
    out = N.PlanOut()
    N.check(N.load_library().jsv_derive(
        lw.ctx, lw.handle, C.byref(req), C.byref(probe),
        n_items.ctypes.data_as(C.POINTER(C.c_int32)),
        items.ctypes.data_as(C.POINTER(C.c_uint32)), C.byref(out)))
    return _config_from(out, app, lw, demand_rps)


def validate_configuration(config: Configuration, app, profile, request: PlanRequest):
    """Constraint verdicts with margins, computed on the GPU (329-361)."""
    lw = _problem(app, profile)
    req, keep = LW.request_struct(lw, request, PlannerOptions())
    probe = LW.probe_struct(app, lw, request.demand_rps)
    T = len(lw.ids)
    lat = np.zeros(T)
    cap = np.zeros(T)
    dem = np.zeros(T)
    for t, ti in lw.index.items():
        lat[ti] = config.latency_ms[t]
        cap[ti] = config.capacity_rps[t]
        dem[ti] = config.demand_rps[t]
    mask = 0
    for t in config.structurally_infeasible:
        mask |= 1 << lw.index[t]
    out = N.PlanOut()
    fp = C.POINTER(C.c_double)
    N.check(N.load_library().jsv_validate(
        lw.ctx, lw.handle, C.byref(req), C.byref(probe), lat.ctypes.data_as(fp),
        cap.ctypes.data_as(fp), dem.ctypes.data_as(fp), int(config.total_slices),
        float(config.a_obj), mask, C.byref(out)))
    g = app.graph
    vs = []
    for i, p in enumerate(lw.paths):
        mg = out.lat_margin[i]
        vs.append(ConstraintVerdict("latency", "->".join(p), mg >= 0, mg))
    for t in g.topological_order:
        mg = out.thr_margin[lw.index[t]]
        vs.append(ConstraintVerdict("throughput", t, mg >= 0, mg))
    vs.append(ConstraintVerdict("resources", "", out.res_margin >= 0, out.res_margin))
    vs.append(ConstraintVerdict("accuracy", "", out.acc_margin >= 0, out.acc_margin))
    bad = config.structurally_infeasible
    vs.append(ConstraintVerdict("coverage", ",".join(bad), not bad,
                                0.0 if not bad else -float(len(bad))))
    return tuple(vs)


def brute_force_plan(app, profile, request: PlanRequest, caps: OracleCaps = OracleCaps()) -> PlanResult:
    """Exhaustive solver for tiny instances, on the GPU (reference planner.py:1191-1272).

    Every instance-count map over the request space's profile keys (counts up to
    ``caps.max_count``, within the slice budget) is derived and validated by
    ``jsv_brute_force``; the argmax uses plan()'s tie-break.  The caps and the
    refusal messages are the reference's; the map count is ``stats.nodes``.
    """
    t0 = time.perf_counter()
    graph = app.graph
    if len(graph.task_ids) > caps.max_tasks:
        raise ConfigError(f"oracle refuses: {len(graph.task_ids)} tasks > cap {caps.max_tasks}")
    lw = _problem(app, profile)
    sub = 2 * int(bool(request.space.accuracy_scaling)) + int(bool(request.space.spatial_partitioning))
    for t in graph.task_ids:
        ti = lw.index[t]
        rows = [lw.keys[ti][k] for k in lw.sub_tuples[ti][sub]]
        if (len({r[0] for r in rows}) > caps.max_variants or len({r[1] for r in rows}) > caps.max_segments
                or len({r[2] for r in rows}) > caps.max_batches):
            raise ConfigError(f"oracle refuses: task {t!r} exceeds variant/segment/batch caps")
    req, keep = LW.request_struct(lw, request, PlannerOptions())
    probe = LW.probe_struct(app, lw, float(request.demand_rps))
    n = C.c_int64()
    found = np.zeros(1, dtype=np.int32)
    out = N.PlanOut()
    N.check(N.load_library().jsv_brute_force(
        lw.ctx, lw.handle, C.byref(req), C.byref(probe), int(caps.max_count),
        int(caps.max_assignments), C.byref(n), found.ctypes.data_as(C.POINTER(C.c_int32)),
        C.byref(out)))
    stats = SolverStats(nodes=int(n.value), wall_ms=(time.perf_counter() - t0) * 1000.0)
    if not found[0]:
        return PlanResult(False, None, None, lw.a_max, None, (), stats)
    cfg = _config_from(out, app, lw, request.demand_rps)
    return PlanResult(True, cfg, cfg.objective, lw.a_max, None, _verdicts_from(out, app, lw), stats)


def pool_dump(app, profile, request: PlanRequest, options: PlannerOptions | None = None,
              device=None) -> dict:
    """Stage-1 pools computed on the GPU, in the reference's frontier order (test helper)."""
    options = options or PlannerOptions()
    lw, _ = _prepare(app, profile, request, options, device)
    req, keep = LW.request_struct(lw, request, options)
    probe = LW.probe_struct(app, lw, request.demand_rps)
    lib = N.load_library()
    g = app.graph
    out = {}
    cap = max(1, options.pareto_width)
    for t in g.topological_order:
        ti = lw.index[t]
        outd = len(g.successors[t])
        n = C.c_int32()
        trunc = C.c_int32()
        nit = np.zeros(cap, dtype=np.int32)
        its = np.zeros((cap, N.MAX_ITEMS), dtype=np.uint32)
        st = np.zeros((cap, 4 + outd), dtype=np.float64)
        N.check(lib.jsv_pool_dump(lw.ctx, lw.handle, C.byref(req), C.byref(probe), ti, cap,
                                  C.byref(n), nit.ctypes.data_as(C.POINTER(C.c_int32)),
                                  its.ctypes.data_as(C.POINTER(C.c_uint32)),
                                  st.ctypes.data_as(C.POINTER(C.c_double)), C.byref(trunc)))
        rows = []
        for k in range(n.value):
            items = []
            for i in range(nit[k]):
                w = int(its[k, i])
                vid, seg, batch = lw.keys[ti][w >> 16]
                items.append([vid, seg.mig, seg.mps, batch, w & 0xFFFF])
            rows.append({"items": items, "slices": int(st[k, 0]), "capacity": float(st[k, 1]),
                         "accuracy": float(st[k, 2]), "latency": float(st[k, 3]),
                         "fanout": [float(x) for x in st[k, 4:4 + outd]]})
        out[t] = rows
    return out
