"""Lower (AppSpec, ProfileTable) to the flat arrays of ``jsv_problem_desc``.

Every string ordering the reference relies on becomes an integer rank here:
task ids (Python code-point order), variant ids, SegmentType (mig, mps) and
profile keys (variant, mig, mps, batch).  Only static metadata is computed on
the host; candidate enumeration, evaluation and search run on the GPU.

Accepts the reference's own AppSpec/ProfileTable objects as well as this
package's (duck-typed on the public attributes).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import ConfigError, ProfileError

MIGS = ("1g", "1g_me", "2g", "3g", "4g", "7g")
MIG_COST = {"1g": 1, "1g_me": 1, "2g": 2, "3g": 3, "4g": 4, "7g": 7}
SEG_RANK = {(m, k): i for i, (m, k) in enumerate((m, k) for m in MIGS for k in (1, 2, 3, 4))}
SEG_7G = SEG_RANK[("7g", 1)]


def _i32(xs) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(xs if len(xs) else [0], dtype=np.int32))


def _f64(xs) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(xs if len(xs) else [0.0], dtype=np.float64))


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


@dataclass
class Lowered:
    """Host mirror of one problem + its native handle."""

    ids: list[str]
    index: dict[str, int]
    topo: list[int]
    decl: list[int]
    edges: list[tuple[int, int]]          # edge id -> (src, dst), grouped by src, dst id-sorted
    edge_index: dict[tuple[str, str], int]
    paths: list[tuple[str, ...]]
    variants: list[list[str]]             # per task, id-sorted
    most_acc: list[int]
    keys: list[list[tuple]]               # per task: (variant id, SegmentType, batch) key order
    key_index: list[dict]                 # per task: (vid, seg, batch) -> local index
    key_cost: list[list[int]]
    key_thr: list[list[float]]
    key_lat: list[list[float]]
    key_var: list[list[int]]
    sub_tuples: list[list[list[int]]]     # [task][2a+s] -> local key indices
    a_max: float
    arrays: dict = field(default_factory=dict)
    handle: C.c_void_p | None = None
    ctx: C.c_void_p | None = None

    def __del__(self):
        if self.handle is not None and N._lib is not None:
            try:
                N._lib.jsv_problem_destroy(self.handle)
            except Exception:
                pass


def _a_max(graph) -> float:
    # max_system_accuracy: fraction-weighted path accuracy at the top variants
    best = {t.id: t.most_accurate.accuracy for t in graph.tasks}
    total = 0.0
    for p in graph.paths:
        prod = 1.0
        for t in p:
            prod *= best[t]
        total += graph.path_fractions[p] * prod
    return total


def lower(app, profile) -> Lowered:
    g = app.graph
    ids = sorted(g.task_ids)
    if len(ids) > N.MAX_TASKS:
        raise ConfigError(f"the sm_100a planner supports up to {N.MAX_TASKS} tasks")
    index = {t: i for i, t in enumerate(ids)}
    topo = [index[t] for t in g.topological_order]
    decl = [index[t] for t in g.task_ids]
    edges: list[tuple[int, int]] = []
    edge_index: dict[tuple[str, str], int] = {}
    succ_off = [0]
    for t in ids:
        for d in g.successors[t]:
            edge_index[(t, d)] = len(edges)
            edges.append((index[t], index[d]))
        succ_off.append(len(edges))
    if len(edges) > N.MAX_EDGES:
        raise ConfigError(f"the sm_100a planner supports up to {N.MAX_EDGES} edges")
    pred_off = [0]
    pred_edge: list[int] = []
    for t in ids:
        for s in g.predecessors[t]:
            pred_edge.append(edge_index[(s, t)])
        pred_off.append(len(pred_edge))
    paths = list(g.paths)
    if len(paths) > N.MAX_PATHS:
        raise ConfigError(f"the sm_100a planner supports up to {N.MAX_PATHS} paths")
    path_off = [0]
    path_task: list[int] = []
    for p in paths:
        path_task.extend(index[t] for t in p)
        path_off.append(len(path_task))
    path_frac = [g.path_fractions[p] for p in paths]

    variants, most_acc = [], []
    var_off, var_acc, var_fac_off, var_fac = [0], [], [], []
    for t in ids:
        task = g.task(t)
        vs = sorted(v.id for v in task.variants)
        variants.append(vs)
        most_acc.append(vs.index(task.most_accurate.id))
        for vid in vs:
            v = task.variant(vid)
            var_acc.append(v.accuracy)
            var_fac_off.append(len(var_fac))
            var_fac.extend(v.factors[d] for d in g.successors[t])
        var_off.append(len(var_acc))

    keys, key_index, key_cost, key_thr, key_lat, key_var = [], [], [], [], [], []
    key_off = [0]
    flat_var, flat_seg, flat_batch, flat_cost, flat_lat, flat_thr = [], [], [], [], [], []
    sub_off = [0]
    sub_key: list[int] = []
    grp_off = [0]
    grp_rep: list[int] = []
    sub_tuples = []
    for ti, t in enumerate(ids):
        vset = {v: i for i, v in enumerate(variants[ti])}
        ks = [k for k in profile.entries_for(t) if k[1] in vset]
        tk = [(k[1], k[2], k[3]) for k in ks]
        keys.append(tk)
        key_index.append({k: i for i, k in enumerate(tk)})
        cost, thr, lat, var = [], [], [], []
        for k in ks:
            e = profile[k]
            cost.append(k[2].slice_cost)
            thr.append(e.throughput_rps)
            lat.append(e.latency_ms)
            var.append(vset[k[1]])
            flat_var.append(vset[k[1]])
            flat_seg.append(SEG_RANK[(k[2].mig, k[2].mps)])
            flat_batch.append(k[3])
            flat_cost.append(k[2].slice_cost)
            flat_lat.append(e.latency_ms)
            flat_thr.append(e.throughput_rps)
        key_cost.append(cost)
        key_thr.append(thr)
        key_lat.append(lat)
        key_var.append(var)
        key_off.append(len(flat_var))
        per_sub = []
        for a in (0, 1):
            for s in (0, 1):
                allowed_v = set(range(len(variants[ti]))) if a else {most_acc[ti]}
                tup = [i for i, k in enumerate(ks)
                       if var[i] in allowed_v and (s or (k[2].mig == "7g" and k[2].mps == 1))]
                per_sub.append(tup)
                sub_key.extend(tup)
                sub_off.append(len(sub_key))
                # variant groups in variant order + representatives (planner.py:518-526)
                groups: dict[int, list[int]] = {}
                for pos, ki in enumerate(tup):
                    groups.setdefault(var[ki], []).append(pos)
                for vi in sorted(groups):
                    idx = groups[vi]
                    best_cap = min(idx, key=lambda i: (-thr[tup[i]] / cost[tup[i]], lat[tup[i]], i))
                    best_lat = min(idx, key=lambda i: (lat[tup[i]], -thr[tup[i]] / cost[tup[i]], i))
                    reps = sorted({best_cap, best_lat})
                    grp_rep.extend([reps[0], reps[1] if len(reps) > 1 else -1])
                grp_off.append(len(grp_rep) // 2)
        sub_tuples.append(per_sub)

    a_max = _a_max(g)
    lw = Lowered(ids, index, topo, decl, edges, edge_index, paths, variants, most_acc, keys,
                 key_index, key_cost, key_thr, key_lat, key_var, sub_tuples, a_max)
    arr = {
        "topo": _i32(topo), "decl": _i32(decl), "succ_off": _i32(succ_off),
        "edge_dst": _i32([d for _, d in edges]), "pred_off": _i32(pred_off),
        "pred_edge": _i32(pred_edge), "path_off": _i32(path_off), "path_task": _i32(path_task),
        "path_frac": _f64(path_frac), "var_off": _i32(var_off), "var_acc": _f64(var_acc),
        "var_fac_off": _i32(var_fac_off), "var_fac": _f64(var_fac), "most_acc": _i32(most_acc),
        "key_off": _i32(key_off), "key_var": _i32(flat_var), "key_seg": _i32(flat_seg),
        "key_batch": _i32(flat_batch), "key_cost": _i32(flat_cost), "key_lat": _f64(flat_lat),
        "key_thr": _f64(flat_thr), "sub_off": _i32(sub_off), "sub_key": _i32(sub_key),
        "grp_off": _i32(grp_off), "grp_rep": _i32(grp_rep),
    }
    lw.arrays = arr
    return lw


def problem_desc(lw: Lowered) -> N.ProblemDesc:
    a = lw.arrays
    d = N.ProblemDesc()
    d.n_tasks = len(lw.ids)
    d.n_edges = len(lw.edges)
    d.n_paths = len(lw.paths)
    d.entry = lw.topo[0]
    for name in ("topo", "decl", "succ_off", "edge_dst", "pred_off", "pred_edge", "path_off",
                 "path_task", "var_off", "var_fac_off", "most_acc", "key_off", "key_var",
                 "key_seg", "key_batch", "key_cost", "sub_off", "sub_key", "grp_off", "grp_rep"):
        setattr(d, name, _ptr(a[name], C.c_int32))
    for name in ("path_frac", "var_acc", "var_fac", "key_lat", "key_thr"):
        setattr(d, name, _ptr(a[name], C.c_double))
    d.a_max = lw.a_max
    return d


def attach(lw: Lowered, ctx) -> Lowered:
    """Upload the lowered problem to the device of ``ctx``."""
    if lw.handle is not None and lw.ctx is ctx:
        return lw
    if lw.a_max <= 0:
        raise ConfigError("degenerate application: maximum attainable accuracy is 0")
    desc = problem_desc(lw)
    h = C.c_void_p()
    N.check(N.load_library().jsv_problem_create(ctx, C.byref(desc), C.byref(h)))
    lw.handle = h
    lw.ctx = ctx
    return lw


def space_bits(space) -> int:
    return ((N.SPACE_A if space.accuracy_scaling else 0) | (N.SPACE_S if space.spatial_partitioning
                                                             else 0)
            | (N.SPACE_T if space.task_graph_informed else 0))


def request_struct(lw: Lowered, request, options, feasible_only=None):
    """(Request, keep-alive arrays) for one planner call (memoised per lowering on
    every field the struct is built from; callers never mutate it)."""
    fo = options.feasible_only if feasible_only is None else feasible_only
    ov = request.factor_overrides
    try:
        key = (int(request.slice_budget), space_bits(request.space), float(request.slack),
               tuple(sorted(ov.items())) if ov else (), int(options.pareto_width),
               int(options.exhaustive_limit), float(options.eps), tuple(options.mix_fractions),
               bool(fo))
    except TypeError:  # (unhashable or unorderable inputs: no memo)
        key = None
    cache = lw.arrays.setdefault("_req_cache", {})
    if key is not None and key in cache:
        return cache[key]
    built = _request_struct(lw, request, options, fo)
    if key is not None:
        if len(cache) >= 64:
            cache.clear()
        cache[key] = built
    return built


def _request_struct(lw: Lowered, request, options, fo):
    r = N.Request()
    r.budget = int(request.slice_budget)
    r.space = space_bits(request.space)
    r.slack = float(request.slack)
    ov = dict(request.factor_overrides or {})
    has = np.zeros(max(1, len(lw.edges)), dtype=np.uint8)
    val = np.zeros(max(1, len(lw.edges)), dtype=np.float64)
    for edge, v in ov.items():
        if edge in lw.edge_index:
            has[lw.edge_index[edge]] = 1
            val[lw.edge_index[edge]] = float(v)
    r.has_override = _ptr(has, C.c_uint8)
    r.override_val = _ptr(val, C.c_double)
    r.pareto_width = int(options.pareto_width)
    r.exhaustive_limit = int(options.exhaustive_limit)
    r.eps = float(options.eps)
    mix = tuple(options.mix_fractions)
    if len(mix) > N.MAX_MIX:
        raise ConfigError(f"at most {N.MAX_MIX} mix fractions are supported")
    r.n_mix = len(mix)
    for i, m in enumerate(mix):
        r.mix[i] = float(m)
    r.feasible_only = 1 if fo else 0
    return r, (has, val)


def check_usable(app, profile, lw: Lowered, request) -> None:
    """ConfigError of _candidate_pool (planner.py:627-630), raised in topological order."""
    sp = request.space
    for t in app.graph.topological_order:
        ti = lw.index[t]
        subs = [2 * a + s for a in ((0, 1) if sp.accuracy_scaling else (0,))
                for s in ((0, 1) if sp.spatial_partitioning else (0,))]
        if not any(lw.sub_tuples[ti][k] for k in subs):
            raise ConfigError(
                f"profile has no usable entries for task {t!r} in the requested space"
            )


def uninformed_statics(app, profile, lw: Lowered, request) -> dict:
    """Static budgets of plan_uninformed (reference planner.py:994-1067), in Python float order."""
    g = app.graph
    slo = app.effective_latency_slo_ms
    spatial = request.space.spatial_partitioning
    worst = {}
    for t in g.task_ids:
        ti = lw.index[t]
        ma = lw.most_acc[ti]
        w = 0.0
        for k, (vid, seg, b) in enumerate(lw.keys[ti]):
            if lw.key_var[ti][k] == ma and (spatial or (seg.mig == "7g" and seg.mps == 1)):
                w = max(w, lw.key_lat[ti][k])
        if w <= 0.0:
            raise ConfigError(f"profile has no usable entries for task {t!r} in the requested space")
        worst[t] = w
    lat_budget = {}
    for t in g.task_ids:
        lat_budget[t] = min(slo * worst[t] / sum(worst[u] for u in p) for p in g.paths_through(t))
    best_hput, best_slices, min_cost = {}, {}, {}
    for t in g.task_ids:
        ti = lw.index[t]
        ma = lw.most_acc[ti]
        rows = [k for k in range(len(lw.keys[ti]))
                if lw.key_var[ti][k] == ma
                and (spatial or (lw.keys[ti][k][1].mig == "7g" and lw.keys[ti][k][1].mps == 1))]
        # tuple order == key order, so the id tie-break (variant, segment, batch) is the index
        best = min(rows, key=lambda k: (-lw.key_thr[ti][k], lw.key_cost[ti][k], k))
        best_hput[t] = lw.key_thr[ti][best]
        best_slices[t] = lw.key_cost[ti][best]
        allowed = set(range(len(lw.variants[ti]))) if request.space.accuracy_scaling else {ma}
        min_cost[t] = min(lw.key_cost[ti][k] for k in range(len(lw.keys[ti]))
                          if lw.key_var[ti][k] in allowed
                          and (spatial or (lw.keys[ti][k][1].mig == "7g"
                                           and lw.keys[ti][k][1].mps == 1)))
    depth = {t: max(len(p) for p in g.paths_through(t)) for t in g.task_ids}
    weight = {t: sum(g.path_fractions[p] for p in g.paths_through(t)) for t in g.task_ids}
    floor = {t: g.task(t).most_accurate.accuracy * app.accuracy_slo ** (1.0 / depth[t])
             for t in g.task_ids}
    return {"lat_budget": lat_budget, "best_hput": best_hput, "best_slices": best_slices,
            "min_cost": min_cost, "weight": weight, "floor": floor}


def probe_struct(app, lw: Lowered, demand: float, statics: dict | None = None) -> N.Probe:
    p = N.Probe()
    p.demand = float(demand)
    p.slo_eff = app.effective_latency_slo_ms
    p.acc_slo = float(app.accuracy_slo)
    p.alpha = float(app.alpha)
    p.beta = float(app.beta)
    if statics:
        for t, ti in lw.index.items():
            p.uni_lat_budget[ti] = statics["lat_budget"][t]
            p.uni_floor[ti] = statics["floor"][t]
            p.uni_weight[ti] = statics["weight"][t]
            p.uni_best_hput[ti] = statics["best_hput"][t]
            p.uni_best_slices[ti] = statics["best_slices"][t]
            p.uni_min_cost[ti] = statics["min_cost"][t]
    return p


def encode_assignment(app, profile, lw: Lowered, m):
    """derive_configuration input checks (planner.py:258-273) + packed items per task."""
    n_items = np.zeros(N.MAX_TASKS, dtype=np.int32)
    items = np.zeros((N.MAX_TASKS, N.MAX_ITEMS), dtype=np.uint32)
    known = set(app.graph.task_ids)
    canon = []
    for key in sorted(m):
        count = m[key]
        if count < 0 or count != int(count):
            raise ConfigError(f"instance count for {key} must be a non-negative integer")
        if count == 0:
            continue
        t, vid, seg, batch = key
        if t not in known:
            raise ConfigError(f"unknown task {t!r} in configuration")
        profile[key]  # ProfileError when absent
        ti = lw.index[t]
        if vid not in lw.variants[ti]:
            raise ConfigError(f"task {t!r} has no variant {vid!r}")
        k = lw.key_index[ti][(vid, seg, batch)]
        if n_items[ti] >= N.MAX_ITEMS:
            raise ConfigError(f"more than {N.MAX_ITEMS} instance types for task {t!r}")
        if int(count) > 0xFFFF:
            raise ConfigError("instance count exceeds 65535")
        items[ti, n_items[ti]] = (k << 16) | int(count)
        n_items[ti] += 1
        canon.append((key, int(count)))
    return n_items, items, tuple(canon)
