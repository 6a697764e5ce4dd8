"""Exact CPU solver for star DAGs (entry -> leaves) -- TEST INFRASTRUCTURE.

An independent checker for configs[3] (the 12-task star) at sizes the
reference's depth-first search does not finish (> 600 s at 12
tasks).  It returns what the reference ``plan()`` returns (planner.py:915-957):
the argmax of (objective desc, total slices asc, canonical m asc) over every
assignment of one Stage-1 pool bundle per task whose derive/validate verdicts
all pass (the semantic contract of DESIGN.md section 2, verified against the
reference's branch-and-bound on the 3..7-task ladder).

Method (plain Python + numpy, sharing nothing with the CUDA fan-out solver but
the pools): the pools come from ``planner_oracle.build_pools`` (the restated
reference Stage 1).  With the entry bundle b0 fixed, every leaf's verdicts
(throughput at demand d0 * fanout, path latency) are independent, and the
leaves couple only through the slice sum and the path-weighted accuracy sum.
A per-b0 max-plus DP over exact slice counts gives, for every total, the best
accuracy sum in real arithmetic; a depth-first enumeration over per-leaf
(slices, accuracy) classes bounded by that DP lists every class vector whose
real-valued objective is within ``delta`` of the best, and each listed vector
is derived and validated exactly by ``planner_oracle.derive/validate`` (the
reference's float order).  The band is widened until the best exact feasible
objective lies ``delta`` above the band's floor, so nothing better can be
outside it.  Within a class every bundle gives the same objective and slices;
the m tie-break picks, task by task in id order, the bundle whose item list is
smallest under tuple order of the concatenated m (planner.py:262, 852).
"""

from __future__ import annotations

import math

import numpy as np

from oracle import planner_oracle as O
from paper_2603_08797_b200.plan_types import PlannerOptions, PlanResult, SolverStats


def _is_star(g) -> bool:
    e = g.topological_order[0]
    return all(g.successors[t] == () or t == e for t in g.task_ids) and \
        set(g.successors[e]) == set(g.task_ids) - {e} and \
        all(g.predecessors[t] == (e,) for t in g.task_ids if t != e)


def _m_key(items, more_after: bool):
    # tuple order of the concatenated m: a strict prefix is smaller only when no
    # later task contributes items (then it ends the whole m)
    return tuple(items) + ((("\U0010ffff",),) if more_after else ())


def star_plan(app, profile, request, options: PlannerOptions | None = None, delta: float = 1e-9):
    """plan() on a star DAG as a PlanResult (stats.nodes = exact evaluations).

    Only feasible plans are claimed: when nothing feasible lies within 1.0 of
    the relaxation optimum it raises instead of guessing a diagnosis."""
    options = options or PlannerOptions()
    g = app.graph
    assert _is_star(g), "star_plan needs entry -> leaves"
    entry = g.topological_order[0]
    leaves = sorted(g.successors[entry])          # id order = path order (paths are sorted)
    pools, truncated = O.build_pools(app, profile, request, options)
    S = request.slice_budget
    slack = request.slack
    ov = dict(request.factor_overrides or {})
    slo = O.slo_eff_of(app)
    a_max = O.a_max_of(g)
    frac = {d: g.path_fractions[(entry, d)] for d in leaves}
    alpha, beta = app.alpha, app.beta
    d0 = float(request.demand_rps)

    # per b0: feasible leaf classes {(slices, acc): [bundles]} and the DP
    per_b0 = []
    for b0 in pools[entry]:
        if not (b0.capacity - d0 * (1.0 + slack) >= 0):
            continue
        classes = []
        ok = True
        for j, d in enumerate(leaves):
            fan = ov[(entry, d)] if (entry, d) in ov else b0.fanout[j]
            dj = 0.0 + d0 * fan
            cl: dict = {}
            if dj == 0.0:
                cl[(0, 1.0)] = [None]
            else:
                for b in pools[d]:
                    if not (b.capacity - dj * (1.0 + slack) >= 0):
                        continue
                    if not (slo - sum([2.0 * b0.latency, 2.0 * b.latency]) >= 0):
                        continue
                    cl.setdefault((b.slices, b.accuracy), []).append(b)
            if not cl:
                ok = False
                break
            classes.append(cl)
        if not ok or b0.slices > S:
            continue
        # F[j][s]: max over leaves j.. of sum frac * acc0 * acc using exactly s slices
        R = S - b0.slices
        F = np.full((len(leaves) + 1, R + 1), -np.inf)
        F[len(leaves), 0] = 0.0
        for j in range(len(leaves) - 1, -1, -1):
            best_at = np.full(R + 1, -np.inf)
            for (s, a) in classes[j]:
                if s <= R:
                    best_at[s] = max(best_at[s], frac[leaves[j]] * (b0.accuracy * a))
            nz = np.nonzero(np.isfinite(best_at))[0]
            for s in nz:
                cand = best_at[s] + F[j + 1, : R + 1 - s]
                F[j, s:] = np.maximum(F[j, s:], cand)
        per_b0.append((b0, classes, F, R))

    ids = sorted(g.task_ids)

    def exact(b0, pick):
        # the m-smallest bundle of every chosen class, task by task in id order
        chosen = {}
        for j, d in enumerate(leaves):
            bs = pick[j]
            if bs == [None]:
                chosen[d] = None
                continue
            pos = ids.index(d)
            more = any(t != d and ids.index(t) > pos and (t == entry or pick[leaves.index(t)] != [None])
                       for t in ids)
            chosen[d] = min(bs, key=lambda b: _m_key(b.items, more))
        m = {(entry, vid, seg, bt): c for (vid, seg, bt), c in b0.items}
        for d, b in chosen.items():
            if b is not None:
                for (vid, seg, bt), c in b.items:
                    m[(d, vid, seg, bt)] = c
        cfg = O.derive(m, app, profile, request.demand_rps, request.factor_overrides)
        vs = O.validate(cfg, app, request)
        if not all(v.passed for v in vs):
            return None
        return cfg, vs

    def est(b0, acc_sum, slices):
        return alpha * (acc_sum / a_max) - beta * slices

    top = -math.inf
    for b0, classes, F, R in per_b0:
        for s in np.nonzero(np.isfinite(F[0]))[0]:
            top = max(top, est(b0, F[0, s], b0.slices + int(s)))
    if top == -math.inf:
        raise RuntimeError("star_plan: no leaf assignment passes the per-leaf verdicts")

    band = delta
    while True:
        floor = top - band
        best = None
        n_exact = 0
        for b0, classes, F, R in per_b0:
            # G[j][r]: best estimate of leaves j.. within r slices
            G = np.full_like(F, -np.inf)
            for j in range(len(leaves) + 1):
                vals = alpha * (F[j] / a_max) - beta * np.arange(R + 1)
                G[j] = np.maximum.accumulate(np.where(np.isfinite(F[j]), vals, -np.inf))
            if G[0, R] - beta * b0.slices < floor - 1e-12:
                continue
            pick = [None] * len(leaves)

            def dfs(j, acc_part, used):
                nonlocal best, n_exact
                rem = R - used
                for (s, a), bs in classes[j].items():
                    if s > rem:
                        continue
                    acc2 = acc_part + frac[leaves[j]] * (b0.accuracy * a)
                    head = alpha * (acc2 / a_max) - beta * (b0.slices + used + s)
                    if j + 1 < len(leaves):
                        # G holds alpha * F / a_max - beta * r; the accuracy sum is additive
                        if head + G[j + 1, rem - s] < floor - 1e-12:
                            continue
                        pick[j] = bs
                        dfs(j + 1, acc2, used + s)
                    else:
                        if head < floor - 1e-12:
                            continue
                        pick[j] = bs
                        hit = exact(b0, pick)
                        n_exact += 1
                        if hit is None:
                            continue
                        key = (hit[0].objective, -hit[0].total_slices)
                        if best is None or key > best[0] or (key == best[0] and hit[0].m < best[1][0].m):
                            best = (key, hit)
                pick[j] = None

            dfs(0, 0.0, 0)
        if best is not None and best[0][0] >= floor + delta:
            cfg, vs = best[1]
            stats = SolverStats(n_exact, 0.0, {t: len(p) for t, p in pools.items()}, tuple(truncated))
            return PlanResult(True, cfg, cfg.objective, a_max, None, vs, stats)
        if band > 1.0:
            # nothing feasible within 1.0 of the real-valued optimum: give up loudly
            raise RuntimeError("star_plan: no feasible plan near the relaxation optimum")
        band *= 16.0
