"""The BASELINE.json workloads as inputs to the planner.

configs[1] / [2]: the paper's XR compound DAG (bundled ar-assistant app, synthetic
profile seed 13) and its 64-point latency x accuracy SLO grid.  configs[3]: the
synthetic wide star DAG, which the reference does not ship -- defined here, with
the same generator tools/make_golden.py uses to pin the 3- and 4-task cases to
the reference.  configs[4]: the traffic-analysis app on a 120-GPU (840-slice)
cluster.  Inputs are regenerated from the bundled knobs; nothing is read from
the reference at run time.
"""

from __future__ import annotations

import dataclasses
import functools
import json
import os

from .model import AppSpec, ModelVariant, Task, TaskGraph, app_from_dict
from .profiles import SegmentType, SynthKnobs, knobs_from_dict, synth_profile

# the reference's three bundled apps and their generator knobs (reference
# pkg/src/sliceserve/apps/*.json), shipped with the package
_APPS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "bundled_apps.json")

C3_LATENCY_SLOS_MS = (800.0, 1000.0, 1200.0, 1400.0, 1550.0, 1800.0, 2000.0, 2500.0)
C3_ACCURACY_SLOS = (0.80, 0.825, 0.85, 0.875, 0.90, 0.925, 0.95, 0.975)


@functools.lru_cache(maxsize=None)
def bundled(name: str):
    """(AppSpec, ProfileTable) of a bundled app with its synthetic profile (knobs file)."""
    with open(_APPS) as fh:
        doc = json.load(fh)[name]
    app = app_from_dict(doc["app"])
    return app, synth_profile(app.graph, knobs_from_dict(doc["knobs"]))


def xr():
    """configs[1]: the XR (ar-assistant) DAG, 1,024 profile entries."""
    return bundled("ar-assistant")


def c3_grid(app: AppSpec | None = None) -> list[AppSpec]:
    """configs[2]: the XR app at every (latency SLO, accuracy SLO) of the 8 x 8 grid."""
    app = app if app is not None else xr()[0]
    return [dataclasses.replace(app, latency_slo_ms=L, accuracy_slo=a)
            for L in C3_LATENCY_SLOS_MS for a in C3_ACCURACY_SLOS]


def star(n_tasks: int = 12):
    """configs[3]: star t00 -> t01..t(n-1), 8 variants per task (accuracy 0.70 + 0.03 j,
    fan-out factors 1.0), segments {1g,2g,3g,4g,7g} x mps {1,2}, batches {1,4,16,64},
    uniform path fractions (the last absorbs rounding), SLOs 1500 ms / 0.85, beta 0.035.
    Plan it at PlanRequest(200.0, 84, A+S+T)."""
    names = [f"t{i:02d}" for i in range(n_tasks)]
    tasks = []
    for i, nm in enumerate(names):
        vs = []
        for j in range(8):
            factors = {d: 1.0 for d in names[1:]} if i == 0 else {}
            vs.append(ModelVariant(f"{nm}_v{j}", 0.70 + 0.03 * j, factors))
        tasks.append(Task(nm, tuple(vs)))
    edges = tuple((names[0], d) for d in names[1:])
    k = n_tasks - 1
    fr = {}
    acc = 0.0
    for i, d in enumerate(names[1:]):
        f = 1.0 / k if i < k - 1 else 1.0 - acc
        fr[(names[0], d)] = f
        acc += f
    graph = TaskGraph(tuple(tasks), edges, fr)
    app = AppSpec("star", graph, 1500.0, 0.85, 1.0, 0.035, 20.0, 10.0)
    segs = tuple(SegmentType(m, p) for m in ("1g", "2g", "3g", "4g", "7g") for p in (1, 2))
    base = {v.id: 10.0 + 3.0 * j for t in tasks for j, v in enumerate(t.variants)}
    knobs = SynthKnobs(base, 0.7, 0.65, 0.15, 0.0, 5, {}, segs, (1, 4, 16, 64))
    return app, synth_profile(graph, knobs)


def layered(widths=(1, 4, 4, 3), variants: int = 8):
    """SURVEY 8(d) configs[3] stress variant: a layered DAG (default 1 -> 4 -> 4 -> 3),
    every task feeding every task of the next layer with fan-out factor 1/outdegree
    (demand conserved per layer), uniform path fractions (the last absorbs
    rounding), the star's variants, segments, batches and SLOs.  Plan it at
    PlanRequest(200.0, 84, A+S+T)."""
    layers = []
    k = 0
    for w in widths:
        layers.append([f"l{k + i:02d}" for i in range(w)])
        k += w
    names = [nm for lay in layers for nm in lay]
    succ = {nm: [] for nm in names}
    for a, b in zip(layers, layers[1:]):
        for u in a:
            succ[u] = list(b)
    tasks = []
    for nm in names:
        vs = []
        for j in range(variants):
            f = {d: 1.0 / len(succ[nm]) for d in succ[nm]}
            vs.append(ModelVariant(f"{nm}_v{j}", 0.70 + 0.03 * j, f))
        tasks.append(Task(nm, tuple(vs)))
    edges = tuple((u, d) for u in names for d in succ[u])
    paths = [[u] for u in layers[0]]
    for lay in layers[1:]:
        paths = [p + [d] for p in paths for d in lay]
    fr = {}
    acc = 0.0
    for i, p in enumerate(paths):
        f = 1.0 / len(paths) if i < len(paths) - 1 else 1.0 - acc
        fr[tuple(p)] = f
        acc += f
    graph = TaskGraph(tuple(tasks), edges, fr)
    app = AppSpec("layered", graph, 1500.0, 0.85, 1.0, 0.035, 20.0, 10.0)
    segs = tuple(SegmentType(m, p) for m in ("1g", "2g", "3g", "4g", "7g") for p in (1, 2))
    base = {v.id: 10.0 + 3.0 * j for t in tasks for j, v in enumerate(t.variants)}
    knobs = SynthKnobs(base, 0.7, 0.65, 0.15, 0.0, 5, {}, segs, (1, 4, 16, 64))
    return app, synth_profile(graph, knobs)


def traffic():
    """configs[4]: traffic-analysis (1,280 profile entries); plan at 840 slices."""
    return bundled("traffic-analysis")
