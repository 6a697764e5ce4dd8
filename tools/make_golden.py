"""Generate golden vectors by running the REFERENCE planner in this container.

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden.py

Imports the read-only reference from /root/reference/pkg/src (CPython 3.12.3,
numpy 2.3 -- the same interpreter the GPU box runs, which matters because the
reference's latency verdict uses the 3.12 Neumaier ``sum``).  Writes small
JSON fixtures under tests/golden/; the GPU box never needs the reference.

Every float goes through ``json`` (repr round-trip), so values are exact.
"""

from __future__ import annotations

import json
import math
import random
import sys
import time
from importlib import resources
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.dont_write_bytecode = True

from sliceserve import planner as P  # noqa: E402
from sliceserve.model import AppSpec, ModelVariant, Task, TaskGraph, load_app  # noqa: E402
from sliceserve.profiles import (  # noqa: E402
    ProfileEntry, ProfileTable, SegmentType, SynthKnobs, load_knobs, synth_profile,
)

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"
APPS = resources.files("sliceserve").joinpath("apps")
BUNDLED = ("social-media", "traffic-analysis", "ar-assistant")


# ----------------------------------------------------------------- serialise


def app_doc(app) -> dict:
    g = app.graph
    return {
        "name": app.name,
        "tasks": [{"id": t.id, "variants": [{"id": v.id, "accuracy": v.accuracy} for v in t.variants]}
                  for t in g.tasks],
        "edges": [{"src": s, "dst": d, "factor": {v.id: v.factors[d] for v in g.task(s).variants}}
                  for s, d in g.edges],
        "path_fractions": [{"path": list(p), "fraction": f} for p, f in g.path_fractions.items()],
        "slo": {"latency_ms": app.latency_slo_ms, "accuracy_frac": app.accuracy_slo},
        "objective": {"alpha": app.alpha, "beta": app.beta},
        "staleness_ms": app.staleness_ms,
        "hop_latency_ms": app.hop_latency_ms,
    }


def profile_rows(table) -> list:
    return [[k[0], k[1], k[2].mig, k[2].mps, k[3], table[k].latency_ms, table[k].throughput_rps]
            for k in table]


def request_doc(req) -> dict:
    ov = None
    if req.factor_overrides:
        ov = [[s, d, v] for (s, d), v in sorted(req.factor_overrides.items())]
    return {"demand": req.demand_rps, "budget": req.slice_budget, "space": req.space.label,
            "slack": req.slack, "overrides": ov}


def options_doc(opt) -> dict:
    return {"pareto_width": opt.pareto_width, "exhaustive_limit": opt.exhaustive_limit,
            "eps": opt.eps, "mix_fractions": list(opt.mix_fractions),
            "feasible_only": opt.feasible_only}


def result_doc(res) -> dict:
    d = P.plan_result_to_dict(res)
    d["stats"].pop("nodes")  # traversal-order dependent; not a parity field
    return d


def pools_doc(app, table, req, opt) -> dict:
    s = P._Search(app, table, req, opt)
    out = {}
    for t, pool in s.pools.items():
        out[t] = [
            {"items": [[v, seg.mig, seg.mps, b, c] for (v, seg, b), c in bnd.items],
             "slices": bnd.slices, "capacity": bnd.capacity, "accuracy": bnd.accuracy,
             "latency": bnd.latency, "fanout": list(bnd.fanout)}
            for bnd in pool
        ]
    return out


def bundled(name):
    app = load_app(str(APPS.joinpath(f"{name}.json")))
    knobs = json.loads(APPS.joinpath(f"{name}.knobs.json").read_text())
    table = synth_profile(app.graph, load_knobs(str(APPS.joinpath(f"{name}.knobs.json"))))
    return app, knobs, table


def knobs_doc(k) -> dict:
    return {"base_latency_ms": dict(k.base_latency_ms), "gamma_batch": k.gamma_batch,
            "gamma_slices": k.gamma_slices, "delta": k.delta, "jitter_sigma": k.jitter_sigma,
            "seed": k.seed, "min_slices": dict(k.min_slices),
            "segments": [{"mig": s.mig, "mps": s.mps} for s in k.segments],
            "batches": list(k.batches)}


def case(name, app, table, req, opt=None, with_pools=False, profile_ref=None, bf=False,
         synth=None):
    opt = opt or P.PlannerOptions()
    t0 = time.perf_counter()
    res = P.plan(app, table, req, opt)
    ms = (time.perf_counter() - t0) * 1e3
    doc = {"name": name, "app": app_doc(app), "request": request_doc(req),
           "options": options_doc(opt), "result": result_doc(res), "ref_ms": ms}
    if profile_ref:
        doc["profile_ref"] = profile_ref
    elif synth is not None:
        doc["synth"] = knobs_doc(synth)
    else:
        doc["profile"] = profile_rows(table)
    if with_pools and req.space.task_graph_informed:
        doc["pools"] = pools_doc(app, table, req, opt)
    if bf:
        try:
            want = P.brute_force_plan(app, table, req)
            doc["brute_force"] = {"feasible": want.feasible, "objective": want.objective}
        except Exception as e:  # oracle refusal
            doc["brute_force"] = {"refused": str(e)}
    return doc


def main() -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    started = time.time()

    # ---- bundled apps + their synthetic profiles (pins synth_profile)
    apps = {}
    tables = {}
    appobjs = {}
    for name in BUNDLED:
        app, knobs, table = bundled(name)
        apps[name] = {"app": app_doc(app), "knobs": knobs, "profile": profile_rows(table)}
        tables[name] = table
        appobjs[name] = app
    (OUT / "apps.json").write_text(json.dumps(apps))

    # ---- single plans on bundled apps (configs 1, 2, XR@300, traffic@400 + spaces grid)
    plans = []
    FULL = P.SearchSpace(True, True, True)
    heads = [("C1_social_600", "social-media", 600.0, 28), ("C2_xr_480", "ar-assistant", 480.0, 28),
             ("xr_300", "ar-assistant", 300.0, 28), ("traffic_400", "traffic-analysis", 400.0, 28)]
    for cname, an, dem, bud in heads:
        plans.append(case(cname, appobjs[an], tables[an], P.PlanRequest(dem, bud, FULL),
                          with_pools=True, profile_ref=an))
    for an in BUNDLED:
        for sp in P.ALL_SPACES:
            for dem in (40.0, 250.0, 900.0):
                plans.append(case(f"{an}_{sp.label}_{dem:g}", appobjs[an], tables[an],
                                  P.PlanRequest(dem, 28, sp), profile_ref=an))
    # larger budgets
    for an, dem, bud in (("traffic-analysis", 9000.0, 840), ("ar-assistant", 2000.0, 84),
                         ("social-media", 3000.0, 84)):
        for sp in (FULL, P.SearchSpace(False, True, True), P.SearchSpace(True, False, True),
                   P.SearchSpace(True, True, False)):
            plans.append(case(f"{an}_{sp.label}_{dem:g}_{bud}", appobjs[an], tables[an],
                              P.PlanRequest(dem, bud, sp), profile_ref=an,
                              with_pools=(sp == FULL)))
    # infeasible / diagnostic cases
    import dataclasses
    xr = appobjs["ar-assistant"]
    plans.append(case("xr_excess_demand", xr, tables["ar-assistant"],
                      P.PlanRequest(5000.0, 28, FULL), profile_ref="ar-assistant"))
    plans.append(case("xr_tight_latency", dataclasses.replace(xr, latency_slo_ms=120.0),
                      tables["ar-assistant"], P.PlanRequest(100.0, 28, FULL),
                      profile_ref="ar-assistant"))
    plans.append(case("xr_tight_accuracy", dataclasses.replace(xr, accuracy_slo=0.999),
                      tables["ar-assistant"], P.PlanRequest(100.0, 3, FULL),
                      profile_ref="ar-assistant"))
    plans.append(case("xr_zero_demand", xr, tables["ar-assistant"], P.PlanRequest(0.0, 28, FULL),
                      profile_ref="ar-assistant"))
    plans.append(case("xr_overrides", xr, tables["ar-assistant"],
                      P.PlanRequest(300.0, 28, FULL, 0.1,
                                    {("detect", "describe"): 1.5, ("describe", "speak"): 0.5}),
                      profile_ref="ar-assistant"))
    plans.append(case("traffic_override_zero", appobjs["traffic-analysis"],
                      tables["traffic-analysis"],
                      P.PlanRequest(300.0, 28, FULL, 0.05, {("detect", "classify-incident"): 0.0}),
                      profile_ref="traffic-analysis"))
    plans.append(case("xr_feasible_only", xr, tables["ar-assistant"],
                      P.PlanRequest(480.0, 28, FULL),
                      P.PlannerOptions(feasible_only=True), profile_ref="ar-assistant"))
    plans.append(case("xr_narrow_width", xr, tables["ar-assistant"],
                      P.PlanRequest(480.0, 28, FULL), P.PlannerOptions(pareto_width=64),
                      with_pools=True, profile_ref="ar-assistant"))
    (OUT / "plans_bundled.json").write_text(json.dumps(plans))
    print("bundled plans", len(plans), f"{time.time() - started:.1f}s", flush=True)

    # ---- tiny oracle instances (reference test_planner.py:389-447, test_acceptance.py:63-78)
    from test_planner import _random_tiny_instance
    tiny = []
    for seed in (987654, 20260814):
        rng = random.Random(seed)
        for i in range(100):
            app, table, req = _random_tiny_instance(rng)
            tiny.append(case(f"tiny_{seed}_{i}", app, table, req, bf=True, with_pools=True))
    rng = random.Random(24601)
    for i in range(60):
        app, table, req = _random_tiny_instance(rng)
        budget = rng.randint(2, 30)
        req = P.PlanRequest(rng.uniform(0.0, 400.0), budget, req.space)
        tiny.append(case(f"mixedscale_{i}", app, table, req))
    (OUT / "plans_tiny.json").write_text(json.dumps(tiny))
    print("tiny", len(tiny), f"{time.time() - started:.1f}s", flush=True)

    # ---- mixed instances (reference test_acceptance.py:84-135 generator)
    import test_acceptance as TA
    captured = []
    real_synth = TA.synth_profile

    def capture(graph, knobs):
        captured.append(knobs)
        return real_synth(graph, knobs)

    TA.synth_profile = capture
    mixed = []
    rng = random.Random(31415926)
    for i in range(160):
        app, table, req = TA._random_mixed_instance(rng)
        mixed.append(case(f"mixed_{i}", app, table, req, synth=captured[-1]))
    TA.synth_profile = real_synth
    (OUT / "plans_mixed.json").write_text(json.dumps(mixed))
    print("mixed", len(mixed), f"{time.time() - started:.1f}s", flush=True)

    # ---- star ladder (config 4 reductions)
    stars = []
    for n in (3, 4):
        app, table, knobs = star_instance(n)
        stars.append(case(f"star_{n}", app, table, P.PlanRequest(200.0, 84, FULL), synth=knobs))
    (OUT / "plans_star.json").write_text(json.dumps(stars))
    print("star", f"{time.time() - started:.1f}s", flush=True)

    # ---- max_demand: bundled apps x 8 spaces @ 28 slices, + XR SLO points
    md = []
    for an in BUNDLED:
        for sp in P.ALL_SPACES:
            t0 = time.perf_counter()
            r = P.max_demand(appobjs[an], tables[an], 28, sp)
            md.append({"name": f"{an}_{sp.label}", "profile_ref": an, "app": app_doc(appobjs[an]),
                       "budget": 28, "space": sp.label, "slack": 0.05, "rel_tol": 1e-3,
                       "demand": r.demand_rps, "probes": r.probes, "plan": result_doc(r.plan),
                       "ref_ms": (time.perf_counter() - t0) * 1e3})
        print("md", an, f"{time.time() - started:.1f}s", flush=True)
    for L, a in ((800.0, 0.85), (1550.0, 0.95), (1000.0, 0.8), (2500.0, 0.975)):
        app = dataclasses.replace(xr, latency_slo_ms=L, accuracy_slo=a)
        t0 = time.perf_counter()
        r = P.max_demand(app, tables["ar-assistant"], 28, FULL)
        md.append({"name": f"xr_grid_{L:g}_{a:g}", "profile_ref": "ar-assistant",
                   "app": app_doc(app), "budget": 28, "space": "A+S+T", "slack": 0.05,
                   "rel_tol": 1e-3, "demand": r.demand_rps, "probes": r.probes,
                   "plan": result_doc(r.plan), "ref_ms": (time.perf_counter() - t0) * 1e3})
    # two-task fixture (reference test_planner.py:548-612)
    from test_planner import two_task_fixture
    app, table = two_task_fixture()
    doubled = ProfileTable({k: ProfileEntry(table[k].latency_ms, 2.0 * table[k].throughput_rps)
                            for k in table})
    for tag, tb in (("two_task", table), ("two_task_doubled", doubled)):
        for budget in (6, 21):
            for sp in P.ALL_SPACES:
                r = P.max_demand(app, tb, budget, sp)
                md.append({"name": f"{tag}_{budget}_{sp.label}", "app": app_doc(app),
                           "profile": profile_rows(tb), "budget": budget, "space": sp.label,
                           "slack": 0.05, "rel_tol": 1e-3, "demand": r.demand_rps,
                           "probes": r.probes, "plan": result_doc(r.plan)})
    (OUT / "max_demand.json").write_text(json.dumps(md))
    print("done", f"{time.time() - started:.1f}s", flush=True)


def star_instance(n_tasks: int):
    """Config 4 generator: star t00 -> t01..; 8 variants x 10 segments x 4 batches."""
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
    return app, synth_profile(graph, knobs), knobs


if __name__ == "__main__":
    main()
