"""Load the golden fixtures (tests/golden/*.json, written by tools/make_golden.py)."""

from __future__ import annotations

import functools
import gzip
import json
import os

from paper_2603_08797_b200.model import app_from_dict
from paper_2603_08797_b200.plan_types import PlannerOptions, PlanRequest, SearchSpace
from paper_2603_08797_b200.profiles import profile_from_rows

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def load(name: str):
    path = os.path.join(GOLDEN, name)
    with (gzip.open(path, "rt") if name.endswith(".gz") else open(path)) as fh:
        return json.load(fh)


@functools.lru_cache(maxsize=None)
def bundled_profile(name: str):
    return profile_from_rows(load("apps.json")[name]["profile"])


def profile_of(doc):
    if "profile_ref" in doc:
        return bundled_profile(doc["profile_ref"])
    if "synth" in doc:
        from paper_2603_08797_b200.model import app_from_dict
        from paper_2603_08797_b200.profiles import knobs_from_dict, synth_profile
        return synth_profile(app_from_dict(doc["app"]).graph, knobs_from_dict(doc["synth"]))
    return profile_from_rows(doc["profile"])


def request_of(r) -> PlanRequest:
    ov = None
    if r.get("overrides"):
        ov = {(s, d): v for s, d, v in r["overrides"]}
    return PlanRequest(r["demand"], r["budget"], SearchSpace.from_label(r["space"]), r["slack"], ov)


def options_of(o) -> PlannerOptions:
    return PlannerOptions(o["pareto_width"], o["exhaustive_limit"], o["eps"],
                          tuple(o["mix_fractions"]), o["feasible_only"])


def case_inputs(doc):
    return app_from_dict(doc["app"]), profile_of(doc), request_of(doc["request"]), options_of(doc["options"])


def result_dict(res) -> dict:
    from paper_2603_08797_b200.plan_types import plan_result_to_dict
    d = plan_result_to_dict(res)
    d["stats"].pop("nodes")
    return d


def pools_dict(pools) -> dict:
    return {
        t: [
            {"items": [[v, seg.mig, seg.mps, b, c] for (v, seg, b), c in bnd.items],
             "slices": bnd.slices, "capacity": bnd.capacity, "accuracy": bnd.accuracy,
             "latency": bnd.latency, "fanout": list(bnd.fanout)}
            for bnd in pool
        ]
        for t, pool in pools.items()
    }


def all_plan_cases():
    out = []
    for f in ("plans_bundled.json", "plans_tiny.json", "plans_mixed.json", "plans_star.json"):
        out.extend(load(f))
    return out
