"""GPU parity: the sm_100a planner (through the C-ABI) against the reference goldens.

Bit-exact: chosen allocations (m), feasibility, binding constraint, pool
sizes / truncation, max-serviceable demand and probe counts; every float in
the serialised result is compared with == (the north-star tolerance of 1e-9
relative is not needed because the kernels reproduce CPython's float order).

Every case runs under both Stage-2 strategies: the level-synchronous
branch-and-bound ("search") and the mixed-radix sweep of the whole Stage-1
cross-product ("exhaustive", for solves of at most 2^32 allocations; larger
ones fall back to the search inside the library).
"""

from __future__ import annotations

import pytest

from golden_io import all_plan_cases, case_inputs, load, profile_of, result_dict

pytestmark = pytest.mark.gpu

EXH_LIMIT = 1 << 32


@pytest.fixture(scope="module", params=["search", "exhaustive"])
def P(request):
    from paper_2603_08797_b200 import planner

    planner.set_strategy(request.param, EXH_LIMIT)
    yield planner
    planner.set_strategy("auto")


def _ids(d):
    return d["name"]


@pytest.mark.parametrize("doc", all_plan_cases(), ids=_ids)
def test_plan_matches_reference(P, doc):
    app, table, req, opt = case_inputs(doc)
    got = result_dict(P.plan(app, table, req, opt))
    assert got == doc["result"]


@pytest.mark.parametrize("doc", [d for d in all_plan_cases() if "pools" in d], ids=_ids)
def test_stage1_pools_match_reference(P, doc):
    app, table, req, opt = case_inputs(doc)
    assert P.pool_dump(app, table, req, opt) == doc["pools"]


@pytest.mark.parametrize("doc", load("max_demand.json"), ids=_ids)
def test_max_demand_matches_reference(P, doc):
    from paper_2603_08797_b200.model import app_from_dict
    from paper_2603_08797_b200.plan_types import SearchSpace

    app = app_from_dict(doc["app"])
    r = P.max_demand(app, profile_of(doc), doc["budget"], SearchSpace.from_label(doc["space"]),
                     doc["slack"], None, doc["rel_tol"])
    assert r.demand_rps == doc["demand"]
    assert r.probes == doc["probes"]
    assert result_dict(r.plan) == doc["plan"]
