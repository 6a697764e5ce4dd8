"""BASELINE configs[2] on the GPU: max-serviceable demand over the XR app's
64-point latency x accuracy SLO grid, solved in one max_demand_grid call
(speculative probes of every point batched per launch) and, as a second
path, point by point through max_demand().  Every demand, probe count and
final plan must equal the reference's (tests/golden/max_demand_c3.json,
written by tools/make_golden_c3.py from the reference itself)."""

from __future__ import annotations

import pytest

from golden_io import load, profile_of, result_dict

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def grid():
    from paper_2603_08797_b200.model import app_from_dict

    docs = load("max_demand_c3.json")
    return docs, [app_from_dict(d["app"]) for d in docs], profile_of(docs[0])


@pytest.mark.parametrize("strategy", ["auto", "search"])
def test_c3_grid_matches_reference(grid, strategy):
    from paper_2603_08797_b200 import planner as P
    from paper_2603_08797_b200.plan_types import SearchSpace

    docs, apps, table = grid
    P.set_strategy(strategy)
    try:
        res = P.max_demand_grid(apps, table, 28, SearchSpace(True, True, True), 0.05, None, 1e-3)
    finally:
        P.set_strategy("auto")
    for d, r in zip(docs, res):
        assert (r.demand_rps, r.probes) == (d["demand"], d["probes"]), d["name"]
        assert result_dict(r.plan) == d["plan"], d["name"]


def test_c3_points_one_by_one(grid):
    from paper_2603_08797_b200 import planner as P
    from paper_2603_08797_b200.plan_types import SearchSpace

    docs, apps, table = grid
    for d, app in list(zip(docs, apps))[::9]:
        r = P.max_demand(app, table, 28, SearchSpace(True, True, True))
        assert (r.demand_rps, r.probes) == (d["demand"], d["probes"]), d["name"]
        assert result_dict(r.plan) == d["plan"], d["name"]


def test_c3_grid_sharded_points(grid):
    """Points split across 3 'ranks' (shard.block_range) and regathered: the
    sweep's multi-GPU decomposition (no collective on the data path)."""
    from paper_2603_08797_b200 import planner as P
    from paper_2603_08797_b200 import shard
    from paper_2603_08797_b200.plan_types import SearchSpace

    docs, apps, table = grid
    out = [None] * len(apps)
    for r in range(3):
        lo, hi = shard.block_range(len(apps), 3, r)
        out[lo:hi] = P.max_demand_grid(apps[lo:hi], table, 28, SearchSpace(True, True, True))
    for d, r in zip(docs, out):
        assert r.demand_rps == d["demand"], d["name"]


@pytest.mark.parametrize("env", [{"JSV_FEAS_BUDGET": "1"}, {"JSV_FEAS_BUDGET": str(1 << 40)},
                                 {"JSV_NO_FEAS_SWEEP": "1"}, {"JSV_NO_S1DEDUP": "1"}])
def test_c3_grid_probe_paths_agree(grid, env, monkeypatch):
    """The feasibility pre-sweep (every probe undecided -> search; every probe
    decided by the sweep; off) and the per-demand Stage-1 dedupe (off) are pure
    performance paths: the sweep's demands and probe counts stay the reference's."""
    from paper_2603_08797_b200 import planner as P
    from paper_2603_08797_b200.plan_types import SearchSpace

    docs, apps, table = grid
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    res = P.max_demand_grid(apps[::4], table, 28, SearchSpace(True, True, True), 0.05, None, 1e-3)
    for d, r in zip(docs[::4], res):
        assert (r.demand_rps, r.probes) == (d["demand"], d["probes"]), d["name"]
        assert result_dict(r.plan) == d["plan"], d["name"]


def test_c3_grid_device_planned(grid, monkeypatch):
    """The configs[2] grid with the exhaustive Stage 2 planned on the device
    (JSV_DEVICE_PLAN: k_x_plan, no host round trip between the stages), budgeted
    feasibility scans included."""
    from paper_2603_08797_b200 import planner as P
    from paper_2603_08797_b200.plan_types import SearchSpace

    monkeypatch.setenv("JSV_DEVICE_PLAN", "1")
    docs, apps, table = grid
    res = P.max_demand_grid(apps, table, 28, SearchSpace(True, True, True), 0.05, None, 1e-3)
    for d, r in zip(docs, res):
        assert (r.demand_rps, r.probes) == (d["demand"], d["probes"]), d["name"]
        assert result_dict(r.plan) == d["plan"], d["name"]
