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


def test_bench_batch_strategies_agree_at_full_size():
    """The bench workload itself (64 XR solves at 240..712 rps, ~1.9e9
    allocations per batch): the exhaustive sweep, the branch-and-bound and the
    one-at-a-time plan() calls return identical results -- three independent
    traversals of the same space (size-independent parity check at full size),
    and the sweep really evaluated every allocation of every cross-product."""
    import bench
    from paper_2603_08797_b200 import planner
    from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace, plan_result_to_dict

    app, table = bench.xr_inputs()
    reqs = [PlanRequest(d, 28, SearchSpace(True, True, True)) for d in bench.demand_points(64, 0, 1)]

    def strip(r):
        d = plan_result_to_dict(r)
        d["stats"].pop("nodes")
        d["stats"].pop("wall_ms", None)
        return d

    try:
        planner.set_strategy("exhaustive", 1 << 40)
        exh = planner.plan_batch(app, table, reqs)
        st = planner.last_stats()
        covered = sum(bench.covered(app, r, q.demand_rps) for r, q in zip(exh, reqs))
        assert st["exh_candidates"] == covered and st["leaves"] == covered
        planner.set_strategy("search")
        srch = planner.plan_batch(app, table, reqs)
    finally:
        planner.set_strategy("auto")
    one = [planner.plan(app, table, q) for q in reqs[::8]]
    assert all(r.feasible for r in exh)
    assert [strip(r) for r in exh] == [strip(r) for r in srch]
    assert [strip(r) for r in exh[::8]] == [strip(r) for r in one]


@pytest.mark.parametrize("env", [{"JSV_NO_FSORT": "1"}, {"JSV_PAIRS_TILED": "1"},
                                 {"JSV_PAIRS_A1": "1"}, {"JSV_NO_RPL": "1"}, {"JSV_NO_TMA": "1"},
                                 {"JSV_NO_FAST": "1"}, {"JSV_NO_FAST": "1", "JSV_NO_RPL": "1"},
                                 {"JSV_NO_FEAS_SWEEP": "1"}, {"JSV_NO_S1DEDUP": "1"},
                                 {"JSV_S1_LEGACY": "1"}, {"JSV_S1_LEGACY": "1", "JSV_PAIRS_TILED": "1"},
                                 {"JSV_NO_PRUNE": "1"}, {"JSV_NO_MKEY": "1"}, {"JSV_NO_SIDE": "1"},
                                 {"JSV_NO_FANOUT": "1"}, {"JSV_DEVICE_PLAN": "1"},
                                 {"JSV_XROUND": "1"}, {"JSV_XROUND": "32"},
                                 {"JSV_DEVICE_PLAN": "1", "JSV_NO_PRUNE": "1"}, {"JSV_NO_S1CACHE": "1"}])
def test_alternative_kernel_paths_match_reference(env, monkeypatch):
    """Every kernel variant the library can pick (frontier ranks by counting vs by
    sorting, tiled vs barrier-free skyline passes, register vs looped sweep, TMA
    vs plain staging, the float evaluator instead of the rank-space fast path --
    the only path for profiles outside `lat_fast`) reproduces the reference
    goldens, on bundled plans, the bench's demands and max_demand points."""
    from paper_2603_08797_b200 import planner, workloads
    from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    docs = load("plans_bundled.json")
    planner.set_strategy("exhaustive", EXH_LIMIT)
    try:
        for doc in docs[::5] + load("plans_mixed.json")[::10]:
            app, table, req, opt = case_inputs(doc)
            assert result_dict(planner.plan(app, table, req, opt)) == doc["result"], doc["name"]
        app, table = workloads.xr()
        rows = load("bench_xr64.json")["solves"][::4]
        reqs = [PlanRequest(r["demand"], 28, SearchSpace(True, True, True)) for r in rows]
        for r, res in zip(rows, planner.plan_batch(app, table, reqs)):
            assert result_dict(res) == r["result"], r["demand"]
        for doc in load("max_demand_c3.json")[::9]:
            _check_md(planner, doc)
    finally:
        planner.set_strategy("auto")


@pytest.mark.parametrize("env", [{}, {"JSV_S1_SPLIT": "1"}, {"JSV_NO_S1SPLIT": "1"},
                                 {"JSV_NO_S1DEDUP": "1"}, {"JSV_NO_S1DEDUP": "1", "JSV_NO_S1SPLIT": "1"}])
def test_stage1_job_scheduling_matches_reference(env, monkeypatch):
    """Fused Stage-1 job scheduling -- 1,024-thread blocks in largest-demand-first order
    for 148..443 jobs (default), the one-wave split of 1,024- and 512-thread blocks
    (JSV_S1_SPLIT), 512-thread pairs (JSV_NO_S1SPLIT) -- changes no result: the bench's
    64 solves (192 jobs) twice in one batch (192 jobs after Stage-1 dedup, 384 without)."""
    from paper_2603_08797_b200 import planner, workloads
    from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    app, table = workloads.xr()
    rows = load("bench_xr64.json")["solves"]
    reqs = [PlanRequest(r["demand"], 28, SearchSpace(True, True, True)) for r in rows]
    planner.set_strategy("exhaustive", EXH_LIMIT)
    try:
        got = planner.plan_batch(app, table, reqs + reqs)
    finally:
        planner.set_strategy("auto")
    for r, res in zip(rows + rows, got):
        assert result_dict(res) == r["result"], r["demand"]


def test_concurrent_threads_match_reference():
    """Four Python threads calling plan_batch / plan on one device at once (ctypes
    releases the GIL; libjsv serialises calls per context, each thread decodes from
    its own page-locked result buffer): every result equals the reference's."""
    import threading

    from paper_2603_08797_b200 import planner, workloads
    from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace

    app, table = workloads.xr()
    rows = load("bench_xr64.json")["solves"]
    errors = []

    def worker(k):
        try:
            mine = rows[k::4]
            reqs = [PlanRequest(r["demand"], 28, SearchSpace(True, True, True)) for r in mine]
            for _ in range(3):
                for r, res in zip(mine, planner.plan_batch(app, table, reqs)):
                    assert result_dict(res) == r["result"], r["demand"]
                one = planner.plan(app, table, reqs[0])
                assert result_dict(one) == mine[0]["result"]
        except Exception as e:  # noqa: BLE001 -- reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def _check_md(P, doc):
    from paper_2603_08797_b200.model import app_from_dict
    from paper_2603_08797_b200.plan_types import SearchSpace

    r = P.max_demand(app_from_dict(doc["app"]), profile_of(doc), doc["budget"],
                     SearchSpace.from_label(doc["space"]), doc["slack"], None, doc["rel_tol"])
    assert (r.demand_rps, r.probes) == (doc["demand"], doc["probes"]), doc["name"]
    assert result_dict(r.plan) == doc["plan"], doc["name"]


def test_bench_workload_matches_reference(P):
    """The bench step itself: the 64 XR solves (240..712.5 rps) against the reference's
    own results (tests/golden/bench_xr64.json), batched as bench.py runs them and one
    at a time."""
    import bench
    from paper_2603_08797_b200 import workloads
    from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace

    gold = load("bench_xr64.json")
    assert [r["demand"] for r in gold["solves"]] == bench.demand_points(64, 0, 1)
    app, table = workloads.xr()
    reqs = [PlanRequest(r["demand"], 28, SearchSpace(True, True, True)) for r in gold["solves"]]
    got = P.plan_batch(app, table, reqs)
    for r, res in zip(gold["solves"], got):
        assert result_dict(res) == r["result"], r["demand"]
    for r in gold["solves"][::16]:
        res = P.plan(app, table, PlanRequest(r["demand"], 28, SearchSpace(True, True, True)))
        assert result_dict(res) == r["result"], r["demand"]


@pytest.mark.parametrize("doc", load("max_demand_840.json"), ids=_ids)
def test_max_demand_840_slices_matches_reference(doc):
    """configs[4](i): max_demand of traffic-analysis at 840 slices in all 8 spaces."""
    from paper_2603_08797_b200 import planner

    _check_md(planner, doc)


def test_star_through_generic_strategies_matches_reference(monkeypatch):
    """JSV_NO_FANOUT: the star ladder solved by the generic strategies instead of
    the fan-out solver (3-4 tasks: beyond that the level-synchronous B&B's
    frontier outgrows device memory -- the fan-out solver's reason to exist)."""
    from paper_2603_08797_b200 import planner

    monkeypatch.setenv("JSV_NO_FANOUT", "1")
    for doc in (load("plans_star.json") + load("plans_star_ladder.json")):
        app, table, req, opt = case_inputs(doc)
        if len(app.graph.task_ids) > 4:
            continue
        assert result_dict(planner.plan(app, table, req, opt)) == doc["result"], doc["name"]


def test_pareto_width_zero_matches_reference():
    """pareto_width = 0 empties every pool: the reference's dead-task "resources" result
    (tests/golden/plans_width0.json, tools/make_golden_width0.py)."""
    from paper_2603_08797_b200 import planner

    for doc in load("plans_width0.json"):
        app, table, req, opt = case_inputs(doc)
        assert result_dict(planner.plan(app, table, req, opt)) == doc["result"], doc["name"]


def test_pareto_width_out_of_range_is_a_config_error():
    from paper_2603_08797_b200 import planner, workloads
    from paper_2603_08797_b200.errors import ConfigError
    from paper_2603_08797_b200.plan_types import PlannerOptions, PlanRequest, SearchSpace

    app, table = workloads.xr()
    for w in (-1, 40000):
        with pytest.raises(ConfigError, match="pareto_width"):
            planner.plan(app, table, PlanRequest(300.0, 28, SearchSpace(True, True, True)),
                         PlannerOptions(pareto_width=w))


@pytest.mark.parametrize("strategy", ["exhaustive", "search"])
def test_stats_nodes_reported(strategy):
    """SolverStats.nodes is filled per plan (the reference counts _visit calls; here:
    allocations compared one by one in the sweep, or frontier prefixes of the
    level-synchronous search) -- positive for a solved plan, 0 for a dead one."""
    from paper_2603_08797_b200 import planner, workloads
    from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace

    app, table = workloads.xr()
    planner.set_strategy(strategy, 1 << 32)
    try:
        res = planner.plan(app, table, PlanRequest(480.0, 28, SearchSpace(True, True, True)))
    finally:
        planner.set_strategy("auto")
    assert res.feasible and res.stats.nodes > 0


@pytest.mark.parametrize("max_slots", ["1", "64", "4096"])
def test_search_with_split_frontiers_matches_reference(max_slots, monkeypatch):
    """The level-synchronous branch-and-bound with its frontier memory bounded
    (JSV_BB_MAX_SLOTS: a level whose children would exceed it is expanded in halves,
    depth-first, recursively): every bundled / tiny / star golden plan -- optimum, m
    tie-breaks, feasible-only first leaves and infeasible binding constraints -- and
    max_demand results are unchanged by the chunking."""
    from paper_2603_08797_b200 import planner
    from paper_2603_08797_b200.plan_types import SearchSpace

    monkeypatch.setenv("JSV_BB_MAX_SLOTS", max_slots)
    planner.set_strategy("search")
    try:
        docs = load("plans_bundled.json")[::4] + load("plans_tiny.json")[::10] + load("plans_star.json")
        for doc in docs:
            app, table, req, opt = case_inputs(doc)
            assert result_dict(planner.plan(app, table, req, opt)) == doc["result"], doc["name"]
        for doc in load("max_demand.json")[::12]:
            from golden_io import app_from_dict

            app = app_from_dict(doc["app"])
            r = planner.max_demand(app, profile_of(doc), doc["budget"], SearchSpace.from_label(doc["space"]),
                                   doc["slack"], None, doc["rel_tol"])
            assert (r.demand_rps, r.probes) == (doc["demand"], doc["probes"]), doc["name"]
            assert result_dict(r.plan) == doc["plan"], doc["name"]
    finally:
        planner.set_strategy("auto")
