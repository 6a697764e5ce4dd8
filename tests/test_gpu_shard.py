"""One solve split across shards: every shard sweeps a
disjoint block of the mixed-radix candidate space (jsv_set_shard) and the
local results are combined with the reference tie-break (shard.pick_sharded).
The shards run one after another on one GPU here -- the combine is exactly
what plan_sharded does after its all-gather -- and the combined result must be
the golden one for every shard count."""

from __future__ import annotations

import pytest

from golden_io import all_plan_cases, case_inputs, result_dict

pytestmark = pytest.mark.gpu

# T-informed solves (the uninformed planner has no Stage-2 search to shard)
CASES = [d for d in all_plan_cases() if "T" in d["request"]["space"].split("+")]


@pytest.fixture(scope="module")
def env():
    from paper_2603_08797_b200 import _native as N
    from paper_2603_08797_b200 import planner, shard

    planner.set_strategy("exhaustive", 1 << 32)
    yield planner, shard, N
    N.set_shard(N.context(), 0, 1)
    planner.set_strategy("auto")


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("doc", CASES[::3], ids=lambda d: d["name"])
def test_sharded_solve_matches_reference(env, doc, world):
    planner, shard, N = env
    app, table, req, opt = case_inputs(doc)
    ctx = N.context()
    parts = []
    try:
        for r in range(world):
            N.set_shard(ctx, r, world)
            parts.append(planner.plan(app, table, req, opt))
    finally:
        N.set_shard(ctx, 0, 1)
    assert result_dict(shard.pick_sharded(parts)) == doc["result"]
