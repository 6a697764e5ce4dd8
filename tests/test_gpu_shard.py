"""One solve split across shards.

Every shard sweeps a disjoint block of the mixed-radix candidate space
(jsv_plan_batch_shard) and the fixed-size local records are combined with the
reference tie-break (shard.pick_record) and the winner re-derived
(shard.combine_sharded) -- exactly what plan_sharded does after its one
all-gather.  Here the shards run one after another on one GPU and the combine
is applied as every rank would apply it; the result must be the golden one for
every shard count and on every rank.  The last tests launch real
multi-process runs (torchrun x2, both ranks on GPU 0 over gloo: the driver's
boxes have one GPU) of plan_sharded and of the point-sharded sweep."""

from __future__ import annotations

import json
import os
import random
import subprocess
import sys

import pytest

from golden_io import all_plan_cases, case_inputs, load, result_dict

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# T-informed solves (the uninformed planner has no Stage-2 search to shard)
CASES = [d for d in all_plan_cases() if "T" in d["request"]["space"].split("+")]


@pytest.fixture(scope="module")
def env():
    from paper_2603_08797_b200 import planner, shard

    planner.set_strategy("exhaustive", 1 << 32)
    yield planner, shard
    planner.set_strategy("auto")


def _sharded(planner, shard, app, table, req, opt, world):
    outs = []
    for r in range(world):
        o, lw, _ = planner.solve_records(app, table, [req], opt, shard=(r, world))
        outs.append(o[0])
    records = [shard.plan_record(o, len(lw.ids)) for o in outs]
    return [shard.combine_sharded(app, table, req, lw, outs[r], records, bool(opt.feasible_only),
                                  opt)
            for r in range(world)]


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("doc", CASES[::3] + [d for d in CASES if "feasible_only" in d["name"]],
                         ids=lambda d: d["name"])
def test_sharded_solve_matches_reference(env, doc, world):
    planner, shard = env
    app, table, req, opt = case_inputs(doc)
    for res in _sharded(planner, shard, app, table, req, opt, world):
        assert result_dict(res) == doc["result"]


def test_sharded_bench_workload_every_rank_agrees(env):
    """The bench's 64 XR solves (reference goldens, tests/golden/bench_xr64.json) split 4 ways."""
    planner, shard = env
    from paper_2603_08797_b200 import workloads
    from paper_2603_08797_b200.plan_types import PlannerOptions, PlanRequest, SearchSpace

    gold = load("bench_xr64.json")
    app, table = workloads.xr()
    for row in gold["solves"][::7]:
        req = PlanRequest(row["demand"], 28, SearchSpace(True, True, True))
        for res in _sharded(planner, shard, app, table, req, PlannerOptions(), 4):
            assert result_dict(res) == row["result"], row["demand"]


def _torchrun(args: list[str], timeout: int = 600) -> list[dict]:
    port = 20000 + random.Random().randrange(20000)
    env = dict(os.environ, JSV_BENCH_ONE_GPU="1", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tests", "mp_shard_worker.py"), *args]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    return [json.loads(line) for line in p.stdout.splitlines() if line.startswith("{")]


def test_torchrun_two_ranks_plan_sharded():
    lines = _torchrun(["plan"])
    assert sorted(x["rank"] for x in lines) == [0, 1]
    for x in lines:
        assert x["mismatches"] == [], x


def test_torchrun_two_ranks_sharded_sweep():
    lines = _torchrun(["sweep"])
    assert sorted(x["rank"] for x in lines) == [0, 1]
    for x in lines:
        assert x["mismatches"] == [], x


def test_torchrun_two_ranks_sharded_day_trace():
    """configs[4]'s day trace with its bins split over two ranks (shard.plan_day_sharded)."""
    lines = _torchrun(["day"])
    assert sorted(x["rank"] for x in lines) == [0, 1]
    for x in lines:
        assert x["cases"] == 288 and x["mismatches"] == [], x



def test_torchrun_two_rank_bench_line():
    """bench.py's multi-rank path (the driver's SCALE run) on one GPU: two ranks over gloo,
    weak-scaled solves, the sweep and configs[4] sharded, one JSON line from rank 0."""
    port = 20000 + random.Random().randrange(20000)
    env = dict(os.environ, JSV_BENCH_ONE_GPU="1", PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    c4 = d["configs4_traffic840"]
    assert c4["trace_plans"] == 1152 and c4["max_demand_rps"]["A+S+T"] == 65152.0
    assert d["sweep"]["points"] == 64


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_star_fanout_matches_goldens(env, world):
    """Row (e3): the fan-out solver of a wide star split over shards by entry bundle
    (each shard's block of b0, one record combine): the 3..7-task ladder against the
    reference and 8/10/12 tasks against the exact star oracle, on every rank."""
    planner, shard = env
    from paper_2603_08797_b200 import workloads
    from paper_2603_08797_b200.plan_types import PlannerOptions, PlanRequest, SearchSpace

    planner.set_strategy("auto")
    for doc in load("plans_star.json") + load("plans_star_ladder.json"):
        app, table, req, opt = case_inputs(doc)
        for res in _sharded(planner, shard, app, table, req, opt, world):
            assert result_dict(res) == doc["result"], doc["name"]
    for doc in load("plans_star_large.json"):
        app, table = workloads.star(doc["n_tasks"])
        req = PlanRequest(200.0, 84, SearchSpace(True, True, True))
        for res in _sharded(planner, shard, app, table, req, PlannerOptions(), world):
            assert result_dict(res) == doc["result"], doc["n_tasks"]

