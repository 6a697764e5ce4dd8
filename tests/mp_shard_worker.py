"""One rank of the multi-process shard tests (tests/test_gpu_shard.py), run by torchrun.

    python -m torch.distributed.run --nproc-per-node 2 ... tests/mp_shard_worker.py plan|sweep

JSV_BENCH_ONE_GPU=1: every rank on GPU 0 with gloo plumbing (one-GPU boxes);
otherwise one GPU per rank over NCCL.  Prints one JSON line per rank with the
golden mismatches it saw.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))


def main() -> None:
    import torch
    import torch.distributed as dist

    mode = sys.argv[1]
    rank = int(os.environ["RANK"])
    local = 0 if os.environ.get("JSV_BENCH_ONE_GPU") == "1" else int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    os.environ["JSV_DEVICE"] = str(local)
    if os.environ.get("JSV_BENCH_ONE_GPU") == "1":
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from golden_io import all_plan_cases, case_inputs, load, result_dict

    from paper_2603_08797_b200 import planner, shard, workloads
    from paper_2603_08797_b200.plan_types import PlannerOptions, PlanRequest, SearchSpace

    bad = []
    if mode == "plan":
        planner.set_strategy("exhaustive", 1 << 32, device=local)
        docs = [d for d in all_plan_cases() if "T" in d["request"]["space"].split("+")][::4]
        for doc in docs:
            app, table, req, opt = case_inputs(doc)
            got = result_dict(shard.plan_sharded(app, table, req, opt, device=local))
            if got != doc["result"]:
                bad.append(doc["name"])
        app, table = workloads.xr()
        for row in load("bench_xr64.json")["solves"][::5]:
            req = PlanRequest(row["demand"], 28, SearchSpace(True, True, True))
            got = result_dict(shard.plan_sharded(app, table, req, PlannerOptions(), device=local))
            if got != row["result"]:
                bad.append(f"bench@{row['demand']}")
        n = len(docs)
    elif mode == "day":
        from paper_2603_08797_b200 import workload as W

        gold = load("day_traffic_840_full.json.gz")
        app, table = workloads.traffic()
        tr = W.DemandTrace(tuple(enumerate(gold["demands"])))
        day = shard.plan_day_sharded(app, table, tr, gold["budget"], SearchSpace(True, True, True),
                                     gold["slack"], device=local)
        for row in gold["plans"]["A+S+T"]:
            d = day[row["bin"]]
            if d.used_fallback != row["used_fallback"] or result_dict(d.plan) != row["plan"]:
                bad.append(f"bin{row['bin']}")
        n = len(day)
    else:
        gold = load("max_demand_c3.json")
        app, table = workloads.xr()
        grid = workloads.c3_grid(app)
        res = shard.sharded_map(grid, lambda pts: planner.max_demand_grid(
            pts, table, 28, SearchSpace(True, True, True), device=local))
        for r, doc in zip(res, gold):
            if (r.demand_rps, r.probes) != (doc["demand"], doc["probes"]) or \
                    result_dict(r.plan) != doc["plan"]:
                bad.append(doc["name"])
        n = len(grid)
    # one write() per line: the ranks share the pipe, and a single write of < PIPE_BUF
    # bytes is not interleaved with the other rank's (print() may split text and newline)
    line = json.dumps({"rank": rank, "world": dist.get_world_size(), "mode": mode, "cases": n,
                       "mismatches": bad}) + "\n"
    os.write(1, line.encode())
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
