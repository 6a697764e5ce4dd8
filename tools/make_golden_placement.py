"""Golden placements from the REFERENCE's placement module (placement.py:150-310).

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_placement.py

Runs the read-only reference in this container and writes
tests/golden/placement.json:
  * pack() of random instance multisets onto random GPU counts (the seeds of
    the reference's own tests plus larger multisets), including tiny node
    budgets so the exhausted-search fallback is pinned;
  * min_gpus() of the same multisets;
  * pack(segments, min_gpus(segments)) of every feasible bundled-app golden plan
    (instance_segments of its configuration: the cli `plan` path, cli.py:173-174);
  * render_plan() strings and one custom geometry.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.dont_write_bytecode = True

from sliceserve.placement import DEFAULT_GEOMETRY, MigGeometry, min_gpus, pack, render_plan  # noqa: E402
from sliceserve.profiles import MIG_SLICE_COST, SegmentType  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"


def plan_doc(plan) -> dict:
    return {"gpu_count": plan.gpu_count,
            "placements": [[p.instance, p.mig, p.gpu, p.start, p.width] for p in plan.placements],
            "unplaced": list(plan.unplaced)}


def main() -> None:
    cases = []
    profiles = list(MIG_SLICE_COST)
    mps = (1, 2, 3, 4)
    for seed, count, kmax, nmax in ((20240812, 150, 10, 6), (20240813, 120, 6, 4),
                                    (424242, 120, 6, 3), (7, 80, 24, 6), (11, 40, 40, 8)):
        rng = random.Random(seed)
        for _ in range(count):
            segs = [SegmentType(rng.choice(profiles), rng.choice(mps))
                    for _ in range(rng.randint(1, kmax))]
            n = rng.randint(0, nmax)
            budget = rng.choice((500_000, 500_000, 40, 3))
            case = {"segs": [[s.mig, s.mps] for s in segs], "gpus": n, "budget": budget,
                    "pack": plan_doc(pack(segs, n, DEFAULT_GEOMETRY, budget))}
            if len(segs) <= 12 or budget != 500_000:
                case["min_gpus"] = min_gpus(segs, DEFAULT_GEOMETRY, budget)
            cases.append(case)
    plans = []
    for doc in json.loads((OUT / "plans_bundled.json").read_text()):
        cfg = doc["result"].get("config")
        if not doc["result"]["feasible"] or not cfg:
            continue
        segs = [SegmentType(e["mig"], e["mps"]) for e in cfg["m"] for _ in range(e["count"])]
        k = min_gpus(segs)
        plans.append({"name": doc["name"], "segs": [[s.mig, s.mps] for s in segs], "min_gpus": k,
                      "pack": plan_doc(pack(segs, k)), "render": render_plan(pack(segs, k))})
    custom = MigGeometry(slices_per_gpu=8, placements={
        "1g": {i: 1 for i in range(8)}, "1g_me": {0: 2, 2: 2, 4: 2, 6: 2},
        "2g": {0: 2, 2: 2, 4: 2, 6: 2}, "3g": {0: 4, 4: 4}, "4g": {0: 4, 4: 4}, "7g": {0: 8}})
    rng = random.Random(99)
    custom_cases = []
    for _ in range(60):
        segs = [SegmentType(rng.choice(profiles), 1) for _ in range(rng.randint(1, 9))]
        n = rng.randint(1, 4)
        custom_cases.append({"segs": [[s.mig, s.mps] for s in segs], "gpus": n,
                             "pack": plan_doc(pack(segs, n, custom)),
                             "min_gpus": min_gpus(segs, custom),
                             "render": render_plan(pack(segs, n, custom), custom)})
    # a wide geometry (48 slices per GPU: six 8-slice blocks of the custom layout),
    # beyond 32-bit occupancy masks
    wide = MigGeometry(slices_per_gpu=48, placements={
        m: {b * 8 + s: w for b in range(6) for s, w in custom.placements[m].items()}
        for m in custom.placements})
    rng = random.Random(4848)
    wide_cases = []
    for _ in range(40):
        segs = [SegmentType(rng.choice(profiles), 1) for _ in range(rng.randint(1, 30))]
        n = rng.randint(1, 3)
        wide_cases.append({"segs": [[s.mig, s.mps] for s in segs], "gpus": n,
                           "pack": plan_doc(pack(segs, n, wide)),
                           "min_gpus": min_gpus(segs, wide)})
    out = {"default_digest": DEFAULT_GEOMETRY.digest(), "cases": cases, "plans": plans,
           "custom_geometry": json.loads(custom.canonical_json()), "custom": custom_cases,
           "wide_geometry": json.loads(wide.canonical_json()), "wide": wide_cases}
    (OUT / "placement.json").write_text(json.dumps(out))
    print(len(cases), "pack cases,", len(plans), "plans,", len(custom_cases), "custom")


if __name__ == "__main__":
    main()
