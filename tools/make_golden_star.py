"""Golden vectors for the configs[3] star ladder (5 and 6 tasks) by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_star.py 5 6

The reference branch-and-bound solves the star DAG up to ~6 tasks (it does
not finish at 12); these points pin the GPU's
large-graph solver.  Writes tests/golden/plans_star_ladder.json.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as MG  # noqa: E402

P = MG.P


def main() -> None:
    out_path = MG.OUT / "plans_star_ladder.json"
    out = json.loads(out_path.read_text()) if out_path.exists() else []
    done = {d["name"] for d in out}
    for n in [int(x) for x in sys.argv[1:]]:
        if f"star_{n}" in done:
            continue
        app, table, knobs = MG.star_instance(n)
        t0 = time.perf_counter()
        doc = MG.case(f"star_{n}", app, table, P.PlanRequest(200.0, 84, P.SearchSpace(True, True, True)),
                      synth=knobs)
        doc["ref_ms"] = (time.perf_counter() - t0) * 1e3
        out.append(doc)
        out_path.write_text(json.dumps(out))
        print(n, doc["result"]["objective"], f"{doc['ref_ms']:.0f} ms", flush=True)


if __name__ == "__main__":
    main()
