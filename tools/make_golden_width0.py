"""Golden plans for pareto_width = 0 (every Stage-1 pool truncated to nothing), written
by the REFERENCE planner here:

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_width0.py

-> tests/golden/plans_width0.json (same case format as tools/make_golden.py)."""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as G  # noqa: E402  (imports the reference from /root/reference)

P = G.P


def main() -> None:
    out = []
    for an in G.BUNDLED:
        app, _, table = G.bundled(an)
        for sp in ("A+S+T", "S+T", "T"):
            req = P.PlanRequest(300.0, 28, P.SearchSpace.from_label(sp))
            out.append(G.case(f"width0_{an}_{sp}", app, table, req, P.PlannerOptions(pareto_width=0),
                              profile_ref=an))
    (G.OUT / "plans_width0.json").write_text(json.dumps(out))
    print("wrote", len(out), "cases")


if __name__ == "__main__":
    main()
