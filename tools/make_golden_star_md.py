"""Golden max_demand results for small configs[3] stars by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_star_md.py 3 4

max_demand(star_n, 84 slices, A+S+T) (planner.py:1125-1175): the feasibility probes
of the bisection -- the path the GPU's fan-out solver answers in verdict mode.
Writes tests/golden/max_demand_star.json (format of tools/make_golden.py's
max_demand cases, the knobs inline)."""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as MG  # noqa: E402

P = MG.P


def main() -> None:
    out_path = MG.OUT / "max_demand_star.json"
    out = json.loads(out_path.read_text()) if out_path.exists() else []
    done = {d["name"] for d in out}
    for n in [int(x) for x in sys.argv[1:]]:
        if f"md_star_{n}" in done:
            continue
        app, table, knobs = MG.star_instance(n)
        sp = P.SearchSpace(True, True, True)
        t0 = time.perf_counter()
        r = P.max_demand(app, table, 84, sp, 0.05, None, 1e-3)
        ms = (time.perf_counter() - t0) * 1e3
        out.append({"name": f"md_star_{n}", "n_tasks": n, "app": MG.app_doc(app),
                    "synth": MG.knobs_doc(knobs), "budget": 84, "space": sp.label, "slack": 0.05,
                    "rel_tol": 1e-3, "demand": r.demand_rps, "probes": r.probes,
                    "plan": MG.result_doc(r.plan), "ref_ms": ms})
        out_path.write_text(json.dumps(out))
        print(n, r.demand_rps, r.probes, f"{ms:.0f} ms", flush=True)


if __name__ == "__main__":
    main()
