"""Golden vectors for BASELINE configs[2] (the XR max-demand grid), by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_c3.py

64 points: latency SLO in {800, 1000, 1200, 1400, 1550, 1800, 2000, 2500} ms x
accuracy SLO in {0.80, 0.825, ..., 0.975},
max_demand(app, profile, 28, A+S+T, slack 0.05, rel_tol 1e-3) on the bundled
ar-assistant app and its synthetic profile (seed 13).  Writes
tests/golden/max_demand_c3.json (demand, probe count, final plan, reference ms).
"""

from __future__ import annotations

import dataclasses
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as MG  # noqa: E402

P = MG.P
LAT = (800.0, 1000.0, 1200.0, 1400.0, 1550.0, 1800.0, 2000.0, 2500.0)
ACC = (0.80, 0.825, 0.85, 0.875, 0.90, 0.925, 0.95, 0.975)


def main() -> None:
    xr, _knobs, table = MG.bundled("ar-assistant")
    full = P.SearchSpace(True, True, True)
    out = []
    t_all = time.perf_counter()
    for L in LAT:
        for a in ACC:
            app = dataclasses.replace(xr, latency_slo_ms=L, accuracy_slo=a)
            t0 = time.perf_counter()
            r = P.max_demand(app, table, 28, full)
            out.append({"name": f"c3_{L:g}_{a:g}", "profile_ref": "ar-assistant",
                        "app": MG.app_doc(app), "budget": 28, "space": "A+S+T", "slack": 0.05,
                        "rel_tol": 1e-3, "demand": r.demand_rps, "probes": r.probes,
                        "plan": MG.result_doc(r.plan), "ref_ms": (time.perf_counter() - t0) * 1e3})
            print(L, a, r.demand_rps, r.probes, f"{out[-1]['ref_ms']:.0f} ms", flush=True)
    (MG.OUT / "max_demand_c3.json").write_text(json.dumps(out))
    print("done", f"{time.perf_counter() - t_all:.1f}s")


if __name__ == "__main__":
    main()
