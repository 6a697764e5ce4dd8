"""Golden sweep CSVs: the REFERENCE CLI's `sweep` command on the bundled apps.

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_sweep.py

For each bundled app: save its synthetic profile with the reference's
save_profile, run `sliceserve.cli sweep --slices 28` (cli.py:131-158) and keep
the CSV bytes.  Writes tests/golden/sweep_csv.json {app: csv text}.
"""

from __future__ import annotations

import json
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as MG  # noqa: E402

from sliceserve import cli as RC  # noqa: E402
from sliceserve.profiles import save_profile  # noqa: E402


def main() -> None:
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name in MG.BUNDLED:
            app, _knobs, table = MG.bundled(name)
            prof = Path(d) / f"{name}.csv"
            save_profile(table, str(prof))
            csv_path = Path(d) / f"{name}.sweep.csv"
            t0 = time.perf_counter()
            rc = RC.main(["sweep", "--app", str(MG.APPS.joinpath(f"{name}.json")), "--profile",
                          str(prof), "--slices", "28", "--out", str(csv_path)])
            out[name] = {"rc": rc, "csv": csv_path.read_text(),
                         "ref_ms": (time.perf_counter() - t0) * 1e3}
            print(name, rc, f"{out[name]['ref_ms']:.0f} ms", flush=True)
    (MG.OUT / "sweep_csv.json").write_text(json.dumps(out))


if __name__ == "__main__":
    main()
