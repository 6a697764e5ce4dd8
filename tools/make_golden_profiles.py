"""Golden digests of the REFERENCE's profile CSV writer (profiles.py:224-257).

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_profiles.py

For each bundled app: synth_profile from its knobs, save_profile to CSV; keeps
the sha256 of the bytes, the row count and the first lines.  Writes
tests/golden/profile_csv.json.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as MG  # noqa: E402

from sliceserve.profiles import save_profile  # noqa: E402


def main() -> None:
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name in MG.BUNDLED:
            _app, _knobs, table = MG.bundled(name)
            p = Path(d) / f"{name}.csv"
            save_profile(table, str(p))
            data = p.read_bytes()
            out[name] = {"sha256": hashlib.sha256(data).hexdigest(), "bytes": len(data),
                         "head": data.decode().splitlines()[:4]}
    (MG.OUT / "profile_csv.json").write_text(json.dumps(out, indent=1))
    print(json.dumps(out, indent=1)[:800])


if __name__ == "__main__":
    main()
