"""The 8-space sweep (reference CLI `sweep`, cli.py:131-158) over the GPU planner:
the CSV must equal, byte for byte, the one the reference CLI wrote for the
bundled apps (tests/golden/sweep_csv.json, tools/make_golden_sweep.py)."""

from __future__ import annotations

import json

import pytest

from golden_io import load


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["social-media", "traffic-analysis", "ar-assistant"])
def test_sweep_csv_byte_identical(tmp_path, name):
    from paper_2603_08797_b200 import sweep, workloads

    app, table = workloads.bundled(name)
    out = tmp_path / "sweep.csv"
    sweep.write_sweep_csv(out, sweep.sweep_rows(app, table, 28))
    assert out.read_text() == load("sweep_csv.json")[name]["csv"]


@pytest.mark.gpu
def test_sweep_command_line(tmp_path):
    """Files in, CSV out, through the module's command line."""
    from paper_2603_08797_b200 import sweep, workloads
    from paper_2603_08797_b200.model import app_to_dict
    from paper_2603_08797_b200.profiles import save_profile

    app, table = workloads.bundled("ar-assistant")
    (tmp_path / "app.json").write_text(json.dumps(app_to_dict(app)))
    save_profile(table, tmp_path / "profile.csv")
    rc = sweep.main(["--app", str(tmp_path / "app.json"), "--profile", str(tmp_path / "profile.csv"),
                     "--slices", "28", "--out", str(tmp_path / "s.csv")])
    assert rc == 0
    assert (tmp_path / "s.csv").read_text() == load("sweep_csv.json")["ar-assistant"]["csv"]


def test_sweep_columns_match_reference_header():
    from paper_2603_08797_b200 import sweep

    for doc in load("sweep_csv.json").values():
        assert doc["csv"].splitlines()[0] == ",".join(sweep.SWEEP_COLUMNS)
