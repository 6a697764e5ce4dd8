"""The 8-space sweep: the reference CLI's
``sweep`` command (cli.py:131-158) over the GPU planner.

For each search space in ``ALL_SPACES`` order (Unopt, T, A, A+T, S, S+T, A+S,
A+S+T): the max-serviceable demand, the share of the slice budget its plan
uses and the ratio to Unopt, written as the same CSV, byte for byte
(``repr`` floats, empty cells where the reference leaves them empty, the
error message of a failed space in the last column).

    python -m paper_2603_08797_b200.sweep --app APP.json --profile PROFILE.csv \
        --slices 28 --out sweep.csv

The run manifest the reference CLI writes next to its artifacts is not
reproduced (CLI plumbing, out of scope).
"""

from __future__ import annotations

import argparse
import csv
import sys
from pathlib import Path

from .errors import NativeError, SliceServeError
from .plan_types import ALL_SPACES

SWEEP_COLUMNS = ("space", "max_demand_rps", "pct_slices_used", "ratio_vs_unopt", "error")


def sweep_rows(app, profile, slices: int, slack: float = 0.05) -> list[list[str]]:
    """Rows of the sweep CSV (reference cli.py:134-151)."""
    from . import planner

    rows = []
    unopt_demand = None
    for space in ALL_SPACES:
        label = space.label
        try:
            best = planner.max_demand(app, profile, slices, space, slack)
            demand = best.demand_rps
            pct = (100.0 * best.plan.config.total_slices / slices
                   if best.plan.config is not None else 0.0)
            if label == "Unopt":
                unopt_demand = demand
            ratio = "" if not unopt_demand else repr(demand / unopt_demand)
            rows.append([label, repr(demand), repr(pct), ratio, ""])
        except NativeError:
            raise  # a GPU/library failure is not a planner outcome
        except SliceServeError as exc:
            rows.append([label, "", "", "", str(exc)])
    return rows


def write_sweep_csv(path: str | Path, rows: list[list[str]]) -> None:
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(SWEEP_COLUMNS)
        writer.writerows(rows)


def main(argv: list[str] | None = None) -> int:
    from .model import load_app
    from .profiles import load_profile

    ap = argparse.ArgumentParser(prog="paper_2603_08797_b200.sweep",
                                 description="max serviceable demand for all 8 search spaces")
    ap.add_argument("--app", required=True, help="application spec JSON")
    ap.add_argument("--profile", required=True, help="profile table CSV")
    ap.add_argument("--slices", type=int, required=True, help="slice budget")
    ap.add_argument("--slack", type=float, default=0.05, help="capacity slack fraction")
    ap.add_argument("--out", required=True, help="write sweep CSV here")
    args = ap.parse_args(argv)
    try:
        rows = sweep_rows(load_app(args.app), load_profile(args.profile), args.slices, args.slack)
        write_sweep_csv(args.out, rows)
    except (SliceServeError, OSError) as exc:
        print(f"sliceserve: error: {exc}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
