"""configs[4] traces and the batched analytical day plan (paper_2603_08797_b200.workload)
against tests/golden/day_traffic_840_full.json.gz, written by the reference
(tools/make_golden_full.py day): the 288-bin trace, the predictor's demands, and
run_day's planning decisions (plan at the prediction, memoised max_demand
fallback) for EVERY bin in A+S+T and the three ablations -- the 1,152 plans the
bench's configs[4] extra times."""

from __future__ import annotations

import pytest

from golden_io import load, result_dict


@pytest.fixture(scope="module")
def gold():
    return load("day_traffic_840_full.json.gz")


def test_gen_trace_bit_identical(gold):
    from paper_2603_08797_b200 import workload as W

    a, b, sig, n = gold["shape"]
    tr = W.gen_trace(W.TraceShape(a, b, sig, n), gold["scale"], gold["seed"])
    assert list(tr.demands) == gold["demands"]


def test_predicted_demands_match_reference(gold):
    from paper_2603_08797_b200 import workload as W

    tr = W.DemandTrace(tuple(enumerate(gold["demands"])))
    assert W.predicted_demands(tr, gold["slack"]) == gold["predicted"]


def test_trace_csv_round_trip(tmp_path, gold):
    from paper_2603_08797_b200 import workload as W

    tr = W.DemandTrace(tuple(enumerate(gold["demands"])))
    p = tmp_path / "trace.csv"
    W.save_trace(p, tr)
    assert W.load_trace(p) == tr


@pytest.mark.gpu
@pytest.mark.parametrize("space", ["A+S+T", "S+T", "A+T", "A+S"])
def test_plan_day_matches_reference(gold, space):
    from paper_2603_08797_b200 import workload as W
    from paper_2603_08797_b200 import workloads
    from paper_2603_08797_b200.plan_types import SearchSpace

    app, table = workloads.traffic()
    tr = W.DemandTrace(tuple(enumerate(gold["demands"])))
    day = W.plan_day(app, table, tr, gold["budget"], SearchSpace.from_label(space), gold["slack"])
    assert len(gold["plans"][space]) == len(day) == 288
    for row in gold["plans"][space]:
        d = day[row["bin"]]
        assert d.predicted_rps == gold["predicted"][row["bin"]]
        assert d.used_fallback == row["used_fallback"], row["bin"]
        assert result_dict(d.plan) == row["plan"], row["bin"]


@pytest.mark.gpu
def test_plan_day_parts_match_reference(gold):
    """The ranks' shares (plan_day(part=...), as shard.plan_day_sharded and the
    bench's sharded configs[4] extra use them) reassemble the reference's day."""
    from paper_2603_08797_b200 import workload as W
    from paper_2603_08797_b200 import workloads
    from paper_2603_08797_b200.plan_types import SearchSpace
    from paper_2603_08797_b200.shard import block_range

    app, table = workloads.traffic()
    tr = W.DemandTrace(tuple(enumerate(gold["demands"])))
    sp = SearchSpace.from_label("A+S+T")
    for world in (3, 8):
        day = []
        for r in range(world):
            day += W.plan_day(app, table, tr, gold["budget"], sp, gold["slack"],
                              part=block_range(288, world, r))
        assert [d.bin_index for d in day] == list(range(288))
        for row in gold["plans"]["A+S+T"][::3]:
            d = day[row["bin"]]
            assert d.used_fallback == row["used_fallback"], row["bin"]
            assert result_dict(d.plan) == row["plan"], row["bin"]
