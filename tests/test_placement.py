"""Placement drop-in (placement.py) against the reference's own placements.

Goldens: tools/make_golden_placement.py ran the reference pack/min_gpus/render
here (tests/golden/placement.json).  jsv_pack / jsv_min_gpus are host code in
libjsv, so these run in the CPU suite.  The behavioural cases mirror the
reference's test_placement.py.
"""

from __future__ import annotations

import json
import os
import random

import pytest

from golden_io import load
from paper_2603_08797_b200.errors import GeometryError
from paper_2603_08797_b200.placement import (
    DEFAULT_GEOMETRY,
    MigGeometry,
    instance_segments,
    load_geometry,
    min_gpus,
    pack,
    render_plan,
)
from paper_2603_08797_b200.profiles import MIG_SLICE_COST, SegmentType

G = load("placement.json")


def segs_of(rows):
    return [SegmentType(m, p) for m, p in rows]


def plan_doc(plan) -> dict:
    return {"gpu_count": plan.gpu_count,
            "placements": [[p.instance, p.mig, p.gpu, p.start, p.width] for p in plan.placements],
            "unplaced": list(plan.unplaced)}


def test_geometry_digest_matches_reference():
    assert DEFAULT_GEOMETRY.digest() == G["default_digest"]
    assert DEFAULT_GEOMETRY.starts("3g") == [(0, 4), (4, 3)]
    assert DEFAULT_GEOMETRY.starts("1g_me") == [(0, 2), (2, 2), (4, 2), (6, 1)]


def test_pack_and_min_gpus_match_reference_goldens():
    exact_used = 0
    for c in G["cases"]:
        segs = segs_of(c["segs"])
        got = pack(segs, c["gpus"], DEFAULT_GEOMETRY, c["budget"])
        assert plan_doc(got) == c["pack"], c
        if "min_gpus" in c:
            assert min_gpus(segs, DEFAULT_GEOMETRY, c["budget"]) == c["min_gpus"], c
        exact_used += bool(c["pack"]["placements"]) and c["gpus"] > 0
    assert exact_used > 100


def test_bundled_plans_pack_like_the_reference_cli():
    for c in G["plans"]:
        segs = segs_of(c["segs"])
        k = min_gpus(segs)
        assert k == c["min_gpus"], c["name"]
        plan = pack(segs, k)
        assert plan_doc(plan) == c["pack"], c["name"]
        assert render_plan(plan) == c["render"], c["name"]


def test_custom_geometry_matches_reference(tmp_path):
    p = tmp_path / "geom.json"
    p.write_text(json.dumps(G["custom_geometry"]))
    geo = load_geometry(p)
    for c in G["custom"]:
        segs = segs_of(c["segs"])
        plan = pack(segs, c["gpus"], geo)
        assert plan_doc(plan) == c["pack"]
        assert min_gpus(segs, geo) == c["min_gpus"]
        assert render_plan(plan, geo) == c["render"]


def test_instance_segments_of_golden_configs():
    from paper_2603_08797_b200.plan_types import Configuration

    for doc in load("plans_bundled.json")[:12]:
        cfg = doc["result"].get("config")
        if not cfg:
            continue
        m = tuple(((e["task"], e["variant"], SegmentType(e["mig"], e["mps"]), e["batch"]), e["count"])
                  for e in cfg["m"])
        fake = Configuration.__new__(Configuration)
        object.__setattr__(fake, "m", m)
        want = tuple(SegmentType(e["mig"], e["mps"]) for e in cfg["m"] for _ in range(e["count"]))
        assert instance_segments(fake) == want


# ----------------------------------------------- reference behavioural cases


def segs(*migs):
    return [SegmentType(m, 1) for m in migs]


def test_geometry_validation_messages():
    with pytest.raises(GeometryError, match="exceeds"):
        MigGeometry(slices_per_gpu=7, placements={**DEFAULT_GEOMETRY.placements, "7g": {1: 7}})
    with pytest.raises(GeometryError, match="below"):
        MigGeometry(slices_per_gpu=7, placements={**DEFAULT_GEOMETRY.placements, "4g": {0: 3}})
    with pytest.raises(GeometryError, match="missing"):
        MigGeometry(slices_per_gpu=7, placements={"1g": {0: 1}})


def test_geometry_json_round_trip_and_bad_file(tmp_path):
    p = tmp_path / "geom.json"
    p.write_text(DEFAULT_GEOMETRY.canonical_json())
    assert load_geometry(p) == DEFAULT_GEOMETRY
    bad = tmp_path / "bad.json"
    bad.write_text('{"profiles": {"1g": "nope"}}')
    with pytest.raises(GeometryError, match="bad geometry file"):
        load_geometry(bad)


def test_packing_known_answers():
    assert pack(segs(*["1g"] * 7), 1).footprint_slices == 7
    plan = pack(segs("4g", "2g", "1g"), 1)
    assert {(p.mig, p.start) for p in plan.placements} == {("4g", 0), ("2g", 4), ("1g", 6)}
    assert len(pack(segs("4g", "4g"), 1).unplaced) == 1 and min_gpus(segs("4g", "4g")) == 2
    assert min_gpus(segs("3g", "3g")) == 1
    plan = pack(segs("3g", "1g", "1g", "1g", "1g"), 1)  # exact search: 3g moves to start 4
    assert plan.fully_placed
    three = next(p for p in plan.placements if p.mig == "3g")
    assert (three.start, three.width) == (4, 3)
    assert min_gpus(segs("3g", "2g", "2g")) == 1
    assert sorted(p.start for p in pack(segs(*["1g_me"] * 4), 1).placements) == [0, 2, 4, 6]
    assert min_gpus(segs(*["1g"] * 28)) == 4
    assert pack(segs(*["1g"] * 28), 4).fully_placed and not pack(segs(*["1g"] * 28), 3).fully_placed
    assert pack([SegmentType("2g", 1), SegmentType("2g", 4)], 1).fully_placed
    assert min_gpus([]) == 0
    with pytest.raises(GeometryError, match="non-negative"):
        pack(segs("1g"), -1)
    assert render_plan(pack(segs("4g", "2g", "1g"), 2)) == "gpu0 |aaaabbc|\ngpu1 |.......|"
    assert "unplaced: 7g/mps1" in render_plan(pack(segs("7g", "7g"), 1))


def test_random_packings_are_geometry_clean():
    rng = random.Random(20240812)
    profiles = list(MIG_SLICE_COST)
    for _ in range(150):
        items = segs(*rng.choices(profiles, k=rng.randint(1, 10)))
        n = rng.randint(1, 6)
        plan = pack(items, n)
        grid = {}
        for p in plan.placements:
            allowed = DEFAULT_GEOMETRY.placements[p.mig]
            assert p.start in allowed and allowed[p.start] == p.width
            for c in range(p.start, p.start + p.width):
                assert (p.gpu, c) not in grid
                grid[(p.gpu, c)] = p.instance
        assert len(plan.placements) + len(plan.unplaced) == len(items)


def test_wide_geometry_matches_reference(tmp_path):
    """48 slices per GPU (64-bit occupancy masks in libjsv): the reference's packings."""
    p = tmp_path / "wide.json"
    p.write_text(json.dumps(G["wide_geometry"]))
    geo = load_geometry(p)
    for c in G["wide"]:
        segs = segs_of(c["segs"])
        assert plan_doc(pack(segs, c["gpus"], geo)) == c["pack"]
        assert min_gpus(segs, geo) == c["min_gpus"]
