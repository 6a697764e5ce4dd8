"""CPU-only tests: C-ABI surface, host lowering, numerics helpers, multi-process plumbing."""

from __future__ import annotations

import ctypes as C
import os
import random
import re
import subprocess
import tempfile

import pytest

from golden_io import case_inputs, load
from oracle import planner_oracle as O
from paper_2603_08797_b200 import _lower as LW
from paper_2603_08797_b200 import _native as N
from paper_2603_08797_b200.model import app_from_dict
from paper_2603_08797_b200.profiles import profile_from_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "jsv.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(N.LIB_PATH):
        from paper_2603_08797_b200 import _build
        _build.build()
    return N.load_library()


def header_functions() -> list[str]:
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(jsv_\w+)\(", src, re.M)))


def test_library_exports_every_header_symbol(lib):
    names = header_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
        assert n in N.EXPORTS, f"{n} not bound in _native.EXPORTS"


def test_no_cpu_fallback_without_gpu(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    assert lib.jsv_context_create(0, C.byref(h)) == 4  # JSV_ERR_NODEV
    assert b"no CPU fallback" in lib.jsv_last_error()
    from paper_2603_08797_b200 import planner as P
    from paper_2603_08797_b200.errors import NativeError

    app, table, req, opt = case_inputs(load("plans_bundled.json")[0])
    with pytest.raises(NativeError):
        P.plan(app, table, req, opt)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2603_08797_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", text, re.M), f


C_LAYOUT = r"""
#include <stdio.h>
#include <stddef.h>
#include "jsv.h"
#define P(T) printf(#T " %zu\n", sizeof(T));
#define O(T, f) printf(#T "." #f " %zu\n", offsetof(T, f));
int main(void) {
  P(jsv_problem_desc) P(jsv_request) P(jsv_probe) P(jsv_plan_out) P(jsv_demand_out) P(jsv_stats)
  O(jsv_request, mix) O(jsv_request, feasible_only) O(jsv_probe, uni_min_cost)
  O(jsv_plan_out, items) O(jsv_plan_out, hput) O(jsv_plan_out, lat_margin)
  O(jsv_plan_out, acc_margin) O(jsv_problem_desc, a_max) O(jsv_stats, leaf_work)
  return 0;
}
"""


def test_ctypes_layout_matches_the_c_header():
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "l.c")
        exe = os.path.join(d, "l")
        open(src, "w").write(C_LAYOUT)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    got = dict(line.rsplit(" ", 1) for line in out.strip().splitlines())
    py = {"jsv_problem_desc": N.ProblemDesc, "jsv_request": N.Request, "jsv_probe": N.Probe,
          "jsv_plan_out": N.PlanOut, "jsv_demand_out": N.DemandOut, "jsv_stats": N.Stats}
    for name, cls in py.items():
        assert int(got[name]) == C.sizeof(cls), name
    for key, val in got.items():
        if "." in key:
            s, f = key.split(".")
            assert int(val) == getattr(py[s], f).offset, key


def pysum_restated(xs):
    """The device PySum (jsv_internal.cuh): CPython 3.12 sum() of floats from int 0."""
    if not xs:
        return 0
    f, c = 0.0 + xs[0], 0.0
    for x in xs[1:]:
        t = f + x
        if abs(f) >= abs(x):
            c += (f - t) + x
        else:
            c += (x - t) + f
        f = t
    if c and c == c and abs(c) != float("inf"):
        f += c
    return f


def test_device_pysum_algorithm_matches_cpython_sum():
    rng = random.Random(7)
    differs = 0
    for _ in range(20000):
        xs = [2.0 * rng.uniform(1.0, 900.0) for _ in range(rng.randint(1, 6))]
        assert pysum_restated(xs) == sum(xs)
        naive = 0.0
        for x in xs:
            naive += x
        differs += naive != sum(xs)
    assert differs > 100  # the compensated sum genuinely differs from naive summation


@pytest.mark.parametrize("name", ["social-media", "traffic-analysis", "ar-assistant"])
def test_lowering_ranks_and_subspaces_follow_python_order(name):
    doc = load("apps.json")[name]
    app = app_from_dict(doc["app"])
    table = profile_from_rows(doc["profile"])
    lw = LW.lower(app, table)
    assert lw.ids == sorted(app.graph.task_ids)
    for ti, t in enumerate(lw.ids):
        task = app.graph.task(t)
        keys = lw.keys[ti]
        assert keys == sorted(keys, key=lambda k: (k[0], k[1].mig, k[1].mps, k[2]))
        for a in (0, 1):
            for s in (0, 1):
                rows = O.tuples_of(task, table, O.variants_in(task, bool(a)), O.segments_in(bool(s)))
                got = [keys[i] for i in lw.sub_tuples[ti][2 * a + s]]
                assert got == [(r[0], r[1], r[2]) for r in rows]


def test_uninformed_statics_match_the_oracle():
    for doc in load("plans_bundled.json"):
        app, table, req, opt = case_inputs(doc)
        if req.space.task_graph_informed:
            continue
        lw = LW.lower(app, table)
        st = LW.uninformed_statics(app, table, lw, req)
        lat_b, _, _, weight, floor = O.uninformed_budgets(app, table, req)
        assert st["lat_budget"] == lat_b
        assert st["weight"] == weight
        assert st["floor"] == floor


# ------------------------------------------------------------ multi-process

def _record(feasible, obj, sl, items_per_task):
    out = N.PlanOut()
    out.feasible = out.has_config = int(feasible)
    out.objective = obj
    out.total_slices = sl
    for t, items in enumerate(items_per_task):
        out.n_items[t] = len(items)
        for k, w in enumerate(items):
            out.items[t][k] = w
    return out


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2603_08797_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank 0: (0.5, 7 slices, m = ((0,k1,2),)); rank 1: same objective and slices,
    # m = ((0,k1,1),(1,k0,1)) -> smaller m wins the tie (reference planner.py:850-854)
    mine = [_record(1, 0.5, 7, [[(1 << 16) | 2], []]),
            _record(1, 0.5, 7, [[(1 << 16) | 1], [1]])][rank]
    gathered = shard.all_gather_records(shard.plan_record(mine, 2))
    items = list(range(11))
    mapped = shard.sharded_map(items, lambda xs: [x * x for x in xs])
    q.put((rank, gathered, shard.pick_record(gathered, 2), shard.pick_record(gathered, 2, True),
           mapped))
    dist.destroy_process_group()


def test_gloo_two_rank_record_combine_and_sharded_map():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.Random().randrange(2000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    outs.sort()
    (_, g0, w0, f0, m0), (_, g1, w1, f1, m1) = outs
    assert g0 == g1 and len(g0) == 2 and len(g0[0]) == 3 + 2 * 17
    assert w0 == w1 == 1          # the tie goes to the smaller m
    assert f0 == f1 == 0          # feasible_only: the lowest feasible rank (first DFS leaf)
    assert m0 == m1 == [x * x for x in range(11)]


def test_pick_record_reference_tie_break():
    from paper_2603_08797_b200 import shard

    rec = lambda *a: shard.plan_record(_record(*a), 2)  # noqa: E731
    infeasible = rec(0, 9.0, 1, [[(3 << 16) | 1], []])
    a = rec(1, 0.4, 9, [[(1 << 16) | 1], [(2 << 16) | 1]])
    b = rec(1, 0.4, 8, [[(1 << 16) | 1], [(2 << 16) | 3]])   # fewer slices wins
    c = rec(1, 0.41, 12, [[(5 << 16) | 1], []])              # higher objective wins
    pre = rec(1, 0.4, 8, [[(1 << 16) | 1], []])               # strict prefix of b's m
    assert shard.pick_record([infeasible, infeasible], 2) is None
    assert shard.pick_record([infeasible, a, b], 2) == 2
    assert shard.pick_record([a, c, b], 2) == 1
    assert shard.pick_record([b, pre], 2) == 1
    assert shard.pick_record([infeasible, a, c], 2, feasible_only=True) == 1
    # every bit of the objective survives the wire format
    words = rec(1, -0.1234567890123, 3, [[7], [8]])
    assert shard._record_key(words, 2)[0] == -0.1234567890123


def test_block_range_partitions_exactly():
    from paper_2603_08797_b200.shard import block_range

    for n in range(0, 40):
        for w in range(1, 9):
            spans = [block_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_workloads_star_matches_golden_generator():
    """configs[3]'s in-repo generator reproduces the star cases pinned to the reference."""
    from golden_io import load, profile_of

    from paper_2603_08797_b200 import workloads
    from paper_2603_08797_b200.model import app_from_dict
    from paper_2603_08797_b200.profiles import profile_to_rows

    for doc in load("plans_star.json"):
        n = int(doc["name"].split("_")[1])
        app, table = workloads.star(n)
        assert app == app_from_dict(doc["app"])
        assert profile_to_rows(table) == profile_to_rows(profile_of(doc))


def test_workloads_c3_grid_matches_golden_slos():
    from golden_io import load

    from paper_2603_08797_b200 import workloads

    grid = workloads.c3_grid()
    docs = load("max_demand_c3.json")
    assert [(a.latency_slo_ms, a.accuracy_slo) for a in grid] == \
        [(d["app"]["slo"]["latency_ms"], d["app"]["slo"]["accuracy_frac"]) for d in docs]


def _gloo_plan_sharded_worker(rank, world, port, q):
    """plan_sharded's host pipeline on 4 gloo ranks with the GPU calls faked:
    solve_records (the shard's jsv_plan_batch_shard), derive_record (jsv_derive of
    the winner) and decode_records (the result decoder) are recorded, so the test
    sees exactly which shard record every rank adopts."""
    import types

    import torch.distributed as dist

    from paper_2603_08797_b200 import planner, shard
    from paper_2603_08797_b200.plan_types import PlannerOptions

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank 0 and 2 tie on (objective, slices) and differ in m (rank 2's is smaller);
    # rank 1 has fewer slices at a lower objective; rank 3's shard is infeasible
    local = {0: _record(1, 0.5, 7, [[(4 << 16) | 2], []]),
             1: _record(1, 0.4, 3, [[(0 << 16) | 1], []]),
             2: _record(1, 0.5, 7, [[(1 << 16) | 2], []]),
             3: _record(0, 0.0, 0, [[], []])}[rank]
    local.pool_size[0] = 100 + rank
    seen = {}
    lw = types.SimpleNamespace(ids=["a", "b"])

    def solve_records(app, prof, reqs, opt=None, apps=None, device=None, shard=None):
        seen["shard"] = shard
        return [local], lw, None

    def derive_record(app, prof, lw_, req, n_items, items):
        seen["derived"] = (list(n_items[:2]), [list(items[0][:1]), list(items[1][:1])])
        return _record(1, 0.5, 7, [[items[0][0]], []])

    planner.solve_records = solve_records
    planner.derive_record = derive_record
    planner.decode_records = lambda outs, app, lw_, reqs, wall=0.0: [
        (outs[0].objective, outs[0].total_slices, outs[0].items[0][0], outs[0].pool_size[0])]
    res = shard.plan_sharded(None, None, None)
    derived = seen.pop("derived", None)
    res_first = shard.plan_sharded(None, None, None, PlannerOptions(feasible_only=True))
    q.put((rank, seen["shard"], derived, res, res_first))
    dist.destroy_process_group()


def test_gloo_four_rank_plan_sharded_combine():
    """plan_sharded: each rank sweeps its shard, ONE all-gather of the fixed-size
    records, the reference tie-break (objective, slices, m) on every rank, the
    winner re-derived where it is not local; an infeasible shard never wins."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.Random().randrange(2000, 4000)
    procs = [ctx.Process(target=_gloo_plan_sharded_worker, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, sh, derived, res, res_first in outs:
        assert sh == (rank, 4)
        # the winner is rank 2's record: objective 0.5, 7 slices, item (1 << 16) | 2;
        # Stage-1 statistics (pool sizes) stay the local rank's
        assert res == (0.5, 7, (1 << 16) | 2, 100 + rank)
        assert (derived is None) == (rank == 2)
        # feasible_only: the lowest feasible rank (0) holds the first DFS leaf
        assert res_first[:3] == (0.5, 7, (4 << 16) | 2)


def test_profile_csv_byte_identical_to_reference(tmp_path):
    """Profile ingestion: our save_profile writes the reference's
    bytes (digests from tools/make_golden_profiles.py) and load_profile reads them back."""
    import hashlib

    from golden_io import load

    from paper_2603_08797_b200 import workloads
    from paper_2603_08797_b200.profiles import load_profile, profile_to_rows, save_profile

    for name, doc in load("profile_csv.json").items():
        _app, table = workloads.bundled(name)
        p = tmp_path / f"{name}.csv"
        save_profile(table, p)
        data = p.read_bytes()
        assert hashlib.sha256(data).hexdigest() == doc["sha256"], name
        assert profile_to_rows(load_profile(p)) == profile_to_rows(table)


def _legacy_result(out, app, lw, request):
    """The per-field decode (_config_from/_verdicts_from) the batch decoder replaced."""
    from paper_2603_08797_b200 import planner as P
    from paper_2603_08797_b200.plan_types import PlanResult, SolverStats

    g = app.graph
    sizes, cut = {}, []
    for t in g.topological_order:
        ti = lw.index[t]
        if out.pool_present[ti]:
            sizes[t] = int(out.pool_size[ti])
            if out.truncated[ti]:
                cut.append(t)
    stats = SolverStats(int(out.nodes), 0.0, sizes, tuple(cut))
    if not out.has_config:
        return PlanResult(False, None, None, lw.a_max, P._binding(out.binding), (), stats)
    cfg = P._config_from(out, app, lw, request.demand_rps)
    vs = P._verdicts_from(out, app, lw)
    if out.feasible:
        return PlanResult(True, cfg, cfg.objective, lw.a_max, None, vs, stats)
    return PlanResult(False, cfg, None, lw.a_max, P._binding(out.binding), vs, stats)


@pytest.mark.parametrize("name", ["ar-assistant", "traffic-analysis"])
def test_batch_decode_equals_per_field_decode(name):
    """planner._results_from (numpy view, batch-wide) == the per-field ctypes decode."""
    import json

    from paper_2603_08797_b200 import planner as P
    from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace, plan_result_to_dict

    with open(os.path.join(os.path.dirname(__file__), "golden", "apps.json")) as fh:
        doc = json.load(fh)[name]
    app = app_from_dict(doc["app"])
    table = profile_from_rows(doc["profile"])
    lw = LW.lower(app, table)
    rng = random.Random(7)
    n = 24
    outs = (N.PlanOut * n)()
    reqs = []
    T, E, Pn = len(lw.ids), len(lw.edges), len(lw.paths)
    for i, o in enumerate(outs):
        o.has_config = int(i % 5 != 0)
        o.feasible = int(i % 3 != 0)
        o.binding = rng.randrange(-1, 5)
        o.objective, o.a_obj = rng.random(), rng.random()
        o.nodes = rng.randrange(1000)
        o.total_slices = rng.randrange(40)
        o.uncovered_mask = rng.randrange(1 << T) if i % 4 == 0 else 0
        o.res_margin, o.acc_margin = rng.uniform(-5, 5), rng.uniform(-1, 1)
        for ti in range(T):
            o.pool_size[ti] = rng.randrange(500)
            o.pool_present[ti] = rng.randrange(2)
            o.truncated[ti] = rng.randrange(2)
            o.n_items[ti] = rng.randrange(4)
            for k in range(o.n_items[ti]):
                o.items[ti][k] = (rng.randrange(len(lw.keys[ti])) << 16) | rng.randrange(1, 9)
                o.hput[ti][k] = rng.uniform(0, 900)
            o.latency[ti], o.capacity[ti] = rng.uniform(0, 500), rng.uniform(0, 900)
            o.demand[ti], o.accuracy[ti] = rng.uniform(0, 900), rng.random()
            o.slices[ti] = rng.randrange(30)
            o.thr_margin[ti] = rng.uniform(-50, 50)
        for e in range(E):
            o.fanout[e] = rng.uniform(0, 3)
        for p in range(Pn):
            o.path_acc[p], o.lat_margin[p] = rng.random(), rng.uniform(-100, 100)
        reqs.append(PlanRequest(100.0 + i, 28, SearchSpace(True, True, True)))
    got = P._results_from(outs, [app] * n, lw, reqs, 0.0)
    for i in range(n):
        want = _legacy_result(outs[i], app, lw, reqs[i])
        assert got[i] == want
        assert plan_result_to_dict(got[i]) == plan_result_to_dict(want)
        assert repr(got[i]) == repr(want)


@pytest.mark.parametrize("name", ["ar-assistant", "traffic-analysis", "social-media"])
def test_c_decoder_equals_python_decoder(name):
    """csrc/jsv_decode.c builds exactly the objects planner._results_py builds."""
    import json

    from paper_2603_08797_b200 import planner as P
    from paper_2603_08797_b200.plan_types import PlanRequest, SearchSpace, plan_result_to_dict

    assert P._DEC is not None, "the C decoder (_jsvdecode) is not built"
    with open(os.path.join(os.path.dirname(__file__), "golden", "apps.json")) as fh:
        doc = json.load(fh)[name]
    app = app_from_dict(doc["app"])
    lw = LW.lower(app, profile_from_rows(doc["profile"]))
    rng = random.Random(11)
    n = 40
    outs = (N.PlanOut * n)()
    T, E, Pn = len(lw.ids), len(lw.edges), len(lw.paths)
    reqs = []
    for i, o in enumerate(outs):
        o.has_config = int(i % 6 != 0)
        o.feasible = int(i % 3 != 0)
        o.binding = rng.randrange(-1, 5)
        o.objective, o.a_obj = rng.random(), rng.random()
        o.nodes = rng.randrange(1 << 40)
        o.total_slices = rng.randrange(900)
        o.uncovered_mask = rng.randrange(1 << T) if i % 4 == 0 else 0
        o.res_margin = rng.choice([rng.uniform(-5, 5), 0.0, -0.0, float("nan")])
        o.acc_margin = rng.uniform(-1, 1)
        for ti in range(T):
            o.pool_size[ti] = rng.randrange(500)
            o.pool_present[ti] = rng.randrange(2)
            o.truncated[ti] = rng.randrange(2)
            o.n_items[ti] = rng.randrange(N.MAX_ITEMS + 1)
            for k in range(o.n_items[ti]):
                o.items[ti][k] = (rng.randrange(len(lw.keys[ti])) << 16) | rng.randrange(1, 900)
                o.hput[ti][k] = rng.uniform(0, 900)
            o.latency[ti], o.capacity[ti] = rng.uniform(0, 500), rng.uniform(0, 900)
            o.demand[ti], o.accuracy[ti] = rng.uniform(0, 900), rng.random()
            o.slices[ti] = rng.randrange(30)
            o.thr_margin[ti] = rng.uniform(-50, 50)
        for e in range(E):
            o.fanout[e] = rng.uniform(0, 3)
        for p in range(Pn):
            o.path_acc[p], o.lat_margin[p] = rng.random(), rng.uniform(-100, 100)
        reqs.append(PlanRequest(100.0 + i * 0.5, 28, SearchSpace(True, True, True)))
    got = P._results_from(outs, [app] * n, lw, reqs, 1.25)
    want = P._results_py(outs, [app] * n, lw, reqs, 1.25)
    assert len(got) == n
    for g, w in zip(got, want):
        assert repr(g) == repr(w)
        # (json text: NaN margins compare equal as text, not as floats)
        assert json.dumps(plan_result_to_dict(g)) == json.dumps(plan_result_to_dict(w))
        assert type(g) is type(w) and type(g.stats) is type(w.stats)
        if w.config is not None:
            assert g.config.m == w.config.m and list(g.config.hput) == list(w.config.hput)
            assert list(g.config.demand_rps) == list(w.config.demand_rps)
    # leaf objects (verdicts, stats, their tuples) are built untracked by the
    # cyclic GC; a gc pass finds nothing to collect and the values stay intact
    import gc

    for g in got:
        assert all(not gc.is_tracked(v) for v in g.verdicts)
        assert not gc.is_tracked(g.verdicts) and not gc.is_tracked(g.stats)
    gc.collect()
    assert [repr(g) for g in got] == [repr(w) for w in want]
