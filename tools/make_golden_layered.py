"""Golden plans for small layered DAGs (SURVEY 8(d) configs[3] stress variant) by the
REFERENCE, for the shapes its branch-and-bound finishes:

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_layered.py 1,2,1 1,2,2,1 ...

Same generator as paper_2603_08797_b200.workloads.layered (every task feeds every task
of the next layer with factor 1/outdegree, uniform path fractions, the star's
variants / segments / batches / SLOs), PlanRequest(200.0, 84, A+S+T).  Writes
tests/golden/plans_layered.json."""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as MG  # noqa: E402

P = MG.P


def layered_instance(widths, variants=8):
    layers, k = [], 0
    for w in widths:
        layers.append([f"l{k + i:02d}" for i in range(w)])
        k += w
    names = [nm for lay in layers for nm in lay]
    succ = {nm: [] for nm in names}
    for a, b in zip(layers, layers[1:]):
        for u in a:
            succ[u] = list(b)
    tasks = []
    for nm in names:
        vs = [MG.ModelVariant(f"{nm}_v{j}", 0.70 + 0.03 * j, {d: 1.0 / len(succ[nm]) for d in succ[nm]})
              for j in range(variants)]
        tasks.append(MG.Task(nm, tuple(vs)))
    edges = tuple((u, d) for u in names for d in succ[u])
    paths = [[u] for u in layers[0]]
    for lay in layers[1:]:
        paths = [p + [d] for p in paths for d in lay]
    fr, acc = {}, 0.0
    for i, p in enumerate(paths):
        f = 1.0 / len(paths) if i < len(paths) - 1 else 1.0 - acc
        fr[tuple(p)] = f
        acc += f
    graph = MG.TaskGraph(tuple(tasks), edges, fr)
    app = MG.AppSpec("layered", graph, 1500.0, 0.85, 1.0, 0.035, 20.0, 10.0)
    segs = tuple(MG.SegmentType(m, p) for m in ("1g", "2g", "3g", "4g", "7g") for p in (1, 2))
    base = {v.id: 10.0 + 3.0 * j for t in tasks for j, v in enumerate(t.variants)}
    knobs = MG.SynthKnobs(base, 0.7, 0.65, 0.15, 0.0, 5, {}, segs, (1, 4, 16, 64))
    return app, MG.synth_profile(graph, knobs), knobs


def main() -> None:
    out_path = MG.OUT / "plans_layered.json"
    out = json.loads(out_path.read_text()) if out_path.exists() else []
    done = {d["name"] for d in out}
    for spec in sys.argv[1:]:
        widths = tuple(int(x) for x in spec.split(","))
        name = "layered_" + "-".join(map(str, widths))
        if name in done:
            continue
        app, table, knobs = layered_instance(widths)
        t0 = time.perf_counter()
        doc = MG.case(name, app, table, P.PlanRequest(200.0, 84, P.SearchSpace(True, True, True)),
                      synth=knobs)
        doc["ref_ms"] = (time.perf_counter() - t0) * 1e3
        doc["widths"] = list(widths)
        out.append(doc)
        out_path.write_text(json.dumps(out))
        print(name, doc["result"]["objective"], f"{doc['ref_ms']:.0f} ms", flush=True)


if __name__ == "__main__":
    main()
