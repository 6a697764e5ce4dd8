"""Print the GPU vs golden diff of one named golden plan case (debug helper)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_io import all_plan_cases, case_inputs, result_dict
from paper_2603_08797_b200 import planner as P
for name in sys.argv[1:]:
    doc = [d for d in all_plan_cases() if d["name"] == name][0]
    app, table, req, opt = case_inputs(doc)
    got = result_dict(P.plan(app, table, req, opt))
    want = doc["result"]
    for k in want:
        if got[k] != want[k]:
            print(name, "DIFF", k, "\n  got ", json.dumps(got[k])[:1500], "\n  want", json.dumps(want[k])[:1500])
    print(name, "stats", P.last_stats())
