"""In-graph cost (warm) of each fused V-cycle leg per level, and of the V-cycle from level 1,
for several leg settings (col_min_n: column legs from this level size; col_pipe: ring depth).

  python tools/legs_probe.py --workload c4_weak_2049 '{"col_min_n": 1000000}' ...
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4_weak_2049")
ap.add_argument("--levels", default="1,2,3")
ap.add_argument("--out", default="")
ap.add_argument("sets", nargs="*", default=["{}"])
a = ap.parse_args()
p = config_problem(a.workload)
for st in a.sets:
    prm = dict({"vectors": "high_order", "inner_maxit": 10, "coarsest_n": 512}, **json.loads(st))
    H = helm.helm_setup(p, prm)
    row = {"set": json.loads(st), "env": {k: v for k, v in os.environ.items() if k.startswith("HELM_PROBE")}}
    for l in [int(v) for v in a.levels.split(",")]:
        n = H.levels[l][0] * H.levels[l][1]
        for leg in ("vc_down", "vc_up"):
            us = H.helm_bench_graph(leg, l, 20)
            row[f"{leg}{l}"] = round(us, 2)
        row[f"n{l}"] = n
    row["vc1"] = round(H.helm_bench_graph("vcycle", 1, 20), 2)
    row["vc2"] = round(H.helm_bench_graph("vcycle", 2, 20), 2)
    print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "a") as fh:
            fh.write(json.dumps(row) + "\n")
    H.close()
