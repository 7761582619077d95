"""In-graph cost of the str-Glk E apply (tile vs column-streaming kernel) and of the inner
Arnoldi regions at a workload's sizes, for a few parameter sets.

  python tools/e_probe.py --workload c4_weak_2049 --cols 1,24,48
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
ap.add_argument("--cols", default="1,24,44")
ap.add_argument("--sets", default='[{"e_stream":0,"fuse_dots":1},{"e_stream":1,"fuse_dots":0},{"e_stream":0,"fuse_dots":0}]')
a = ap.parse_args()
p = config_problem(a.workload)
base = {"vectors": "high_order", "coarse_op": "galerkin", "inner_maxit": 200, "inner_restart": 50, "coarsest_n": 512}
for st in json.loads(a.sets):
    H = helm.helm_setup(p, dict(base, **st))
    n1 = H.levels[1][0] * H.levels[1][1]
    row = {"set": st, "apply_E": round(H.helm_bench_graph("apply_E", 0, 20), 2)}
    row["E_GBps"] = round(64 * n1 / (row["apply_E"] * 1e-6) / 1e9, 1)
    for j in [int(c) for c in a.cols.split(",")]:
        row[f"e_dots@{j}"] = round(H.helm_bench_graph("e_dots", j, 4), 2)
        row[f"dcgs@{j}"] = round(H.helm_bench_graph("dcgs", j, 4), 2)
        row[f"inner_iter@{j}"] = round(H.helm_bench_graph("inner_iter", j, 4), 2)
    print(json.dumps(row), flush=True)
    H.close()
