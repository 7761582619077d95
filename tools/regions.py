"""In-graph (warm) cost of the solve's regions and of each kernel of the inner Arnoldi step at a
workload's sizes (helm_bench_graph; the regions replay the solve's own kernels).

  python tools/regions.py --workload c4_weak_2049 --params '{"inner_maxit": 100}' --cols 1,25,50,90
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
ap.add_argument("--params", default="{}")
ap.add_argument("--cols", default="1,25,50,90")
args = ap.parse_args()
p = config_problem(args.workload)
prm = dict({"vectors": "high_order", "coarse_op": "galerkin", "inner_maxit": 100, "coarsest_n": 512},
           **json.loads(args.params))
H = helm.helm_setup(p, prm)
lv = [ny * nx for (ny, nx, _) in H.levels]
print(json.dumps({"workload": args.workload, "levels": [list(x[:2]) for x in H.levels], "params": prm}), flush=True)
for name, arg, reps in (("vcycle", 0, 5), ("vcycle", 1, 20), ("vcycle", 2, 20), ("vcycle", 3, 20),
                        ("apply_E", 0, 20), ("apply_A", 0, 20)):
    print(json.dumps({"region": name, "arg": arg, "us": round(H.helm_bench_graph(name, arg, reps), 2)}), flush=True)
for j in [int(c) for c in args.cols.split(",")]:
    row = {"col": j}
    for name in ("e_dots", "dcgs_reduce", "dcgs_update", "dcgs", "inner_iter"):
        row[name] = round(H.helm_bench_graph(name, j, 4), 2)
    n1 = lv[1]
    row["update_GBps"] = round((16.0 * j + 64) * n1 / (row["dcgs_update"] * 1e-6) / 1e9, 1)
    row["e_dots_GBps"] = round(((64 + 16 * (j + 1) + 16) * n1) / (row["e_dots"] * 1e-6) / 1e9, 1)
    print(json.dumps(row), flush=True)
H.close()
