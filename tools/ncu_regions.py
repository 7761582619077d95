"""ncu target: one instance of a helm_bench_graph region at a workload's sizes (plain graph, no
conditional nodes, so ncu profiles each kernel node).  The first replay is the warm-up launch.

  ncu --set full -c 16 python tools/ncu_regions.py --workload c4_weak_2049 --region inner_iter --col 25
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
ap.add_argument("--region", default="inner_iter")
ap.add_argument("--col", type=int, default=25)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
p = config_problem(a.workload)
prm = dict({"vectors": "high_order", "coarse_op": "galerkin", "inner_maxit": 100, "coarsest_n": 512},
           **json.loads(a.params))
H = helm.helm_setup(p, prm)
print(json.dumps({"region": a.region, "col": a.col, "us": H.helm_bench_graph(a.region, a.col, a.reps)}))
H.close()
