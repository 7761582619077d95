"""Per-kernel device time and achieved GB/s (helm_bench_kernel) at a workload's sizes."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c1_k400")
ap.add_argument("--inner-maxit", type=int, default=1000)
ap.add_argument("--nvec", default="1,8,32,128,256,512,1000")
args = ap.parse_args()
p = config_problem(args.workload)
H = helm.helm_setup(p, {"vectors": "high_order", "coarse_op": "galerkin", "inner_maxit": args.inner_maxit,
                        "coarsest_n": 512})
for name, arg, reps in (("vcycle", 0, 50), ("vcycle", 1, 50), ("vcycle", 2, 50), ("vcycle", 3, 50), ("apply_E", 0, 50),
                        ("apply_A", 0, 50), ("dcgs", 1, 10), ("dcgs", 20, 10), ("dcgs", 40, 8)):
    print(json.dumps({"region": name, "arg": arg, "graph_us": round(H.helm_bench_graph(name, arg, reps), 2)}),
          flush=True)
for name in ("apply_A", "vc_down", "vc_up", "apply_E"):
    us, nb = H.helm_bench_kernel(name, 1, 20, True)
    print(json.dumps({"kernel": name, "us": round(us, 2), "GBps": round(nb / us / 1e3, 1)}), flush=True)
for nv in [int(v) for v in args.nvec.split(",")]:
    for name in ("gs_dots", "gs_update"):
        us, nb = H.helm_bench_kernel(name, nv, 10, True)
        print(json.dumps({"kernel": name, "nvec": nv, "us": round(us, 2), "GBps": round(nb / us / 1e3, 1)}), flush=True)
