"""Time-to-solution of a workload under solver-engine variants (same method, same kernels):
graph vs host-polled loops, single-CTA tail threshold."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c1_k400")
ap.add_argument("--inner-maxit", type=int, default=50)
args = ap.parse_args()
p = config_problem(args.workload)
b = torch.from_numpy(p.b).cuda()
VARIANTS = [{"coarsest_n": 512}, {"coarsest_n": 512, "coop": 0}, {"coarsest_n": 512, "pdl": 0},
            {"coarsest_n": 512, "graph": 0}, {"coarsest_n": 0}]
for v in VARIANTS:
    prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": args.inner_maxit, **v}
    H = helm.helm_setup(p, prm)
    H.solve(b, 1e-6, 2000)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        x, rep = H.solve(b, 1e-6, 2000)
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"variant": v, "seconds": round(min(ts), 4), "outer": rep["outer_iterations"],
                      "inner_total": rep["inner_iterations_total"], "kernels": rep["kernels"],
                      "us_per_inner_it": round(1e6 * min(ts) / max(1, rep["inner_iterations_total"]), 1)}), flush=True)
    H.close()
