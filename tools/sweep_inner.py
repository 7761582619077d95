"""Explore the inner coarse-solve setting on the GPU: outer iterations and time-to-solution
for a workload under several (vectors, coarse_op, inner_tol, inner_maxit) choices."""
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
ap.add_argument("--workloads", default="c1_k50,c1_k100,c1_k200,c1_k400")
ap.add_argument("--budget", type=float, default=60.0, help="max seconds per solve")
args = ap.parse_args()
SETTINGS = [
    ("high_order", "galerkin", 1e-1, 1000), ("high_order", "galerkin", 1e-1, 400), ("high_order", "galerkin", 1e-1, 200),
    ("high_order", "galerkin", 1e-1, 100), ("high_order", "galerkin", 1e-1, 50),
    ("high_order", "red_glk2", 1e-1, 1000), ("high_order", "red_glk2", 1e-1, 200), ("high_order", "red_glk2", 1e-1, 100),
    ("bilinear", "galerkin", 1e-1, 200), ("bilinear", "red_o4", 1e-1, 200),
]
for w in args.workloads.split(","):
    p = config_problem(w)
    b = torch.from_numpy(p.b).cuda()
    for vec, op, itol, imax in SETTINGS:
        H = helm.helm_setup(p, {"vectors": vec, "coarse_op": op, "inner_tol": itol, "inner_maxit": imax})
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = H.solve(b, 1e-6, 600)
        dt = time.perf_counter() - t0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = H.solve(b, 1e-6, 600)
        dt = time.perf_counter() - t0
        print(json.dumps({"workload": w, "vectors": vec, "op": op, "inner_tol": itol, "inner_maxit": imax,
                          "outer": rep["outer_iterations"], "conv": rep["converged"],
                          "inner_mean": rep["inner_iterations_total"] / max(1, rep["inner_solves"]),
                          "seconds": round(dt, 4), "kernels": rep["kernels"]}), flush=True)
        H.close()
        if dt > args.budget:
            print(json.dumps({"workload": w, "skip": "budget"}), flush=True)
