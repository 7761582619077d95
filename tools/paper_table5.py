"""PAPER.md Table 5 (wedge problem, APD-preconditioned outer Krylov) on the B200 path: outer
iteration counts for str-Glk and the re-discretised coarse operators, coarse problem solved by
CSLP-FGMRES to 1e-8.  Our wedge interfaces are a reading of Figure 1 (R18), so the
counts are comparable in trend, not digit for digit."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import wedge_problem  # noqa: E402

# PAPER.md lines 973-979 (Table 5): (nodes x, nodes y, f) -> {op: outer}
PAPER = {
    (73, 121, 10): {"galerkin": 7, "red_o2": 22, "red_o4": 22, "red_o6": 22, "red_cmpo4": 22, "red_glk1": 12, "red_glk2": 9},
    (145, 241, 20): {"galerkin": 6, "red_o2": 28, "red_o4": 27, "red_o6": 27, "red_cmpo4": 28, "red_glk1": 12, "red_glk2": 9},
    (289, 481, 20): {"galerkin": 6, "red_o2": 31, "red_o4": 31, "red_cmpo4": 32},
    (289, 481, 40): {"galerkin": 6, "red_o2": 31, "red_o4": 29, "red_o6": 29, "red_cmpo4": 30, "red_glk1": 12, "red_glk2": 9},
    (577, 961, 80): {"galerkin": 6, "red_o2": 37, "red_o4": 30, "red_cmpo4": 31, "red_glk1": 12, "red_glk2": 9},
}
OPS = ["galerkin", "red_o2", "red_o4", "red_o6", "red_cmpo4", "red_glk1", "red_glk2"]
ap = argparse.ArgumentParser()
ap.add_argument("--inner-tol", type=float, default=1e-8)
ap.add_argument("--inner-maxit", type=int, default=2000)
args = ap.parse_args()
res = {}
for (nx, ny, f), ref in PAPER.items():
    p = wedge_problem(float(f), (nx, ny))
    b = torch.from_numpy(p.b).cuda()
    for op in OPS:
        if op not in ref:
            continue
        H = helm.helm_setup(p, {"vectors": "high_order", "coarse_op": op, "inner_tol": args.inner_tol,
                                "inner_maxit": args.inner_maxit})
        t0 = time.perf_counter()
        x, rep = H.solve(b, 1e-6, 300)
        dt = time.perf_counter() - t0
        H.close()
        res[(nx, ny, f, op)] = rep["outer_iterations"]
        print(json.dumps({"grid": f"{nx}x{ny}", "f": f, "op": op, "outer": rep["outer_iterations"],
                          "paper": ref[op], "conv": rep["converged"], "seconds": round(dt, 3)}), flush=True)
print("\n| grid | f | " + " | ".join(OPS) + " |")
print("|---|---|" + "---|" * len(OPS))
for (nx, ny, f), ref in PAPER.items():
    cells = [f"{res[(nx, ny, f, op)]} ({ref[op]})" if (nx, ny, f, op) in res else "-" for op in OPS]
    print(f"| {nx}x{ny} | {f} | " + " | ".join(cells) + " |")
