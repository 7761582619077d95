"""Every BASELINE.json config on one B200 with the bench method (APD vectors, CSLP (1, 0.5),
coarse CSLP-FGMRES to 1e-1 capped at 50, hierarchy cut at <= 512 unknowns, outer FGMRES to
1e-6 from 0): time to solution, outer / inner iterations, true residual.  configs[1] runs both
coarse options (str-Glk and the re-discretised ReD-Glk2 stencil).  Multi-GPU configs run their
single-GPU piece (the per-GPU block of the weak-scaling run, the whole strong-scaling grid)."""
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
ap.add_argument("--names", default="c0_tiny,c1_k50,c1_k100,c1_k200,c1_k400,c2_wedge_f10,c2_wedge_f20,c2_wedge_f40,"
                                   "c3_marm_f10_2945,c3_marm_f20_2945,c4_weak_2049")
ap.add_argument("--ops", default="galerkin,red_glk2")
ap.add_argument("--maxit", type=int, default=2000)
args = ap.parse_args()
for name in args.names.split(","):
    t0 = time.perf_counter()
    p = config_problem(name)
    gen = time.perf_counter() - t0
    b = torch.from_numpy(p.b).cuda()
    ops = args.ops.split(",") if name.startswith("c1_") else ["galerkin"]
    for op in ops:
        prm = {"vectors": "high_order", "coarse_op": op, "inner_tol": 0.1, "inner_maxit": 50, "coarsest_n": 512}
        try:
            H = helm.helm_setup(p, prm)
            H.solve(b, 1e-6, args.maxit)          # warm-up (graph capture)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            x, rep = H.solve(b, 1e-6, args.maxit)
            dt = time.perf_counter() - t1
            # true residual with the library's own operator
            r = H.apply_A(x)
            rr = float(torch.linalg.vector_norm(r - b) / torch.linalg.vector_norm(b))
            H.close()
            print(json.dumps({"config": name, "op": op, "nx": p.nx, "ny": p.ny, "bc": p.bc,
                              "kh_max": round(p.kh_max, 4), "seconds": round(dt, 4),
                              "outer": rep["outer_iterations"], "converged": rep["converged"],
                              "inner_total": rep["inner_iterations_total"], "true_relres": rr,
                              "its_per_s": round(rep["outer_iterations"] / dt, 1), "input_gen_s": round(gen, 1)}),
                  flush=True)
        except Exception as e:   # report and continue
            print(json.dumps({"config": name, "op": op, "error": str(e)[:200]}), flush=True)
    del b
    torch.cuda.empty_cache()
