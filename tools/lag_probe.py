"""A/B of the lagged step B (helm_params.lag_stepb) on the c1_k400 bench solve: time to solution,
outer / inner iteration counts and the in-graph DCGS / inner-iteration regions."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

for wl, itol in (("c1_k400", 0.1), ("c1_k100", 0.1), ("c1_k100", 0.5)):
    p = config_problem(wl)
    for lag in (0, 1):
        H = helm.helm_setup(p, {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": itol, "inner_maxit": 50,
                                "coarsest_n": 512, "lag_stepb": lag})
        out = {"workload": wl, "inner_tol": itol, "lag": lag}
        if wl == "c1_k400":
            out["dcgs25"] = round(H.helm_bench_graph("dcgs", 25, 3), 2)
            out["inner_iter25"] = round(H.helm_bench_graph("inner_iter", 25, 3), 2)
        b = torch.from_numpy(p.b).cuda()
        x = torch.empty_like(b)
        for _ in range(2):
            H.solve(b, 1e-6, 2000, x)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            _, rep = H.solve(b, 1e-6, 2000, x)
        torch.cuda.synchronize()
        out["solve_s"] = round((time.perf_counter() - t0) / 3, 4)
        out.update({k: rep[k] for k in ("outer_iterations", "inner_iterations_total", "inner_iterations_max")})
        out["x_sum"] = float(x.abs().sum())
        print(json.dumps(out), flush=True)
        H.close()
