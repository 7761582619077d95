"""A/B of the cluster-summed pass 1 (helm_params.dots_cluster) on the c1_k400 bench solve."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

p = config_problem("c1_k400")
for dc in (0, 1):
    H = helm.helm_setup(p, {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 50,
                            "coarsest_n": 512, "dots_cluster": dc})
    out = {"dots_cluster": dc}
    for j in (5, 25, 45):
        out[f"dcgs{j}"] = round(H.helm_bench_graph("dcgs", j, 3), 2)
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
    out.update({k: rep[k] for k in ("outer_iterations", "inner_iterations_total", "relres")})
    print(json.dumps(out), flush=True)
    H.close()
