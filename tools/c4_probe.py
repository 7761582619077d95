"""configs[4] pieces on one GPU: the 2049^2-per-GPU weak-scaling block (k = 1280, Dirichlet,
kh = 0.625) with larger coarse-solve caps, reporting convergence and time (budgeted)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

p = config_problem("c4_weak_2049")
b = torch.from_numpy(p.b).cuda()
for cap, maxit in ((100, 1500), (200, 800), (400, 400)):
    H = helm.helm_setup(p, {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": cap,
                            "coarsest_n": 512})
    t0 = time.perf_counter()
    x, rep = H.solve(b, 1e-6, maxit)
    dt = time.perf_counter() - t0
    r = H.apply_A(x)
    rr = float(torch.linalg.vector_norm(r - b) / torch.linalg.vector_norm(b))
    print(json.dumps({"config": "c4_weak_2049", "inner_maxit": cap, "outer": rep["outer_iterations"],
                      "converged": rep["converged"], "true_relres": rr, "seconds": round(dt, 2),
                      "inner_total": rep["inner_iterations_total"]}), flush=True)
    H.close()
