"""BASELINE configs[4] strong grid (8191^2, k = 1000) on one B200 with the s-step coarse solve:
convergence within the outer basis that fits the memory, per coarse-solve budget (probe).

  python tools/strong_sstep.py '{"inner_maxit": 1200, "inner_restart": 80}' 60 ...  (params, maxit pairs)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

p = config_problem("c4_strong_8193")
b = torch.from_numpy(p.b).cuda()
args = sys.argv[1:]
for i in range(0, len(args), 2):
    prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "coarsest_n": 512, "sstep": 8,
           "sstep_passes": 1}
    prm.update(json.loads(args[i]))
    maxit = int(args[i + 1])
    H = helm.helm_setup(p, prm)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = H.solve(b, 1e-6, maxit)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    rr = float(torch.linalg.vector_norm(H.apply_A(x) - b) / torch.linalg.vector_norm(b))
    print(json.dumps({"problem": "c4_strong_8193", "nx": p.nx, "params": prm, "maxit": maxit,
                      "outer": rep["outer_iterations"], "converged": rep["converged"], "true_relres": rr,
                      "seconds": round(dt, 2), "inner_total": rep["inner_iterations_total"],
                      "inner_max": rep["inner_iterations_max"], "restarts": rep["restarts"]}), flush=True)
    H.close()
    del x
    torch.cuda.empty_cache()
