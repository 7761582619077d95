"""One BASELINE config solved with the bench method under parameter variants (A/B of solver
options on a single case): outer / inner counts, convergence, time.
  python tools/case_probe.py c3_marm_f40_2945 '{"lag_stepb": 0}' '{"lag_stepb": 1}'"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

p = config_problem(sys.argv[1])
for extra in sys.argv[2:]:
    prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 50, "coarsest_n": 512}
    prm.update(json.loads(extra))
    H = helm.helm_setup(p, prm)
    b = torch.from_numpy(p.b).cuda()
    for rnd in range(int(os.environ.get("CASE_SOLVES", "1"))):   # repeated solves on one context
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = H.solve(b, 1e-6, int(os.environ.get("CASE_MAXIT", "400")))
        torch.cuda.synchronize()
        print(json.dumps({"case": sys.argv[1], "params": json.loads(extra), "solve": rnd,
                          "s": round(time.perf_counter() - t0, 3),
                          **{k: rep[k] for k in ("outer_iterations", "converged", "relres", "inner_iterations_total",
                                                 "inner_iterations_max", "restarts")}}), flush=True)
    H.close()
