"""BASELINE configs[4] strong-scaling grid on one B200 (8191^2 unknowns, k = 1000, h = 1/8192,
Dirichlet point source): outer iterations per second over a bounded number of outer iterations
(the full solve needs hundreds), bench method, FGMRES restarted at the memory cap."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

maxit = int(sys.argv[1]) if len(sys.argv) > 1 else 10
t0 = time.perf_counter()
p = config_problem("c4_strong_8193")
gen = time.perf_counter() - t0
prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 50, "coarsest_n": 512}
t0 = time.perf_counter()
H = helm.helm_setup(p, prm)
b = torch.from_numpy(p.b).cuda()
torch.cuda.synchronize()
setup = time.perf_counter() - t0
H.solve(b, 1e-6, 2)                      # warm (graph capture)
torch.cuda.synchronize()
t0 = time.perf_counter()
_, rep = H.solve(b, 1e-6, maxit)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(json.dumps({"config": "c4_strong_8193", "nx": p.nx, "ny": p.ny, "outer_iterations": rep["outer_iterations"],
                  "relres": rep["relres"], "inner_total": rep["inner_iterations_total"], "seconds": round(dt, 3),
                  "outer_its_per_s": round(rep["outer_iterations"] / dt, 3), "setup_s": round(setup, 2),
                  "input_gen_s": round(gen, 2), "levels": [lv[:2] for lv in H.levels]}), flush=True)
