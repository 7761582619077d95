"""BASELINE configs on one B200 with the bench method (APD + str-Glk, coarse FGMRES(48) to 1e-1
capped at 192) in the one-vector and the s-step (s = 8, one pass; reading R28) coarse-solve form:
time to 1e-6, outer / inner iterations, true residual (probe)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

names = (sys.argv[1] if len(sys.argv) > 1 else
         "c1_k400,c2_wedge_f40,c3_marm_f20_2945,c3_marm_f40_2945,c3_marm_f20_5889,c3_marm_f40_5889").split(",")
for name in names:
    p = config_problem(name)
    b = torch.from_numpy(p.b).cuda()
    for ss in (0, 8):
        prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 192,
               "inner_restart": 48, "coarsest_n": 512, "sstep": ss, "sstep_passes": 1}
        H = helm.helm_setup(p, prm)
        H.solve(b, 1e-6, 3)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = H.solve(b, 1e-6, 2000)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        rr = float(torch.linalg.vector_norm(H.apply_A(x) - b) / torch.linalg.vector_norm(b))
        print(json.dumps({"config": name, "nx": p.nx, "ny": p.ny, "sstep": ss, "seconds": round(dt, 3),
                          "outer": rep["outer_iterations"], "converged": rep["converged"],
                          "inner_total": rep["inner_iterations_total"], "true_relres": rr}), flush=True)
        H.close()
