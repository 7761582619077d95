"""Outer iteration counts of BASELINE configs[4]'s weak-scaling family (reading R27: N unit squares
stacked in y at h = 1/2048, k = 1280) solved as ONE grid on one GPU with the bench method: what a
decomposed N-GPU solve has to reproduce (the decomposition changes no arithmetic but the order of
the rank sums).  python tools/weak_counts.py 1 2   (WEAK_K / WEAK_NCELLS: a smaller analogue, same kh)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads.media import strip_problem  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [1, 2]:
    p = strip_problem(float(os.environ.get("WEAK_K", "1280")), int(os.environ.get("WEAK_NCELLS", "2048")), n)
    b = torch.from_numpy(p.b).cuda()
    cap = int(os.environ.get("WEAK_CAP", "192")) * (n if os.environ.get("WEAK_CAP_SCALE") else 1)
    prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": cap,
           "inner_restart": int(os.environ.get("WEAK_M", "48")), "coarsest_n": 512, "sstep": 8, "sstep_passes": 1}
    H = helm.helm_setup(p, prm)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = H.solve(b, 1e-6, 1000)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    rr = float(torch.linalg.vector_norm(H.apply_A(x) - b) / torch.linalg.vector_norm(b))
    print(json.dumps({"k": p.meta["k"], "cap": cap, "strips": n, "nx": p.nx, "ny": p.ny, "outer": rep["outer_iterations"],
                      "converged": rep["converged"], "restarts": rep["restarts"], "seconds_incl_capture": round(dt, 2),
                      "inner_total": rep["inner_iterations_total"], "true_relres": rr}), flush=True)
    H.close()
    del b, x
    torch.cuda.empty_cache()
