"""s-step coarse solve (reading R28) against the one-vector form on a workload: time to 1e-6,
outer / inner counts, true residual, per variant (probe).

  python tools/sstep_probe.py [workload] [s:passes ...]     e.g. c4_weak_2049 0 8:2 8:1 6:1
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4_weak_2049"
variants = sys.argv[2:] or ["0", "8:2", "8:1"]
maxit = int(os.environ.get("PROBE_MAXIT", "1000"))
p = config_problem(name)
b = torch.from_numpy(p.b).cuda()
base = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1,
        "inner_maxit": int(os.environ.get("PROBE_CAP", "160")), "inner_restart": int(os.environ.get("PROBE_M", "40")),
        "coarsest_n": 512}
for v in variants:
    s, _, ps = v.partition(":")
    prm = dict(base, sstep=int(s), sstep_passes=int(ps or 2))
    if "PROBE_GRAPH" in os.environ:   # 0: host-polled loops (ncu sees every kernel)
        prm["graph"] = int(os.environ["PROBE_GRAPH"])
    if "PROBE_OUTER" in os.environ:   # fgmres | gcr
        prm["outer"] = os.environ["PROBE_OUTER"]
    if "PROBE_SHIFT" in os.environ:
        prm["sstep_shift"] = float(os.environ["PROBE_SHIFT"])
    H = helm.helm_setup(p, prm)
    H.solve(b, 1e-6, 2)   # capture + warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = H.solve(b, 1e-6, maxit)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    r = H.apply_A(x)
    rr = float(torch.linalg.vector_norm(r - b) / torch.linalg.vector_norm(b))
    print(json.dumps({"workload": name, "sstep": int(s), "passes": int(ps or 2), "outer": rep["outer_iterations"],
                      "converged": rep["converged"], "true_relres": rr, "seconds": round(dt, 3),
                      "inner_total": rep["inner_iterations_total"], "inner_max": rep["inner_iterations_max"],
                      "us_per_inner": round(1e6 * dt / max(1, rep["inner_iterations_total"]), 1),
                      "kernels": rep["kernels"]}), flush=True)
    H.close()
