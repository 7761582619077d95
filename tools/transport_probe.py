"""Decomposed c1_k400 at one rank over each transport (one GPU): time per solve, to see what the
exchange machinery costs by itself (with one rank nothing crosses a link)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

p = config_problem("c1_k400")
prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 50, "coarsest_n": 512,
       "dist_levels": 3}
b = torch.from_numpy(p.b).cuda()
for name, kw, extra in (("peer-graph", {"peer_exchange": lambda h: [h]}, {}),
                        ("peer-hostloop", {"peer_exchange": lambda h: [h]}, {"graph": 0}),
                        ("nccl", {"nccl_id": helm.nccl_unique_id()}, {})):
    H = helm.HelmDist(p.nx, p.ny, p.h, p.bc, p.k, 0, 1, params=dict(prm, **extra), **kw)
    H.solve(b, 1e-6, 2000)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, rep = H.solve(b, 1e-6, 2000)
    torch.cuda.synchronize()
    print(json.dumps({"transport": name, "s": round(time.perf_counter() - t0, 4), "outer": rep["outer_iterations"],
                      "kernels": rep["kernels"]}), flush=True)
    H.close()
