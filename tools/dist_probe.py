"""Decomposed solve on ONE GPU with thread ranks (HELM_COMM_THREADS): time per solve of the
c1_k400 bench problem split into P row strips (the ranks share the GPU, so this measures the
decomposition's overhead -- halos, rank sums, all-gathers, host-polled loops -- not scaling),
next to the single-GPU context in host-polled (graph = 0) and graph mode."""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

p = config_problem("c1_k400")
prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 50, "coarsest_n": 512}
b = torch.from_numpy(p.b).cuda()
for graph in (1, 0):
    H = helm.helm_setup(p, dict(prm, graph=graph))
    H.solve(b, 1e-6, 2000)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, rep = H.solve(b, 1e-6, 2000)
    torch.cuda.synchronize()
    print(json.dumps({"ranks": "single", "graph": graph, "s": round(time.perf_counter() - t0, 4),
                      "outer": rep["outer_iterations"]}), flush=True)
    H.close()
for P in (1, 2, 4):
    grp = helm.ThreadGroup(P)
    res = [None] * P

    def work(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            H = helm.HelmDist(p.nx, p.ny, p.h, p.bc, p.k, r, P, group=grp, params=prm, stream=s)
            bo = torch.from_numpy(np.ascontiguousarray(p.b[H.row0:H.row0 + H.nrows])).cuda()
            H.solve(bo, 1e-6, 2000)
            s.synchronize()
            t0 = time.perf_counter()
            _, rep = H.solve(bo, 1e-6, 2000)
            s.synchronize()
            res[r] = (time.perf_counter() - t0, rep["outer_iterations"], rep["kernels"])
            H.close()

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    print(json.dumps({"ranks": P, "transport": "threads", "s": round(max(r[0] for r in res), 4),
                      "outer": res[0][1], "kernels_per_rank": res[0][2]}), flush=True)
    grp.close()
