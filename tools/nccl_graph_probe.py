"""NCCL transport at one rank with every rank sum issued (exchange_at_one_rank): the decomposed
solve host-polled vs captured into the CUDA graph with conditional nodes (HELM_NCCL_GRAPH=1)."""
import os, sys, json, time
sys.path.insert(0, '/root/repo')
import torch
from paper_2308_06152_b200 import helm
from workloads import config_problem
p = config_problem(sys.argv[1] if len(sys.argv) > 1 else "c1_k100")
prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 192, "inner_restart": 48,
       "coarsest_n": 512, "sstep": int(sys.argv[2]) if len(sys.argv) > 2 else 0, "sstep_passes": 1, "dist_levels": 3}
for g in (0, 1):
    uid = helm.nccl_unique_id()
    try:
        H = helm.HelmDist(p.nx, p.ny, p.h, p.bc, p.k, 0, 1, nccl_id=uid, params=dict(prm, graph=g), exchange_at_one_rank=True)
        b = torch.from_numpy(p.b).cuda()
        H.solve(b, 1e-6, 3)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        x, rep = H.solve(b, 1e-6, 1000)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(json.dumps({"problem": p.name, "sstep": prm["sstep"], "graph": g, "outer": rep["outer_iterations"], "inner": rep["inner_iterations_total"], "s": round(dt, 3), "graph_param": H.params.graph}), flush=True)
        H.close()
    except Exception as e:
        print("graph", g, "FAILED", repr(e)[:600], flush=True)
