"""A/B of V-cycle build variants (HELM_LIB): fine / inner V-cycle and inner iteration in graph, time to solution."""
import json, os, sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2308_06152_b200 import helm
from workloads import config_problem
p = config_problem("c1_k400")
H = helm.helm_setup(p, {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 50, "coarsest_n": 512})
out = {"lib": os.path.basename(os.environ.get("HELM_LIB", "libhelm.so")), "vc0": round(H.helm_bench_graph("vcycle", 0, 20), 2), "vc1": round(H.helm_bench_graph("vcycle", 1, 20), 2), "inner25": round(H.helm_bench_graph("inner_iter", 25, 3), 2)}
b = torch.from_numpy(p.b).cuda(); x = torch.empty_like(b)
for _ in range(2): H.solve(b, 1e-6, 2000, x)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(3): _, rep = H.solve(b, 1e-6, 2000, x)
torch.cuda.synchronize(); out["solve_s"] = round((time.perf_counter() - t0) / 3, 4); out["outer"] = rep["outer_iterations"]
print(json.dumps(out), flush=True)
