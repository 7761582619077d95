import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2308_06152_b200 import helm
from workloads import config_problem
p = config_problem("c1_k400")
for cm in (1 << 20, 1 << 16, 1 << 14, 0):
    H = helm.helm_setup(p, {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 50, "coarsest_n": 512, "col_min_n": cm})
    b = torch.from_numpy(p.b).cuda(); x = torch.empty_like(b)
    for _ in range(2): H.solve(b, 1e-6, 2000, x)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(3): _, rep = H.solve(b, 1e-6, 2000, x)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 3
    print("col_min_n", cm, "s/solve", round(dt, 4), rep["outer_iterations"], "vcycle us", round(H.helm_bench_graph("vcycle", 1, 20), 2))
    H.close()
