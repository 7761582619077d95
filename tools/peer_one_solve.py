import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2308_06152_b200 import helm
from workloads import config_problem
p = config_problem("c1_k100")
prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 50, "coarsest_n": 512, "dist_levels": 3, "graph": 0}
H = helm.HelmDist(p.nx, p.ny, p.h, p.bc, p.k, 0, 1, params=prm, peer_exchange=lambda h: [h], exchange_at_one_rank=True)
b = torch.from_numpy(p.b).cuda()
x, rep = H.solve(b, 1e-6, 2000)
torch.cuda.synchronize()
print(rep)
