"""One solve of a workload with the bench method (for ncu launch lists / captures): setup, one
solve, print the report.
  python tools/profile_solve.py --workload c1_k400 [--inner-maxit 50] [--coarsest-n 512] [--graph 1]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c1_k100")
ap.add_argument("--vectors", default="high_order")
ap.add_argument("--coarse-op", default="galerkin")
ap.add_argument("--inner-tol", type=float, default=1e-1)
ap.add_argument("--inner-maxit", type=int, default=50)
ap.add_argument("--coarsest-n", type=int, default=512)
ap.add_argument("--inner-restart", type=int, default=0)
ap.add_argument("--maxit", type=int, default=2000)
ap.add_argument("--graph", type=int, default=1)
ap.add_argument("--warm", type=int, default=0)
ap.add_argument("--sstep", type=int, default=0)
ap.add_argument("--sstep-passes", type=int, default=1)
args = ap.parse_args()
p = config_problem(args.workload)
H = helm.helm_setup(p, {"vectors": args.vectors, "coarse_op": args.coarse_op, "inner_tol": args.inner_tol,
                        "inner_maxit": args.inner_maxit, "inner_restart": args.inner_restart, "graph": args.graph, "coarsest_n": args.coarsest_n,
                        "sstep": args.sstep, "sstep_passes": args.sstep_passes})
b = torch.from_numpy(p.b).cuda()
for _ in range(args.warm + 1):
    x, rep = H.solve(b, 1e-6, args.maxit)
torch.cuda.synchronize()
print(json.dumps(rep))
