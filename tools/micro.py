"""BASELINE configs[4] microbenchmark kernels on a 16385^2-node Dirichlet grid (16383^2 complex128
unknowns): the A apply and the fused V-cycle legs on level 0, L2 flushed before each launch.
Used stand-alone and under ncu (few launches)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16385)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--kernels", default="apply_A,vc_down,vc_up")
ap.add_argument("--col-pipe", default="0")
args = ap.parse_args()
m = args.n - 2
h = 1.0 / (args.n - 1)
k = torch.full((m, m), 0.625 / h, dtype=torch.float64, device="cuda")
for cp in [int(c) for c in args.col_pipe.split(",")]:
    H = helm.Helm(m, m, h, "dirichlet", k, {"inner_maxit": 2, "col_pipe": cp})
    for name in args.kernels.split(","):
        us, nb = H.helm_bench_kernel(name, arg=0, reps=args.reps, flush=True)
        print(json.dumps({"kernel": name, "col_pipe": cp, "us": round(us, 1), "GBps": round(nb / us / 1e3, 1)}),
              flush=True)
    H.close()
