"""Debug: one V-cycle with the TMA column legs on every level of a small grid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import random_field, random_k  # noqa: E402

for (nx, ny, bc, cm) in [(255, 127, "dirichlet", 100000), (255, 127, "dirichlet", 0), (31, 31, "dirichlet", 0),
                         (193, 97, "sommerfeld", 0)]:
    k = random_k((ny, nx), 12, 10, 90)
    H = helm.Helm(nx, ny, 1 / (nx + 1), bc, k, {"col_min_n": cm, "tma": 1})
    u = random_field((ny, nx), 15)
    y = H.vcycle(0, torch.from_numpy(u).cuda())
    torch.cuda.synchronize()
    print("ok", nx, ny, bc, cm, float(y.abs().sum()), flush=True)
    H.close()
