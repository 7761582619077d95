"""16383^2 microbench legs and whole V-cycle with TMA row staging on / off (in-graph and flushed
single-kernel timings)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_06152_b200 import helm  # noqa: E402

peaks = bench.load_peaks()
n = 16385
m = n - 2
h = 1.0 / (n - 1)
k = torch.full((m, m), 0.625 / h, dtype=torch.float64, device="cuda")
for tma in (3, 1, 0):
    H = helm.Helm(m, m, h, "dirichlet", k, {"inner_maxit": 2, "coarsest_n": 512, "tma": tma})
    row = {"tma": tma}
    for name in ("vc_down", "vc_up"):
        us, nb = H.helm_bench_kernel(name, arg=0, reps=10, flush=True)
        row[name] = {"us": round(us, 1), "frac": round(nb / (us * 1e-6) / 1e9 / peaks["hbm_gbs"], 4)}
    lv = [ny * nx for (ny, nx, _) in H.levels]
    vb = sum(104.0 * lv[l] for l in range(len(lv) - 1)) + 16.0 * lv[-1] ** 2 + 32.0 * lv[-1]
    us = H.helm_bench_graph("vcycle", 0, 5)
    row["vcycle0"] = {"us": round(us, 1), "frac": round(vb / (us * 1e-6) / 1e9 / peaks["hbm_gbs"], 4)}
    print(json.dumps(row), flush=True)
    H.close()
