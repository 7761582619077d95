"""In-graph warm cost of the s-step coarse-solve kernels on a workload's coarse level (probe;
DESIGN.md §6d): pass partials / update per block column J with their algorithmic GB/s, the
reduction, one powers step (V-cycle + E in residual mode), E in residual and plain mode.

  python tools/sstep_regions.py [workload] [s] [m]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4_weak_2049"
s = int(sys.argv[2]) if len(sys.argv) > 2 else 8
m = int(sys.argv[3]) if len(sys.argv) > 3 else 40
p = config_problem(name)
H = helm.helm_setup(p, {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 160,
                        "inner_restart": m, "coarsest_n": 512, "sstep": s, "sstep_passes": 1})
n1 = H.levels[1][0] * H.levels[1][1]
peak = 6547.8
out = {"workload": name, "s": s, "m": m, "variant": os.environ.get("HELM_PROBE_BGS_MMA", "default")}
for J in range(0, m, s):
    rows = J + 1 + s
    us = H.helm_bench_graph("ss_dots", J, 5)
    out[f"dots_J{J}"] = [round(us, 1), round(16.0 * rows * n1 / (us * 1e-6) / 1e9 / peak, 3)]
    us = H.helm_bench_graph("ss_update", J, 5)
    out[f"upd_J{J}"] = [round(us, 1), round(16.0 * (J + 1 + 2 * s) * n1 / (us * 1e-6) / 1e9 / peak, 3)]
out["reduce"] = round(H.helm_bench_graph("ss_reduce", m - s, 10), 1)
out["power"] = round(H.helm_bench_graph("ss_power", 0, 10), 1)
out["E_res"] = round(H.helm_bench_graph("ss_e", 0, 10), 1)
out["E"] = round(H.helm_bench_graph("apply_E", 0, 10), 1)
out["vcycle1"] = round(H.helm_bench_graph("vcycle", 1, 10), 1)
print(json.dumps(out), flush=True)
