"""The inner E apply (fused Z^T A Z, k_galerkin_apply) of the c1_k400 hierarchy on level 1, a few
warm launches -- stand-alone timing, or the target of one `ncu --set full -k regex:galerkin` capture."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

p = config_problem("c1_k400")
H = helm.helm_setup(p, {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 50,
                        "coarsest_n": 512})
for flush in (False, True):
    us, nb = H.helm_bench_kernel("apply_E", arg=1, reps=int(sys.argv[1]) if len(sys.argv) > 1 else 20, flush=flush)
    print(json.dumps({"kernel": "apply_E", "level": 1, "flush": flush, "us": round(us, 2), "GBps": round(nb / us / 1e3, 1)}))
print(json.dumps({"graph_region_us": round(H.helm_bench_graph("apply_E", 1, 20), 2)}))
H.close()
