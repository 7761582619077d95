"""In-graph cost of one E apply at a workload's coarse level (str-Glk, high-order vectors)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402
p = config_problem(sys.argv[1] if len(sys.argv) > 1 else "c4_weak_2049")
for es in (1, 0):
    H = helm.helm_setup(p, {"vectors": "high_order", "coarse_op": "galerkin", "inner_maxit": 8, "coarsest_n": 512, "e_stream": es})
    print(json.dumps({"lib": os.environ.get("HELM_LIB", "default"), "e_stream": es,
                      "apply_E_us": round(H.helm_bench_graph("apply_E", 0, 20), 2)}), flush=True)
    H.close()
