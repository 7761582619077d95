"""V-cycle from levels 0-3 on the configs[4] weak block for several column-leg thresholds
(col_min_n), ring depths (col_pipe 1: 4 rows, 6: 6 rows, 2: 8 down / 6 up; adaptive segments)
and coarsest-level cuts (in-graph, warm)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

p = config_problem(sys.argv[1] if len(sys.argv) > 1 else "c4_weak_2049")
for cm, cp, cn in ((1 << 20, 1, 512), (1000000, 1, 512), (1000000, 6, 512), (1000000, 2, 512), (200000, 2, 512),
                   (1 << 20, 1, 1000), (1 << 20, 1, 128)):
    H = helm.helm_setup(p, {"vectors": "high_order", "inner_maxit": 10, "coarsest_n": cn, "col_min_n": cm, "col_pipe": cp})
    print(json.dumps({"col_min_n": cm, "col_pipe": cp, "coarsest_n": cn, "vc1": round(H.helm_bench_graph("vcycle", 1, 20), 2),
                      "vc0": round(H.helm_bench_graph("vcycle", 0, 5), 2), "vc2": round(H.helm_bench_graph("vcycle", 2, 20), 2),
                      "vc3": round(H.helm_bench_graph("vcycle", 3, 20), 2)}), flush=True)
    H.close()
