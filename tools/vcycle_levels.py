"""In-graph V-cycle cost from each level of the c1_k400 bench hierarchy (warm, back-to-back)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

p = config_problem("c1_k400")
for extra in ({}, {"coarsest_n": 128}, {"coarsest_n": 128, "tail_max_n": 2048, "tail_cluster": 1},
              {"coarsest_n": 128, "tail_max_n": 512, "tail_cluster": 1}, {"coarsest_n": 128, "tail_max_n": 8192, "tail_cluster": 1},
              {"coarsest_n": 128, "tail_max_n": 2048, "tail_cluster": 4}, {"coarsest_n": 32, "tail_max_n": 2048, "tail_cluster": 1}):
    prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 50, "coarsest_n": 512}
    prm.update(extra)
    H = helm.helm_setup(p, prm)
    out = {"cfg": extra, "levels": [lv[:2] for lv in H.levels]}
    for l in range(1, len(H.levels)):
        out[f"vc{l}"] = round(H.helm_bench_graph("vcycle", l, 20), 2)
    print(json.dumps(out), flush=True)
    H.close()
