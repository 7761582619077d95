"""In-graph cost of each kernel of the delayed-CGS2 step (HELM_GB_DCGS_MASK: 1 dots, 2 reduceA,
4 update) at several basis sizes, c1_k400 inner level."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2308_06152_b200 import helm  # noqa: E402
    from workloads import config_problem  # noqa: E402
    p = config_problem("c1_k400")
    H = helm.helm_setup(p, {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 50,
                            "coarsest_n": 512})
    out = {"mask": int(sys.argv[1])}
    for j in (5, 25, 45):
        out[f"j{j}"] = round(H.helm_bench_graph("dcgs", j, 3), 2)
    print(json.dumps(out), flush=True)
    sys.exit(0)
for mask in (7, 1, 2, 4, 3, 6):
    env = dict(os.environ, HELM_GB_DCGS_MASK=str(mask))
    subprocess.run([sys.executable, os.path.abspath(__file__), str(mask)], env=env, check=True)
