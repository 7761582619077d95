import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402
p = config_problem("c4_weak_2049")
H = helm.helm_setup(p, {"vectors": "high_order", "coarse_op": "galerkin", "inner_maxit": 200, "inner_restart": 50, "coarsest_n": 512})
row = {"rev": os.environ.get("HELM_UPD_REV")}
for j in (12, 24, 44):
    for r in ("dcgs_update", "dcgs", "inner_iter"):
        row[f"{r}@{j}"] = round(H.helm_bench_graph(r, j, 4), 2)
print(json.dumps(row))
