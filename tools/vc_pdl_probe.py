"""V-cycle from each level of the c4_weak_2049 hierarchy, in graph, with and without PDL
(params.pdl), plus the level-1 legs: the effect of loading set-up / earlier-launch inputs before
the PDL wait (k_vc_up, k_gemv)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402
p = config_problem(sys.argv[1] if len(sys.argv) > 1 else "c4_weak_2049")
for pdl in ((1, 0) if len(sys.argv) > 2 else (1,)):
    prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 48, "coarsest_n": 512,
           "pdl": pdl}
    H = helm.helm_setup(p, prm)
    out = {"pdl": pdl}
    for l in range(1, len(H.levels)):
        out[f"vc{l}"] = round(H.helm_bench_graph("vcycle", l, 20), 2)
    for l in (1, 2):
        out[f"down{l}"] = round(H.helm_bench_graph("vc_down", l, 20), 2)
        out[f"up{l}"] = round(H.helm_bench_graph("vc_up", l, 20), 2)
    print(json.dumps(out), flush=True)
    H.close()
