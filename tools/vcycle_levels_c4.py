import json, os, sys
sys.path.insert(0, '/root/repo')
from paper_2308_06152_b200 import helm
from workloads import config_problem
p = config_problem("c4_weak_2049")
for extra in ({}, {"tail_max_n": 4096, "tail_cluster": 16}, {"tail_max_n": 1024, "tail_cluster": 8}):
    prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 48, "coarsest_n": 512}
    prm.update(extra)
    H = helm.helm_setup(p, prm)
    out = {"cfg": extra, "levels": [lv[:2] for lv in H.levels]}
    for l in range(1, len(H.levels)):
        out[f"vc{l}"] = round(H.helm_bench_graph("vcycle", l, 20), 2)
    for l in range(1, len(H.levels) - 1):
        try:
            out[f"down{l}"] = round(H.helm_bench_graph("vc_down", l, 20), 2)
            out[f"up{l}"] = round(H.helm_bench_graph("vc_up", l, 20), 2)
        except Exception as e:
            pass
    print(json.dumps(out), flush=True)
    H.close()
