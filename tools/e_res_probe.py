"""In-graph cost of the E apply in residual mode (the s-step powers' k_glk_stream<2,1>) and in
plain mode at a workload's coarse level, with the bench method (helm_bench_graph regions)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402
import bench  # noqa: E402
p = config_problem(sys.argv[1] if len(sys.argv) > 1 else "c4_weak_2049")
prm = dict(bench.DEFAULT_METHOD, **bench.DEFAULT_SSTEP)
H = helm.helm_setup(p, prm)
n1 = H.levels[1][0] * H.levels[1][1]
for region, nb in (("ss_e", 80.0), ("apply_E", 64.0)):
    us = H.helm_bench_graph(region, 0, 20)
    print(json.dumps({"workload": p.name if hasattr(p, "name") else sys.argv[1:], "region": region, "us": round(us, 2),
                      "GBps": round(nb * n1 / us / 1e3, 1)}), flush=True)
H.close()
