"""A/B of libhelm build variants (tools/build_variants.py) on a workload: in-graph region costs
(inner iteration at several basis columns, V-cycle from level 1, E apply) and, optionally, a
truncated solve (the first `--outer` outer iterations, device time).  Each variant runs in its
own process (HELM_LIB is read at import).

  python tools/ab_libs.py base l2h1 l2h2 --outer 40
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, os, sys, torch
sys.path.insert(0, %r)
from paper_2308_06152_b200 import helm
from workloads import config_problem
a = json.loads(sys.argv[1])
p = config_problem(a["workload"])
prm = dict({"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 200,
            "inner_restart": 50, "coarsest_n": 512}, **a["params"])
H = helm.helm_setup(p, prm)
row = {"lib": a["lib"]}
for j in a["cols"]:
    row[f"it@{j}"] = round(H.helm_bench_graph("inner_iter", j, 4), 2)
row["vc1"] = round(H.helm_bench_graph("vcycle", 1, 20), 2)
row["E"] = round(H.helm_bench_graph("apply_E", 0, 20), 2)
for j in a["cols"]:
    row[f"dcgs@{j}"] = round(H.helm_bench_graph("dcgs", j, 4), 2)
if a["outer"] > 0:
    b = torch.from_numpy(p.b).cuda()
    x = torch.empty_like(b)
    H.solve(b, 1e-6, 2, x)
    ts = []
    for _ in range(a["reps"]):
        H.helm_flush_l2(256 << 20)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); _, rep = H.solve(b, 1e-6, a["outer"], x); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    row["solve_s"] = round(min(ts), 4)
    row["inner_total"] = rep["inner_iterations_total"]
    row["relres"] = rep["relres"]
    row["us_per_inner"] = round(1e6 * min(ts) / max(1, rep["inner_iterations_total"]), 2)
H.close()
print("ABROW " + json.dumps(row), flush=True)
""" % ROOT

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+", help="variant names (base = libhelm.so)")
ap.add_argument("--workload", default="c4_weak_2049")
ap.add_argument("--cols", default="1,24,44")
ap.add_argument("--outer", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--params", default="{}")
ap.add_argument("--out", default="")
a = ap.parse_args()
rows = []
for lib in a.libs:
    env = dict(os.environ)
    path = os.path.join(ROOT, "paper_2308_06152_b200", "libhelm.so" if lib == "base" else f"libhelm_{lib}.so")
    env["HELM_LIB"] = path
    arg = {"lib": lib, "workload": a.workload, "cols": [int(c) for c in a.cols.split(",")], "outer": a.outer,
           "reps": a.reps, "params": json.loads(a.params)}
    r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(arg)], env=env, capture_output=True, text=True)
    line = [l for l in r.stdout.splitlines() if l.startswith("ABROW ")]
    row = json.loads(line[0][6:]) if line else {"lib": lib, "error": r.stderr[-800:]}
    print(json.dumps(row), flush=True)
    rows.append(row)
if a.out:
    with open(a.out, "a") as fh:
        for row in rows:
            fh.write(json.dumps(dict(row, workload=a.workload, params=json.loads(a.params))) + "\n")
