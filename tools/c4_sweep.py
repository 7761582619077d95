"""Method sweep on a BASELINE configs[4] problem on one GPU: time-to-1e-6 for several solver
settings (outer FGMRES / GCR, coarse-solve cap, restart, tolerance, vectors, coarse operator).
Each setting is one JSON object on the command line (or a file of them, one per line); one
result line per setting is appended to --out.

  python tools/c4_sweep.py --problem c4_weak_2049 '{"inner_maxit": 100}' '{"inner_restart": 30, ...}'
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import config_problem  # noqa: E402

BASE = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 0.1, "inner_maxit": 100, "coarsest_n": 512}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problem", default="c4_weak_2049")
    ap.add_argument("--out", default="gpurun_out/c4_sweep.jsonl")
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--warm", type=int, default=0, help="untimed solves before the timed one (graph capture)")
    ap.add_argument("settings", nargs="+")
    a = ap.parse_args()
    settings = []
    for s in a.settings:
        if os.path.exists(s):
            settings += [json.loads(l) for l in open(s) if l.strip()]
        else:
            settings.append(json.loads(s))
    t0 = time.perf_counter()
    p = config_problem(a.problem)
    gen = time.perf_counter() - t0
    b = torch.from_numpy(p.b).cuda()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    for st in settings:
        st = dict(st)
        maxit = st.pop("maxit", 1000)
        prm = dict(BASE, **st)
        H = helm.helm_setup(p, prm)
        for _ in range(a.warm):
            H.solve(b, a.tol, maxit)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        x, rep = H.solve(b, a.tol, maxit)
        dt = time.perf_counter() - t1
        r = H.apply_A(x)
        rr = float(torch.linalg.vector_norm(r - b) / torch.linalg.vector_norm(b))
        line = {"problem": a.problem, "nx": p.nx, "ny": p.ny, "params": prm, "maxit": maxit,
                "outer": rep["outer_iterations"], "converged": rep["converged"], "true_relres": rr,
                "seconds": round(dt, 3), "inner_total": rep["inner_iterations_total"],
                "inner_max": rep["inner_iterations_max"], "inner_restarts": rep["inner_restarts"],
                "restarts": rep["restarts"], "input_gen_s": round(gen, 1)}
        print(json.dumps(line), flush=True)
        with open(a.out, "a") as fh:
            fh.write(json.dumps(line) + "\n")
        H.close()
        del x, r
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
