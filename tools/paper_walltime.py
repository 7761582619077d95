"""The paper's wall-clock experiments (DelftBlue, Fortran + MPI) next to the same runs on one
B200, as context (not a target): PAPER.md:1069 (MP-2b, k = 320, 513^2, APD + ReD-Glk2: GMRES with
the coarse solver at 1e-6 -> 145.41 s; GCR with the coarse solver at 1e-1 -> 9.48 s) and
PAPER.md:1004-1013 (Marmousi, 12 processes, APD-GMRES, CSLP-GMRES coarse solve: 737x241 f = 10
str-Glk 120.67 s / ReD-Glk2 164.79 s; 1473x481 f = 20: 1039.96 s / 1376.40 s).  Our Marmousi is the
seeded synthetic of the same shape (R18), so those rows compare like-sized problems, not
the same velocity model.  Times on B200: one solve after a warm-up (graph capture) solve."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import marmousi_like_problem, mp_problem  # noqa: E402


def timed(p, prm, maxit=2000):
    H = helm.helm_setup(p, prm)
    b = torch.from_numpy(p.b).cuda()
    H.solve(b, 1e-6, maxit)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, rep = H.solve(b, 1e-6, maxit)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    H.close()
    return dt, rep


rows = []
p = mp_problem(320.0, 512, "sommerfeld")
for outer, itol, paper in (("fgmres", 1e-6, 145.41), ("gcr", 1e-1, 9.48)):
    dt, rep = timed(p, {"vectors": "high_order", "coarse_op": "red_glk2", "inner_tol": itol, "inner_maxit": 4000,
                        "outer": outer})
    r = {"case": f"MP-2b k=320 513^2 APD+ReD-Glk2 {outer} coarse tol {itol:g}", "paper_s": paper,
         "b200_s": round(dt, 3), "outer": rep["outer_iterations"], "inner_mean": round(rep["inner_iterations_total"] /
                                                                                       max(1, rep["inner_solves"]), 1),
         "converged": rep["converged"]}
    print(json.dumps(r), flush=True)
    rows.append(r)
for (nx, ny), f, papers in (((737, 241), 10.0, {"galerkin": 120.67, "red_glk2": 164.79}),
                            ((1473, 481), 20.0, {"galerkin": 1039.96, "red_glk2": 1376.40})):
    p = marmousi_like_problem(f, (nx, ny))
    for op, paper in papers.items():
        dt, rep = timed(p, {"vectors": "high_order", "coarse_op": op, "inner_tol": 1e-6, "inner_maxit": 4000})
        r = {"case": f"Marmousi-shaped {nx}x{ny} f={f:g} APD+{op} FGMRES coarse tol 1e-6", "paper_s (12 procs)": paper,
             "b200_s": round(dt, 3), "outer": rep["outer_iterations"],
             "inner_mean": round(rep["inner_iterations_total"] / max(1, rep["inner_solves"]), 1),
             "converged": rep["converged"]}
        print(json.dumps(r), flush=True)
        rows.append(r)
