"""PAPER.md Tables 9-10 (weak scaling, non-constant wavenumber, DelftBlue MPI: np processes)
re-run as single solves on one B200 -- context, not a target: APD + str-Glk, outer GMRES
(here FGMRES) with the coarse solver at 1e-6, or GCR with the coarse solver at 1e-1 (PAPER.md
§6.3).  The wedge is our reconstruction (R18), the Marmousi model the seeded synthetic."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import marmousi_like_problem, wedge_problem  # noqa: E402

# (label, builder, np, paper GMRES (its, coarse its, s), paper GCR (its, coarse its, s)) -- PAPER.md:1115-1140
CASES = [
    ("Wedge f=40 577x961", lambda: wedge_problem(40.0, (577, 961)), 6, (9, 251, 53.41), (10, 46, 4.86)),
    ("Wedge f=40 1153x1921", lambda: wedge_problem(40.0, (1153, 1921)), 24, (10, 259, 68.59), (10, 43, 5.75)),
    ("Marmousi f=10 737x241", lambda: marmousi_like_problem(10.0, (737, 241)), 3, (10, 414, 103.92), (11, 63, 10.55)),
    ("Marmousi f=10 1473x481", lambda: marmousi_like_problem(10.0, (1473, 481)), 12, (9, 378, 111.20), (10, 58, 12.08)),
    ("Marmousi f=10 2945x961", lambda: marmousi_like_problem(10.0, (2945, 961)), 48, (9, 383, 156.45), (10, 58, 17.72)),
]


def timed(p, prm):
    H = helm.helm_setup(p, prm)
    b = torch.from_numpy(p.b).cuda()
    H.solve(b, 1e-6, 500)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, rep = H.solve(b, 1e-6, 500)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    H.close()
    return dt, rep


lines = ["| case | np (paper) | GMRES its (coarse) paper | s paper | FGMRES its (coarse) B200 | s B200 | GCR its (coarse) paper | s paper | GCR its (coarse) B200 | s B200 |",
         "|---|---|---|---|---|---|---|---|---|---|"]
for label, build, np_, pg, pc in CASES:
    p = build()
    out = {}
    for outer, itol in (("fgmres", 1e-6), ("gcr", 1e-1)):
        dt, rep = timed(p, {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": itol, "inner_maxit": 4000,
                            "outer": outer})
        out[outer] = (rep["outer_iterations"], round(rep["inner_iterations_total"] / max(1, rep["inner_solves"])),
                      round(dt, 3), rep["converged"])
    print(json.dumps({"case": label, "np": np_, "paper_gmres": pg, "paper_gcr": pc, "b200": out}), flush=True)
    g, c = out["fgmres"], out["gcr"]
    lines.append(f"| {label} | {np_} | {pg[0]} ({pg[1]}) | {pg[2]} | {g[0]} ({g[1]}) | {g[2]} | {pc[0]} ({pc[1]}) | "
                 f"{pc[2]} | {c[0]} ({c[1]}) | {c[2]} |")
print("\n".join(lines))
