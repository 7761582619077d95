"""Reproduce PAPER.md Tables 1-2 (MP-2a Dirichlet / MP-2b Sommerfeld, A-DEF1 with the bilinear
deflation vectors, outer Krylov to 1e-6) on the B200 path: outer iteration counts for str-Glk and
ReD-O2, the coarse problem solved by CSLP-FGMRES to a tight tolerance (1e-8; the paper's
parenthesised CGP counts are for its own coarse tolerance).  Also the Appendix B table's
ReD-9ptO2 rows (Dirichlet, APD vectors).  Prints JSON lines and a markdown table with the
paper's counts beside ours."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2308_06152_b200 import helm  # noqa: E402
from workloads import mp_problem  # noqa: E402

# PAPER.md:862-870 (Table 1, CSLP-GMRES columns) and :893-901 (Table 2)
T1 = {(33, 20): (8, 21, 9), (65, 40): (16, 41, 20), (129, 80): (44, 95, 70), (65, 20): (6, 17, 6),
      (129, 40): (9, 20, 9)}
T2 = {(33, 20): (9, 20, 9), (65, 40): (13, 26, 13), (129, 80): (22, 41, 24), (65, 20): (6, 17, 6), (129, 40): (7, 19, 7),
      (257, 80): (10, 20, 8)}
# PAPER.md:1323-1327 (Appendix B): ReD-9ptO2, ReD-O2, ReD-O4
TB = {(129, 40): (15, 17, 14), (257, 80): (20, 28, 19), (321, 100): (27, 37, 22)}


def run(p, vec, op, precond="adef1"):
    H = helm.helm_setup(p, {"vectors": vec, "coarse_op": op, "inner_tol": 1e-8, "inner_maxit": 3000,
                            "precond": precond})
    b = torch.from_numpy(p.b).cuda()
    t0 = time.perf_counter()
    _, rep = H.solve(b, 1e-6, 400)
    dt = time.perf_counter() - t0
    H.close()
    return rep["outer_iterations"], rep["converged"], round(rep["inner_iterations_total"] / max(1, rep["inner_solves"])), dt


lines = []
for bc, table, name in (("dirichlet", T1, "Table 1 (MP-2a)"), ("sommerfeld", T2, "Table 2 (MP-2b)")):
    lines.append(f"\n{name}, A-DEF1, bilinear vectors: outer its (mean coarse its) -- paper / B200\n")
    lines.append("| grid | k | kh | str-Glk paper | str-Glk B200 | ReD-O2 paper | ReD-O2 B200 | TLKM paper | TLKM B200 |")
    lines.append("|---|---|---|---|---|---|---|---|---|")
    for (nodes, k), (pg, pr, pt) in table.items():
        p = mp_problem(float(k), nodes - 1, bc)
        g = run(p, "bilinear", "galerkin")
        r = run(p, "bilinear", "red_o2")
        tl = run(p, "bilinear", "red_o2", "tlkm")
        print(json.dumps({"table": name, "nodes": nodes, "k": k, "galerkin": g, "red_o2": r, "tlkm": tl}), flush=True)
        lines.append(f"| {nodes}² | {k} | {k / (nodes - 1):.4g} | {pg} | {g[0]} ({g[2]}) | {pr} | {r[0]} ({r[2]}) | "
                     f"{pt} | {tl[0]} ({tl[2]}) |")
lines.append("\nAppendix B (MP-2a, APD vectors): outer its -- paper / B200\n")
lines.append("| grid | k | 9ptO2 paper | 9ptO2 B200 | O2 paper | O2 B200 | O4 paper | O4 B200 |")
lines.append("|---|---|---|---|---|---|---|---|")
for (nodes, k), (p9, p2, p4) in TB.items():
    p = mp_problem(float(k), nodes - 1, "dirichlet")
    r9, r2, r4 = (run(p, "high_order", op) for op in ("red_9pto2", "red_o2", "red_o4"))
    print(json.dumps({"table": "appendix B", "nodes": nodes, "k": k, "red_9pto2": r9, "red_o2": r2, "red_o4": r4}),
          flush=True)
    lines.append(f"| {nodes}² | {k} | {p9} | {r9[0]} | {p2} | {r2[0]} | {p4} | {r4[0]} |")
print("\n".join(lines))
