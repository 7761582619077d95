"""Golden pins from the paper's printed iteration counts (tests/golden/)."""
import json
import os

import pytest

import oracle
from workloads import mp_problem

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_iteration_counts.json")))


def _cases():
    for key, bc in (("table1_mp2a_dirichlet", "dirichlet"), ("table2_mp2b_sommerfeld", "sommerfeld")):
        for row in GOLD[key]["rows"]:
            yield pytest.param(bc, row, id=f"{bc}-{row['nodes']}")


@pytest.mark.parametrize("bc,row", list(_cases()))
def test_outer_iterations_match_paper(bc, row):
    """A-DEF1 + str-Glk with an exact coarse solve (the paper solves it to 1e-12).
    Our outer method is FGMRES with the true residual (the paper: left-preconditioned GMRES
    with the preconditioned residual), so we allow max(2, 15%) iterations of difference."""
    p = mp_problem(float(row["k"]), row["nodes"] - 1, bc)
    x, rep = oracle.solve(p, oracle.SolverParams(coarse_op="galerkin", inner_solver="direct"))
    assert rep["converged"] and rep["relres"] <= 1e-6
    tol = max(2, int(0.15 * row["outer"] + 0.999))
    assert abs(rep["outer_iterations"] - row["outer"]) <= tol, (rep["outer_iterations"], row)


@pytest.mark.parametrize("row", GOLD["tables12_adef1_red_o2"]["rows"], ids=lambda r: f"{r['bc']}-{r['nodes']}")
def test_red_o2_costs_about_2_5x_str_glk(row):
    """Tables 1-2: with bilinear vectors the re-discretised ReD-O2 coarse operator needs ~2.5x
    the str-Glk outer iterations (paper: 21/8, 41/16, 20/9, 26/13).  The oracle must show
    ReD-O2 >= 2x str-Glk and stay within 30% of the printed ReD-O2 count (reading R10)."""
    p = mp_problem(float(row["k"]), row["nodes"] - 1, row["bc"])
    _, rg = oracle.solve(p, oracle.SolverParams(coarse_op="galerkin", inner_solver="direct", maxit=300))
    _, rr = oracle.solve(p, oracle.SolverParams(coarse_op="red_o2", inner_solver="direct", maxit=300))
    assert rr["outer_iterations"] >= 2 * rg["outer_iterations"], (rr["outer_iterations"], rg["outer_iterations"])
    assert abs(rr["outer_iterations"] - row["red_o2"]) <= 0.3 * row["red_o2"] + 1, (rr["outer_iterations"], row)


def test_appendix_b_red9pt_between_o4_and_o2():
    """Appendix B: ReD-9ptO2 needs no more iterations than ReD-O2 and no fewer than ReD-O4
    (129^2, k = 40: 15 between 14 and 17).  The oracle (APD vectors, exact coarse solve)
    reproduces the ordering; its absolute counts are ~1.5x the printed ones at this kh
    (22 / 24 / 25, reading R22), so only the ordering is pinned."""
    row = GOLD["appendixB_red9pt"]["rows"][0]
    p = mp_problem(float(row["k"]), row["nodes"] - 1, "dirichlet")
    its = {}
    for op in ("red_o4", "red_9pto2", "red_o2"):
        _, r = oracle.solve(p, oracle.SolverParams(coarse_op=op, vectors="high_order", inner_solver="direct",
                                                   maxit=200))
        assert r["converged"]
        its[op] = r["outer_iterations"]
    assert its["red_o4"] <= its["red_9pto2"] <= its["red_o2"], its


@pytest.mark.parametrize("row", GOLD["tables12_tlkm_red_o2"]["rows"], ids=lambda r: f"{r['bc']}-{r['nodes']}-{r['k']}")
def test_tlkm_tables12(row):
    """Tables 1-2, TLKM column: the practical TLKM with ReD-O2 (reading R23, exact coarse solve)
    takes the printed outer iteration counts within 3 (the band of the Table 4 pins)."""
    p = mp_problem(float(row["k"]), row["nodes"] - 1, row["bc"])
    _, r = oracle.solve(p, oracle.SolverParams(preconditioner="tlkm", coarse_op="red_o2", inner_solver="direct",
                                               maxit=300))
    assert r["converged"]
    assert abs(r["outer_iterations"] - row["tlkm"]) <= 3, (r["outer_iterations"], row)
