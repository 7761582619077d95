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


def test_appendix_b_red9pt_counts_algorithm1():
    """Appendix B, 129^2, k = 40: ReD-9ptO2 15, ReD-O2 17, ReD-O4 14 outer
    iterations.  Reproduced exactly by Algorithm 1 as printed -- LEFT-preconditioned GMRES with
    the preconditioned relative residual (reading R26) -- with the APD vectors and an exact
    coarse solve.  (Right-preconditioned FGMRES with the true residual needs 24 / 25 / 22.)"""
    row = GOLD["appendixB_red9pt"]["rows"][0]
    p = mp_problem(float(row["k"]), row["nodes"] - 1, "dirichlet")
    for op in ("red_9pto2", "red_o2", "red_o4"):
        _, r = oracle.solve(p, oracle.SolverParams(coarse_op=op, vectors="high_order", inner_solver="direct",
                                                   outer="gmres_left", maxit=200))
        assert r["converged"]
        assert r["outer_iterations"] == row[op], (op, r["outer_iterations"], row)


ALG1_ROWS = [  # (table key, row index, bc, vectors, op column, band) -- reading R26
    ("table1_mp2a_dirichlet", 0, "dirichlet", "bilinear", "galerkin", 0),
    ("table1_mp2a_dirichlet", 1, "dirichlet", "bilinear", "galerkin", 0),
    ("table2_mp2b_sommerfeld", 1, "sommerfeld", "bilinear", "galerkin", 1),
    ("table4_mp2b_apd", 0, "sommerfeld", "high_order", "galerkin", 0),
    ("table4_mp2b_apd_red", 1, "sommerfeld", "high_order", "red_o4", 1),
    ("tables12_adef1_red_o2", 1, "dirichlet", "bilinear", "red_o2", 0),
]


@pytest.mark.parametrize("key,idx,bc,vec,op,band", ALG1_ROWS, ids=lambda v: str(v))
def test_algorithm1_left_preconditioned_counts(key, idx, bc, vec, op, band):
    """Tables 1, 2 and 4 with Algorithm 1 as printed (left preconditioning, preconditioned
    residual, MGS, exact coarse solve): the printed outer counts within +-band (0 or 1)."""
    row = GOLD[key]["rows"][idx]
    want = row["outer"] if "outer" in row else row[op]
    p = mp_problem(float(row["k"]), row["nodes"] - 1, bc)
    _, r = oracle.solve(p, oracle.SolverParams(coarse_op=op, vectors=vec, inner_solver="direct",
                                               outer="gmres_left", maxit=300))
    assert r["converged"]
    assert abs(r["outer_iterations"] - want) <= band, (r["outer_iterations"], want)


@pytest.mark.parametrize("row", GOLD["tables12_tlkm_red_o2"]["rows"], ids=lambda r: f"{r['bc']}-{r['nodes']}-{r['k']}")
def test_tlkm_tables12(row):
    """Tables 1-2, TLKM column: the practical TLKM with ReD-O2 (reading R23, exact coarse solve)
    takes the printed outer iteration counts within 3 (the band of the Table 4 pins)."""
    p = mp_problem(float(row["k"]), row["nodes"] - 1, row["bc"])
    _, r = oracle.solve(p, oracle.SolverParams(preconditioner="tlkm", coarse_op="red_o2", inner_solver="direct",
                                               maxit=300))
    assert r["converged"]
    assert abs(r["outer_iterations"] - row["tlkm"]) <= 3, (r["outer_iterations"], row)
