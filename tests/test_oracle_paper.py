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
