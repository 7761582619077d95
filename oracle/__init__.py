"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation (numpy, complex128 / float64) of the
data-parallel hot path of arXiv:2308.06152 ("Matrix-free parallel preconditioned
iterative solvers for the 2D Helmholtz equation discretized with finite differences",
two-level deflation + CSLP).  Every function cites the PAPER.md passage it follows.

Rules:
  * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
    leg may import anything under oracle/.  The product path (paper_2308_06152_b200/)
    never imports it and has no CPU fallback.
  * The oracle shares no code with the CUDA path; both consume the seeded inputs from
    workloads/ (which holds none of the method's arithmetic).
  * Numpy slicing / library primitives (np.linalg.solve, vdot, norm) serve as steps; no
    blocking, fusion or reordering beyond the paper's definitions.

Pins (tests/test_oracle_*.py, -m "not gpu"): discrete Dirichlet eigenfunctions with the
closed-form eigenvalues of Appendix B; textbook Kronecker-sum assembly of A (both BCs) and
of the bilinear prolongation; ghost-point form of the Sommerfeld rows (Eq. 2.8);
full weighting = Z^T/4 and the deflation restriction = Z^T exactly; tensor-product closed form of
the Galerkin coarse operator Z^T A Z; dense
two-grid operator vs the V-cycle; deflation identities P A Z = 0 and Q A Z = Z; dense
solves on tiny grids; printed iteration counts of Tables 1 and 2 (tests/golden/).

Parity pinned for every function listed in DESIGN.md §4; "parity unpinned": none.
"""
from .operators import (  # noqa: F401
    unknown_offset,
    stencil_coefficients,
    apply_operator,
    apply_A,
    apply_M,
)
from .transfer import (coarsenable, coarse_shape, coarse_k, restrict_fw, restrict_bilinear_zt, prolong_bilinear,  # noqa: F401
                       restrict_high_order, prolong_high_order)
from .coarse import apply_coarse_E  # noqa: F401
from .multigrid import Level, build_hierarchy, vcycle, jacobi_diagonal  # noqa: F401
from .krylov import fgmres, gcr, gmres_left  # noqa: F401
from .solver import SolverParams, Solver, solve  # noqa: F401
