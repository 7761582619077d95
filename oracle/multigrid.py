"""ORACLE (test infrastructure only) — CSLP approximated by one geometric multigrid V-cycle.

PAPER.md §3.1: "The inverse of the preconditioner is approximated by a multigrid V-cycle,
which consists of one step of pre-/post- damped Jacobi smoother with a relaxation
parameter of 0.8, full weighting restriction, bilinear interpolation, and a ... solver
for solving the coarsest-grid problem."
§5.1: coarse-level CSLP operators are re-discretised ("we obtain the coarse-grid operator
M_H in the same way that the matrix M_h is obtained on the fine mesh").
§4: coarsening stops at a predefined coarsest grid.

Readings:
  R7  Coarsening continues while both directions are coarsenable (odd unknown count >= 3),
      `max_levels` is not reached and the current level has more than `coarsest_n` unknowns
      (§4: "after reaching a manually predefined coarsest grid size ... the coarsening
      operation will stop"; 0 = coarsen as far as possible); the coarse wavenumber is sampled
      at coincident nodes.
  R8  The coarsest problem is solved exactly (dense LU, np.linalg.solve).  The paper's
      full-GMRES to 1e-8 on the coarsest level approximates this solve.
  R9  The V-cycle starts from a zero initial guess, so the first pre-smoothing sweep is
      u = omega D^{-1} f.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from .operators import apply_M, stencil_coefficients
from .transfer import coarse_k, coarse_shape, coarsenable, prolong_bilinear, restrict_fw


@dataclasses.dataclass
class Level:
    shape: tuple
    h: float
    k: np.ndarray
    bc: str
    beta: tuple
    dense_inv: np.ndarray | None = None   # coarsest level only

    def M(self, u):
        return apply_M(u, self.k, self.h, self.bc, self.beta)


def jacobi_diagonal(level: Level) -> np.ndarray:
    """D = diag(M_h): the centre multiplier ap of Algorithm 2 for the CSLP stencil."""
    ap, *_ = stencil_coefficients(level.k, level.h, level.bc, level.beta)
    return ap


def _dense_matrix(level: Level) -> np.ndarray:
    n = level.shape[0] * level.shape[1]
    Mmat = np.zeros((n, n), dtype=np.complex128)
    for c in range(n):
        e = np.zeros(n, dtype=np.complex128)
        e[c] = 1.0
        Mmat[:, c] = level.M(e.reshape(level.shape)).ravel()
    return Mmat


def build_hierarchy(k: np.ndarray, h: float, bc: str, beta=(1.0, 0.5), max_levels: int = 64,
                    max_coarsest: int = 4096, coarsest_n: int = 0):
    levels = [Level(k.shape, h, k, bc, tuple(beta))]
    while (len(levels) < max_levels and coarsenable(levels[-1].shape, bc)
           and levels[-1].shape[0] * levels[-1].shape[1] > coarsest_n):
        L = levels[-1]
        levels.append(Level(coarse_shape(L.shape, bc), 2.0 * L.h, coarse_k(L.k, bc), bc, tuple(beta)))
    C = levels[-1]
    n = C.shape[0] * C.shape[1]
    if n > max_coarsest:
        raise ValueError(f"coarsest grid {C.shape} too large for the dense coarsest solve")
    Mmat = _dense_matrix(C)
    C.dense_inv = Mmat  # stored matrix; solved with np.linalg.solve at use (R8)
    return levels


def vcycle(levels, f: np.ndarray, l: int = 0, omega: float = 0.8, nu_pre: int = 1, nu_post: int = 1):
    """One V(nu_pre, nu_post) cycle approximating M_l^{-1} f (§3.1)."""
    L = levels[l]
    if l == len(levels) - 1:
        return np.linalg.solve(L.dense_inv, f.ravel()).reshape(L.shape)
    D = jacobi_diagonal(L)
    u = omega * f / D                                   # R9: first sweep from u = 0
    for _ in range(nu_pre - 1):
        u = u + omega * (f - L.M(u)) / D
    r = f - L.M(u)                                      # residual
    fc = restrict_fw(r, L.bc)                           # full weighting (Eq. 3.8)
    ec = vcycle(levels, fc, l + 1, omega, nu_pre, nu_post)
    u = u + prolong_bilinear(ec, L.shape, L.bc)         # bilinear correction (Eq. 3.9)
    for _ in range(nu_post):
        u = u + omega * (f - L.M(u)) / D                # damped Jacobi post-smoothing
    return u
