"""ORACLE (test infrastructure only) — deflation coarse-grid operators E = A_{2h}.

PAPER.md §3.2 "P_h = I_h - A_h Q_h, Q_h = I_{2h}^h A_{2h}^{-1} I_h^{2h},
A_{2h} = I_h^{2h} A_h I_{2h}^h" and §5.2 (matrix-free coarse operators):

  "galerkin"  str-Glk, Eq. 5.7 a-c: interpolation, fine-grid operator, restriction —
              the definition E x = R (A (P x)) applied step by step.
  "red_o2"    ReD-O2, §5.2.3: the 5-point Helmholtz stencil (Eq. 2.7/2.9/2.10) at mesh
              width 2h with the coarse wavenumber.
  "red_o4"    ReD-O4, §5.2.3 Eq. 5.11 (fourth-order Laplacian, 9 taps on a 5-wide cross)
              with second-order stencils where the cross does not fit (§5.2.3 "the
              stencils for the boundary grid points will be changed to that of the
              second-order re-discretization method").

Reading R5: Eq. 5.11 prints the centre as "60 - k^2 (2h)^2" inside the
prefactor 1/(12 (2h)^2); a consistent discretisation of -Delta - k^2 needs
60 - 12 k^2 (2h)^2, i.e. centre 5/H^2 - k^2.  We use the consistent form.
Reading R6: the cross "fits" at a coarse unknown when all four distance-2 neighbours are
nodes of the closed domain (Dirichlet boundary nodes count, holding 0); otherwise the
whole stencil at that point is the second-order one.
"""
from __future__ import annotations

import numpy as np

from .operators import apply_A
from .transfer import coarse_k, coarse_shape, prolong_bilinear, restrict_fw

COARSE_OPS = ("galerkin", "red_o2", "red_o4")


def _red_o4(x, kc, H, bc):
    ny, nx = x.shape
    y2 = apply_A(x, kc, H, bc)
    xp = np.zeros((ny + 4, nx + 4), dtype=np.complex128)
    xp[2:-2, 2:-2] = x
    c = xp[2:-2, 2:-2]
    d1 = xp[2:-2, 1:-3] + xp[2:-2, 3:-1] + xp[1:-3, 2:-2] + xp[3:-1, 2:-2]
    d2 = xp[2:-2, 0:-4] + xp[2:-2, 4:] + xp[0:-4, 2:-2] + xp[4:, 2:-2]
    y4 = (60.0 * c - 16.0 * d1 + d2) / (12.0 * H * H) - kc * kc * c
    fits = np.zeros((ny, nx), dtype=bool)
    if bc == "dirichlet":
        fits[1:ny - 1, 1:nx - 1] = True
    else:
        fits[2:ny - 2, 2:nx - 2] = True
    return np.where(fits, y4, y2)


def apply_coarse_E(x: np.ndarray, k_fine: np.ndarray, h: float, bc: str, op: str = "galerkin") -> np.ndarray:
    """y = E x on the deflation coarse grid (mesh width 2h)."""
    fine_shape = k_fine.shape
    if x.shape != coarse_shape(fine_shape, bc):
        raise ValueError("x is not on the coarse grid")
    if op == "galerkin":
        v1 = prolong_bilinear(x, fine_shape, bc)      # Eq. 5.7a
        v2 = apply_A(v1, k_fine, h, bc)               # Eq. 5.7b
        return restrict_fw(v2, bc)                    # Eq. 5.7c
    kc = coarse_k(k_fine, bc)
    if op == "red_o2":
        return apply_A(x, kc, 2.0 * h, bc)
    if op == "red_o4":
        return _red_o4(x, kc, 2.0 * h, bc)
    raise ValueError(op)
