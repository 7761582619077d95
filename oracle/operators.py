"""ORACLE (test infrastructure only) — matrix-free Helmholtz and CSLP operators.

PAPER.md §2.1 Eq. 2.5-2.7 (5-point stencil of A_h = -Delta_h - I(k^2)),
Eq. 2.8-2.10 (first-order Sommerfeld ghost-point elimination),
Eq. 3.1 (CSLP M = -Delta_h - (beta1 + i beta2) I(k^2)),
§5.1 Algorithm 2 (matrix-free mat-vec with multipliers ap, aw, ae, as, an).

Readings:
  R1  Dirichlet unknowns are the interior nodes; a neighbour on the boundary carries the
      homogeneous Dirichlet datum g = 0, so its multiplier is set to zero (Alg. 2: "set
      the multiplier corresponding to meaningless grid points to zero").
  R2  CSLP shift sign: Eq. 3.1 literally, M = -Delta_h - (beta1 + i beta2) k^2 with the
      configured (beta1, beta2) = (1, 0.5).  This equals §5.1's
      ap = (4 - (beta1 - beta2 i) k^2 h^2)/h^2 with the paper's beta2 = -0.5.
  R3  The Sommerfeld boundary term of M is the same -2 i k h (real k) as in A: the shift
      multiplies only the mass term I(k^2) of Eq. 3.1.
"""
from __future__ import annotations

import numpy as np


def unknown_offset(bc: str) -> int:
    """Node index of unknown 0 (Dirichlet: first interior node; Sommerfeld: boundary node)."""
    if bc == "dirichlet":
        return 1
    if bc == "sommerfeld":
        return 0
    raise ValueError(bc)


def stencil_coefficients(k: np.ndarray, h: float, bc: str, shift=(1.0, 0.0)):
    """Multipliers (ap, aw, ae, as, an) of Algorithm 2 for every unknown.

    Interior (§5.1): ap = (4 - s k^2 h^2)/h^2, aw = ae = as = an = -1/h^2, s = beta1 + i beta2
    (s = 1 gives A_h, Eq. 2.7).
    Sommerfeld edge (Eq. 2.9): the outward multiplier vanishes, the inward one doubles
    (-2/h^2) and ap gains -2 i k h / h^2; corners (Eq. 2.10) get both directions (-4 i k h).
    """
    ny, nx = k.shape
    s = complex(shift[0], shift[1])
    ih2 = 1.0 / (h * h)
    ap = (4.0 - s * k * k * h * h) * ih2 + 0j
    aw = np.full((ny, nx), -ih2, dtype=np.complex128)
    ae = aw.copy()
    as_ = aw.copy()
    an = aw.copy()
    if bc == "dirichlet":
        aw[:, 0] = 0.0
        ae[:, -1] = 0.0
        as_[0, :] = 0.0
        an[-1, :] = 0.0
    elif bc == "sommerfeld":
        if nx < 2 or ny < 2:
            raise ValueError("Sommerfeld grid needs at least 2 nodes per direction")
        # left edge  (ghost u_{-1,j} = u_{1,j} + 2 h i k u_{0,j}, Eq. 2.8)
        aw[:, 0] = 0.0
        ae[:, 0] = -2.0 * ih2
        ap[:, 0] -= 2j * k[:, 0] * h * ih2
        # right edge
        ae[:, -1] = 0.0
        aw[:, -1] = -2.0 * ih2
        ap[:, -1] -= 2j * k[:, -1] * h * ih2
        # bottom edge (j = 0)
        as_[0, :] = 0.0
        an[0, :] = -2.0 * ih2
        ap[0, :] -= 2j * k[0, :] * h * ih2
        # top edge (j = ny-1)
        an[-1, :] = 0.0
        as_[-1, :] = -2.0 * ih2
        ap[-1, :] -= 2j * k[-1, :] * h * ih2
    else:
        raise ValueError(bc)
    return ap, aw, ae, as_, an


def apply_operator(u: np.ndarray, k: np.ndarray, h: float, bc: str, shift=(1.0, 0.0)) -> np.ndarray:
    """Algorithm 2: v(i,j) = ap u(i,j) + ae u(i+1,j) + aw u(i-1,j) + an u(i,j+1) + as u(i,j-1)."""
    ap, aw, ae, as_, an = stencil_coefficients(k, h, bc, shift)
    u = np.asarray(u, dtype=np.complex128)
    v = ap * u
    v[:, 1:] += aw[:, 1:] * u[:, :-1]
    v[:, :-1] += ae[:, :-1] * u[:, 1:]
    v[1:, :] += as_[1:, :] * u[:-1, :]
    v[:-1, :] += an[:-1, :] * u[1:, :]
    return v


def apply_A(u, k, h, bc):
    """Helmholtz operator A_h (Eq. 2.7 / 2.9 / 2.10)."""
    return apply_operator(u, k, h, bc, (1.0, 0.0))


def apply_M(u, k, h, bc, beta=(1.0, 0.5)):
    """CSLP operator M_{h,(beta1,beta2)} (Eq. 3.1, readings R2/R3)."""
    return apply_operator(u, k, h, bc, beta)
