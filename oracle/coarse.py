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
from .transfer import (coarse_k, coarse_shape, prolong_bilinear, prolong_high_order, restrict_fw,
                       restrict_high_order)

COARSE_OPS = ("galerkin", "red_o2", "red_o4", "red_glk1", "red_glk2")

# PAPER.md Eq. 5.12 (Laplacian part, printed) and Eq. 5.14 (wavenumber part, printed).
GLK_LAP = np.array([[-3, -44, -98, -44, -3],
                    [-44, -112, 56, -112, -44],
                    [-98, 56, 980, 56, -98],
                    [-44, -112, 56, -112, -44],
                    [-3, -44, -98, -44, -3]], dtype=np.float64) / 256.0
GLK_MASS = np.array([[1, 28, 70, 28, 1],
                     [28, 784, 1960, 784, 28],
                     [70, 1960, 4900, 1960, 70],
                     [28, 784, 1960, 784, 28],
                     [1, 28, 70, 28, 1]], dtype=np.float64) / 64.0**2


def _red_glk(x, kc, H, bc, variant):
    """ReD-Glk (§5.2.4): re-discretisation with the Galerkin stencils of the higher-order
    vectors, [A_2h] = [-Delta_2h] (Eq. 5.12) - [I(k^2)_2h] (Eq. 5.14) where "for each node
    of the stencil, the wavenumber on the corresponding coarse grid point is used".
    Glk1: second-order stencil (x4, the scale of Z^T A Z) on the two outermost layers.
    Glk2: ghost values fill the taps outside the domain (Eq. 2.8 for Sommerfeld; Eq. 5.18
    u_1 = (u_0 + u_2)/2 for Dirichlet) with ghost wavenumber 0, second-order stencil only on
    the first layer (Dirichlet: the first layer is the boundary node itself, which is not an
    unknown, so every unknown uses the 5x5 stencil).
    Reading R14: the second-order fallback uses 4 A_{2h} so that all rows share the scale
    of Z^T A Z (the 5x5 stencils approximate 4(-Delta - k^2), Eq. 5.13)."""
    ny, nx = x.shape
    y2 = 4.0 * apply_A(x, kc, H, bc)
    # extended arrays with 2 ghost layers
    X = np.zeros((ny + 4, nx + 4), dtype=np.complex128)
    K = np.zeros((ny + 4, nx + 4))
    X[2:-2, 2:-2] = x
    K[2:-2, 2:-2] = kc
    if variant == "red_glk2":
        if bc == "dirichlet":
            # boundary node (value 0) at ext index 1, ghost at ext index 0: u_g = 2*0 - u(first unknown)
            X[2:-2, 0] = -x[:, 0]
            X[2:-2, -1] = -x[:, -1]
            X[0, :] = -X[2, :]
            X[-1, :] = -X[-3, :]
        else:
            # ghost node one layer outside the boundary node: u_g = u_in + 2 i H k_b u_b (Eq. 2.8)
            X[2:-2, 1] = x[:, 1] + 2j * H * kc[:, 0] * x[:, 0]
            X[2:-2, -2] = x[:, -2] + 2j * H * kc[:, -1] * x[:, -1]
            X[1, 1:-1] = X[3, 1:-1] + 2j * H * np.pad(kc[0, :], 1, mode="edge") * X[2, 1:-1]
            X[-2, 1:-1] = X[-4, 1:-1] + 2j * H * np.pad(kc[-1, :], 1, mode="edge") * X[-3, 1:-1]
    y5 = np.zeros((ny, nx), dtype=np.complex128)
    for b in range(-2, 3):
        for a in range(-2, 3):
            xs = X[2 + b:2 + b + ny, 2 + a:2 + a + nx]
            ks = K[2 + b:2 + b + ny, 2 + a:2 + a + nx]
            y5 += (GLK_LAP[b + 2, a + 2] / (H * H)) * xs - GLK_MASS[b + 2, a + 2] * ks * ks * xs
    use5 = np.zeros((ny, nx), dtype=bool)
    if variant == "red_glk1":
        use5[2:ny - 2, 2:nx - 2] = True
    elif bc == "dirichlet":
        use5[:, :] = True
    else:
        use5[1:ny - 1, 1:nx - 1] = True
    return np.where(use5, y5, y2)


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


def apply_coarse_E(x: np.ndarray, k_fine: np.ndarray, h: float, bc: str, op: str = "galerkin",
                   vectors: str = "bilinear") -> np.ndarray:
    """y = E x on the deflation coarse grid (mesh width 2h).
    vectors="bilinear": A-DEF1 (Z = Eq. 3.9, R = Eq. 3.8 = Z^T/4);
    vectors="high_order": APD (Z = Eq. 3.12, R = Eq. 3.14 = Z^T)."""
    fine_shape = k_fine.shape
    if x.shape != coarse_shape(fine_shape, bc):
        raise ValueError("x is not on the coarse grid")
    if vectors == "high_order":
        if op == "galerkin":
            return restrict_high_order(apply_A(prolong_high_order(x, fine_shape, bc), k_fine, h, bc), bc)
        if op in ("red_glk1", "red_glk2"):
            return _red_glk(x, coarse_k(k_fine, bc), 2.0 * h, bc, op)
        raise ValueError(f"coarse op {op} not defined for the higher-order vectors")
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
