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
  "red_o6"    ReD-O6, §5.2.3 Eq. 5.10 (sixth-order Laplacian, 13 taps on a 7-wide cross),
              same boundary rule (reading R6).
  "red_cmpo4" ReD-cmpO4, §5.2.5 Eq. 5.19 with the Singer-Turkel coefficients (gamma = 1):
              a 9-point compact stencil; Sommerfeld ghosts by the fourth-order condition
              u_0 = 2ikh(1 - k^2h^2/6) u_1 + u_2 and the corner ghost u_00 = (u_10 + u_01)/2.
  "red_9pto2" ReD-9ptO2, Appendix B: the same general 3x3 form (Eq. 5.19)
              with the eigenvalue-aligned coefficients a = (4.632, -1.316, 0.158), b = (1, 0, 0);
              Sommerfeld ghosts by the second-order condition u_0 = 2ikh u_1 + u_2 (reading R22).

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
from .transfer import (coarse_k, coarse_shape, prolong_bilinear, prolong_high_order, restrict_bilinear_zt,
                       restrict_high_order)

COARSE_OPS = ("galerkin", "red_o2", "red_o4", "red_o6", "red_cmpo4", "red_9pto2", "red_glk1", "red_glk2")
RED_OPS = ("red_o2", "red_o4", "red_o6", "red_cmpo4", "red_9pto2")   # re-discretisations of A at mesh 2h

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
    Reading R14: the boundary layers use "the standard second-order discretization"
     literally, i.e. A_{2h} of Eq. 2.7/2.9/2.10 at mesh 2h, although the 5x5
    interior stencils carry the factor 4 of Z^T A Z (Eq. 5.13); the paper attributes the extra
    ReD-Glk1 iterations to this "simplified boundary treatment"."""
    ny, nx = x.shape
    y2 = apply_A(x, kc, H, bc)
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


def _red_o6(x, kc, H, bc):
    """ReD-O6: -(2u_{i-3} - 27u_{i-2} + 270u_{i-1} - 490u_i + 270u_{i+1} - 27u_{i+2} + 2u_{i+3})/(180H^2)
    per direction (Eq. 5.10) minus k^2 at the centre; second-order stencil where the
    7-wide cross does not fit in the closed domain (reading R6)."""
    ny, nx = x.shape
    y2 = apply_A(x, kc, H, bc)
    xp = np.zeros((ny + 6, nx + 6), dtype=np.complex128)
    xp[3:-3, 3:-3] = x
    c = xp[3:-3, 3:-3]

    def ring(d):
        return (xp[3:-3, 3 - d:xp.shape[1] - 3 - d] + xp[3:-3, 3 + d:xp.shape[1] - 3 + d] +
                xp[3 - d:xp.shape[0] - 3 - d, 3:-3] + xp[3 + d:xp.shape[0] - 3 + d, 3:-3])
    y6 = (980.0 * c - 270.0 * ring(1) + 27.0 * ring(2) - 2.0 * ring(3)) / (180.0 * H * H) - kc * kc * c
    fits = np.zeros((ny, nx), dtype=bool)
    if bc == "dirichlet":
        fits[2:ny - 2, 2:nx - 2] = True
    else:
        fits[3:ny - 3, 3:nx - 3] = True
    return np.where(fits, y6, y2)


# PAPER.md Eq. 5.19 with the Singer-Turkel coefficients (gamma = 1)
CMP_GAMMA = 1.0
CMP_A = {"0": 10.0 / 3.0, "s": -2.0 / 3.0, "c": -1.0 / 6.0}
CMP_B = {"0": 2.0 / 3.0 + CMP_GAMMA / 36.0, "s": 1.0 / 12.0 - CMP_GAMMA / 72.0, "c": CMP_GAMMA / 144.0}


# PAPER.md Appendix B, Eq. optstcl_k80 (:1300-1304): a_0 = 4.632, a_s = -1.316, a_c = 0.158 with
# b_s = b_c = 0, b_0 = 1 (constraints Eq. CommonConstraints_A/B, :1273-1277)
OPT9_A = {"0": 4.632, "s": -1.316, "c": 0.158}
OPT9_B = {"0": 1.0, "s": 0.0, "c": 0.0}


def _red_cmpo4(x, kc, H, bc):
    """ReD-cmpO4 (Eq. 5.19, Singer-Turkel coefficients, fourth-order ghosts)."""
    return _red_9point(x, kc, H, bc, CMP_A, CMP_B, fourth_order_ghost=True)


def _red_9pto2(x, kc, H, bc):
    """ReD-9ptO2 (Appendix B): the general form with the eigenvalue-aligned
    coefficients; second-order Sommerfeld ghosts (reading R22)."""
    return _red_9point(x, kc, H, bc, OPT9_A, OPT9_B, fourth_order_ghost=False)


def _red_9point(x, kc, H, bc, A, B, fourth_order_ghost):
    """General 3x3 form (Eq. 5.19): y = (1/H^2) sum a_tap u_tap - k_c^2 sum b_tap u_tap
    (a_0, a_s, a_c / b_0, b_s, b_c), k_c the wavenumber of the centre node (reading R19: the form
    carries one k^2 per stencil).  Dirichlet: taps on the boundary hold 0.  Sommerfeld: ghost
    nodes one layer outside the domain, u_ghost = u_inner + 2 i k H (1 - k^2 H^2 / 6) u_boundary
    (fourth-order condition) or u_inner + 2 i k H u_boundary (second order), k
    of the boundary node; the corner ghost is the mean of its two edge-ghost neighbours."""
    ny, nx = x.shape
    X = np.zeros((ny + 2, nx + 2), dtype=np.complex128)
    X[1:-1, 1:-1] = x
    if bc == "sommerfeld":
        if fourth_order_ghost:
            fac = lambda kk: 2j * kk * H * (1.0 - kk * kk * H * H / 6.0)
        else:
            fac = lambda kk: 2j * kk * H
        X[1:-1, 0] = x[:, 1] + fac(kc[:, 0]) * x[:, 0]
        X[1:-1, -1] = x[:, -2] + fac(kc[:, -1]) * x[:, -1]
        X[0, 1:-1] = x[1, :] + fac(kc[0, :]) * x[0, :]
        X[-1, 1:-1] = x[-2, :] + fac(kc[-1, :]) * x[-1, :]
        X[0, 0] = 0.5 * (X[0, 1] + X[1, 0])
        X[0, -1] = 0.5 * (X[0, -2] + X[1, -1])
        X[-1, 0] = 0.5 * (X[-1, 1] + X[-2, 0])
        X[-1, -1] = 0.5 * (X[-1, -2] + X[-2, -1])
    c = X[1:-1, 1:-1]
    side = X[1:-1, :-2] + X[1:-1, 2:] + X[:-2, 1:-1] + X[2:, 1:-1]
    corner = X[:-2, :-2] + X[:-2, 2:] + X[2:, :-2] + X[2:, 2:]
    lap = (A["0"] * c + A["s"] * side + A["c"] * corner) / (H * H)
    mass = B["0"] * c + B["s"] * side + B["c"] * corner
    return lap - kc * kc * mass


def apply_coarse_E(x: np.ndarray, k_fine: np.ndarray, h: float, bc: str, op: str = "galerkin",
                   vectors: str = "bilinear") -> np.ndarray:
    """y = E x on the deflation coarse grid (mesh width 2h).
    vectors="bilinear": A-DEF1 (Z = Eq. 3.9, restriction Z^T = Eq. 3.7 per direction, R10);
    vectors="high_order": APD (Z = Eq. 3.12, R = Eq. 3.14 = Z^T).
    The re-discretised operators (RED_OPS) are the same for both vector kinds: they replace
    A_{2h} as printed, without the factor 4 that Z^T A Z carries for the higher-order vectors
    (reading R21; "P_h is no longer a projection")."""
    fine_shape = k_fine.shape
    if x.shape != coarse_shape(fine_shape, bc):
        raise ValueError("x is not on the coarse grid")
    if op in RED_OPS:
        kc = coarse_k(k_fine, bc)
        H = 2.0 * h
        if op == "red_o2":
            return apply_A(x, kc, H, bc)
        if op == "red_o4":
            return _red_o4(x, kc, H, bc)
        if op == "red_o6":
            return _red_o6(x, kc, H, bc)
        if op == "red_9pto2":
            return _red_9pto2(x, kc, H, bc)
        return _red_cmpo4(x, kc, H, bc)
    if vectors == "high_order":
        if op == "galerkin":
            return restrict_high_order(apply_A(prolong_high_order(x, fine_shape, bc), k_fine, h, bc), bc)
        if op in ("red_glk1", "red_glk2"):
            return _red_glk(x, coarse_k(k_fine, bc), 2.0 * h, bc, op)
        raise ValueError(f"coarse op {op} not defined for the higher-order vectors")
    if op == "galerkin":
        v1 = prolong_bilinear(x, fine_shape, bc)      # Eq. 5.7a
        v2 = apply_A(v1, k_fine, h, bc)               # Eq. 5.7b
        return restrict_bilinear_zt(v2, bc)           # Eq. 5.7c
    raise ValueError(op)
