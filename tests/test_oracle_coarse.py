"""Pins for oracle/coarse.py (deflation coarse operators) and the deflation identities."""
import math

import numpy as np
import pytest

import oracle
from workloads import random_field, random_k
from tests.test_oracle_transfer import _dense, _interp_1d
from tests.test_oracle_operators import _T1


def _A_dense(shape, h, kval, bc):
    ny, nx = shape
    A = (np.kron(np.eye(ny), _T1(nx, h, kval, bc)) + np.kron(_T1(ny, h, kval, bc), np.eye(nx))) / h**2
    return A - kval**2 * np.eye(nx * ny)


@pytest.mark.parametrize("bc,shape", [("dirichlet", (7, 11)), ("sommerfeld", (9, 7))])
def test_galerkin_equals_dense_RAP(bc, shape):
    """E = I_h^{2h} A_h I_{2h}^h = Z^T A Z (§3.2.1, reading R10) with all three factors assembled
    densely from independent textbook forms (Kronecker sum for A, tensor linear interpolation
    for Z, its transpose for the restriction)."""
    h, kval = 1 / 8, 5.0
    Z = np.kron(_interp_1d(shape[0], bc), _interp_1d(shape[1], bc))
    A = _A_dense(shape, h, kval, bc)
    E = Z.T @ A @ Z
    k = np.full(shape, kval)
    cshape = oracle.coarse_shape(shape, bc)
    Eo = _dense(lambda x: oracle.apply_coarse_E(x, k, h, bc, "galerkin"), cshape)
    np.testing.assert_allclose(Eo, E, rtol=1e-13, atol=1e-10)


def test_galerkin_tensor_closed_form():
    """For a tensor-product operator the Galerkin coarse operator is the tensor product of
    1D Galerkin operators.  In 1D (linear interpolation P1 and its transpose) P1^T P1 = [1 6 1]/4
    and P1^T T P1 = [-1 2 -1]/2, so for homogeneous Dirichlet and constant k:
      E = [ (P^T T P)_y (x) (P^T P)_x + (P^T P)_y (x) (P^T T P)_x ] / h^2 - k^2 (P^T P)_y (x) (P^T P)_x.
    (Classic result; at H = 2h the interior Laplacian row is 4 x [-1 2 -1]/H^2 (x) [1 6 1]/8.)"""
    shape, h, kval = (15, 7), 1 / 16, 11.0
    def m1(n):
        return (6 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1)) / 4
    def t1(n):
        return (2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)) / 2
    nyc, nxc = oracle.coarse_shape(shape, "dirichlet")
    E = (np.kron(t1(nyc), m1(nxc)) + np.kron(m1(nyc), t1(nxc))) / h**2 - kval**2 * np.kron(m1(nyc), m1(nxc))
    k = np.full(shape, kval)
    Eo = _dense(lambda x: oracle.apply_coarse_E(x, k, h, "dirichlet", "galerkin"), (nyc, nxc))
    np.testing.assert_allclose(Eo, E, rtol=1e-13, atol=1e-9)


def test_red_o2_is_coarse_helmholtz():
    """ReD-O2 (§5.2.3) = the Eq. 2.7 stencil at mesh width 2h with the coarse wavenumber."""
    shape, h = (9, 13), 0.05
    k = random_k(shape, 9)
    x = random_field(oracle.coarse_shape(shape, "sommerfeld"), 2)
    kc = oracle.coarse_k(k, "sommerfeld")
    np.testing.assert_array_equal(oracle.apply_coarse_E(x, k, h, "sommerfeld", "red_o2"),
                                  oracle.apply_A(x, kc, 2 * h, "sommerfeld"))


def test_red_o4_fourth_order():
    """Eq. 5.11 is the 4th-order central Laplacian: on u = sin(pi x) sin(2 pi y) the interior
    error against -Delta u - k^2 u decays like H^4 (log-log slope 4 +- 0.2)."""
    errs, Hs = [], []
    for n in (16, 32, 64):
        h = 1.0 / (2 * n)                           # fine grid; coarse H = 1/n
        nf = 2 * n - 1
        k = np.full((nf, nf), 3.0)
        H = 2 * h
        xc = np.arange(1, n) * H
        X, Y = np.meshgrid(xc, xc)
        u = np.sin(math.pi * X) * np.sin(2 * math.pi * Y) + 0j
        y = oracle.apply_coarse_E(u, k, h, "dirichlet", "red_o4")
        exact = (5 * math.pi**2 - 9.0) * u
        errs.append(np.max(np.abs(y - exact)[2:-2, 2:-2]))
        Hs.append(H)
    slope = np.polyfit(np.log(Hs), np.log(errs), 1)[0]
    assert abs(slope - 4.0) < 0.2, slope


@pytest.mark.parametrize("bc,shape", [("dirichlet", (15, 15)), ("sommerfeld", (9, 17))])
def test_deflation_identities(bc, shape):
    """With E = Z^T A Z (up to the 1/4) solved exactly:  P_h A Z = 0 (P_h = I - A Q_h) and
    P_{A-DEF1} A Z x = Z x (Eq. 3.21: M^{-1} P_h A Z x + Q_h A Z x)."""
    k = random_k(shape, 5, 5.0, 15.0)
    s = oracle.Solver(k, 1 / 16, bc, oracle.SolverParams(inner_solver="direct"))
    xc = random_field(s.cshape, 3)
    Zx = oracle.prolong_bilinear(xc, shape, bc)
    AZx = s.A(Zx)
    np.testing.assert_allclose(s.Q(AZx), Zx, rtol=0, atol=1e-10 * np.abs(Zx).max())
    np.testing.assert_allclose(AZx - s.A(s.Q(AZx)), 0, atol=1e-9 * np.abs(AZx).max())
    np.testing.assert_allclose(s.adef1(AZx), Zx, atol=1e-9 * np.abs(Zx).max())


def test_red_o6_sixth_order():
    """ReD-O6 (Eq. 5.10, 7-point central second derivative per direction): on
    u = sin(pi x) sin(2 pi y) the interior error against -Delta u - k^2 u decays like H^6."""
    errs, Hs = [], []
    for n in (16, 32, 64):
        h = 1.0 / (2 * n)
        nf = 2 * n - 1
        k = np.full((nf, nf), 3.0)
        H = 2 * h
        xc = np.arange(1, n) * H
        X, Y = np.meshgrid(xc, xc)
        u = np.sin(math.pi * X) * np.sin(2 * math.pi * Y) + 0j
        y = oracle.apply_coarse_E(u, k, h, "dirichlet", "red_o6")
        exact = (5 * math.pi**2 - 9.0) * u
        errs.append(np.max(np.abs(y - exact)[3:-3, 3:-3]))
        Hs.append(H)
    slope = np.polyfit(np.log(Hs), np.log(errs), 1)[0]
    assert abs(slope - 6.0) < 0.3, slope


def test_cmpo4_coefficients_meet_appendix_b_constraints():
    """PAPER.md Appendix B Eq. B.1/B.2: a_0 + 4a_s + 4a_c = 0, a_s + 2a_c = -1,
    b_0 + 4b_s + 4b_c = 1 for the Singer-Turkel coefficients of §5.2.5."""
    from oracle.coarse import CMP_A, CMP_B
    assert abs(CMP_A["0"] + 4 * CMP_A["s"] + 4 * CMP_A["c"]) < 1e-15
    assert abs(CMP_A["s"] + 2 * CMP_A["c"] + 1.0) < 1e-15
    assert abs(CMP_B["0"] + 4 * CMP_B["s"] + 4 * CMP_B["c"] - 1.0) < 1e-15


def _plane_wave(n, kval, theta, bc):
    h = 1.0 / (2 * n)
    H = 2 * h
    if bc == "dirichlet":
        nf = 2 * n - 1
        xc = np.arange(1, n) * H
    else:
        nf = 2 * n + 1
        xc = np.arange(0, n + 1) * H
    X, Y = np.meshgrid(xc, xc)
    u = np.exp(1j * kval * (X * math.cos(theta) + Y * math.sin(theta)))
    return h, H, np.full((nf, nf), kval), u


def test_cmpo4_fourth_order_on_helmholtz_solutions():
    """The compact scheme (Singer & Turkel) is fourth-order for solutions of the Helmholtz
    equation: on a plane wave exp(ik(x cos t + y sin t)) the interior residual decays like H^4."""
    errs, Hs = [], []
    for n in (16, 32, 64):
        h, H, k, u = _plane_wave(n, 6.0, 0.7, "dirichlet")
        y = oracle.apply_coarse_E(u, k, h, "dirichlet", "red_cmpo4")
        errs.append(np.max(np.abs(y)[1:-1, 1:-1]))
        Hs.append(H)
    slope = np.polyfit(np.log(Hs), np.log(errs), 1)[0]
    assert abs(slope - 4.0) < 0.25, slope


def test_cmpo4_sommerfeld_ghost_is_high_order_for_outgoing_waves():
    """The fourth-order Sommerfeld ghost u_0 = 2ikh(1 - k^2h^2/6) u_1 + u_2
    is exact to O(h^5) for the wave leaving through the boundary, so on the left edge (away
    from corners) the residual of exp(-ikx) decays like H^3 (ghost error / H^2), much faster
    than the first-order condition would allow (H^1)."""
    errs, Hs = [], []
    for n in (16, 32, 64):
        h, H, k, u = _plane_wave(n, 6.0, math.pi, "sommerfeld")
        y = oracle.apply_coarse_E(u, k, h, "sommerfeld", "red_cmpo4")
        errs.append(np.max(np.abs(y[2:-2, 0])))
        Hs.append(H)
    slope = np.polyfit(np.log(Hs), np.log(errs), 1)[0]
    assert slope > 2.7, slope


# ---------------------------------------------------------------- ReD-9ptO2 (Appendix B)
def _lam_H(a, b, kval, H, p, q):
    """PAPER.md Appendix B, eigenvalues of the general 3x3 form with homogeneous Dirichlet
    conditions (Eq. eigs_A2h_optstcl, :1285-1290)."""
    cp, cq = np.cos(p * np.pi * H), np.cos(q * np.pi * H)
    k2H2 = kval * kval * H * H
    return ((a["0"] - b["0"] * k2H2) + 2 * (a["s"] - b["s"] * k2H2) * (cp + cq)
            + 4 * (a["c"] - b["c"] * k2H2) * cp * cq) / (H * H)


def test_9pto2_coefficients_meet_appendix_b_constraints():
    """a_0 + 4a_s + 4a_c = 0, a_s + 2a_c = -1, b_0 + 4b_s + 4b_c = 1."""
    from oracle.coarse import OPT9_A, OPT9_B
    assert abs(OPT9_A["0"] + 4 * OPT9_A["s"] + 4 * OPT9_A["c"]) < 1e-12
    assert abs(OPT9_A["s"] + 2 * OPT9_A["c"] + 1.0) < 1e-12
    assert abs(OPT9_B["0"] + 4 * OPT9_B["s"] + 4 * OPT9_B["c"] - 1.0) < 1e-15


def test_9pto2_printed_eigenvalues():
    """The coefficients reproduce the eigenvalues Appendix B prints: for k = 80 and h -> 0,
    lambda_H^{18,18} = -4.5 (the alignment target, :1296-1299); for k = 100 the smallest
    |lambda_H^{p,q}| is ~2.1 at (p, q) = (22, 23) (:1306-1308)."""
    from oracle.coarse import OPT9_A, OPT9_B
    H = 2e-5
    assert abs(_lam_H(OPT9_A, OPT9_B, 80.0, H, 18, 18) + 4.5) < 0.01
    P = np.arange(1, 200)
    pp, qq = np.meshgrid(P, P, indexing="ij")
    lam = _lam_H(OPT9_A, OPT9_B, 100.0, H, pp, qq)
    i = np.unravel_index(np.argmin(np.abs(lam)), lam.shape)
    assert {int(P[i[0]]), int(P[i[1]])} == {22, 23}
    assert abs(abs(lam[i]) - 2.1) < 0.05


def test_9pto2_dirichlet_eigenvectors():
    """Closed form: with constant k and homogeneous Dirichlet conditions the modes
    sin(p pi x) sin(q pi y) are eigenvectors of the 3x3 form with the eigenvalues of
    Eq. eigs_A2h_optstcl (the implementation, including its zero boundary taps)."""
    from oracle.coarse import OPT9_A, OPT9_B
    n, kval = 16, 9.0
    h = 1.0 / (2 * n)
    H = 2 * h
    xc = np.arange(1, n) * H
    X, Y = np.meshgrid(xc, xc)
    kf = np.full((2 * n - 1, 2 * n - 1), kval)
    for p, q in ((1, 1), (3, 7), (15, 2), (8, 8)):
        u = np.sin(p * np.pi * X) * np.sin(q * np.pi * Y) + 0j
        y = oracle.apply_coarse_E(u, kf, h, "dirichlet", "red_9pto2")
        lam = _lam_H(OPT9_A, OPT9_B, kval, H, p, q)
        np.testing.assert_allclose(y, lam * u, atol=1e-9 * abs(lam) + 1e-9)


def test_9pto2_second_order_on_helmholtz_solutions():
    """Consistency: on a plane wave the interior residual of ReD-9ptO2 decays like H^2 (a
    second-order scheme, unlike ReD-cmpO4's H^4)."""
    errs, Hs = [], []
    for n in (16, 32, 64):
        h, H, k, u = _plane_wave(n, 6.0, 0.7, "dirichlet")
        y = oracle.apply_coarse_E(u, k, h, "dirichlet", "red_9pto2")
        errs.append(np.max(np.abs(y)[1:-1, 1:-1]))
        Hs.append(H)
    slope = np.polyfit(np.log(Hs), np.log(errs), 1)[0]
    assert abs(slope - 2.0) < 0.25, slope


def test_9pto2_sommerfeld_ghost_is_second_order():
    """Reading R22: the second-order ghost u_0 = 2ikH u_1 + u_2 leaves an O(H) residual on the
    boundary for the outgoing wave (ghost error O(H^3) / H^2), against O(H^3) with ReD-cmpO4's
    fourth-order ghost."""
    errs, Hs = [], []
    for n in (16, 32, 64):
        h, H, k, u = _plane_wave(n, 6.0, math.pi, "sommerfeld")
        y = oracle.apply_coarse_E(u, k, h, "sommerfeld", "red_9pto2")
        errs.append(np.max(np.abs(y[2:-2, 0])))
        Hs.append(H)
    slope = np.polyfit(np.log(Hs), np.log(errs), 1)[0]
    assert 0.7 < slope < 1.5, slope
