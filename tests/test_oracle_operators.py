"""Pins for oracle/operators.py (A_h, M_h) against what the paper and mathematics fix."""
import math

import numpy as np
import pytest

import oracle
from workloads import random_field, random_k


def _nodes(n_unknown, h, offset):
    return (np.arange(n_unknown) + offset) * h


@pytest.mark.parametrize("p,q", [(1, 1), (2, 3), (5, 1), (7, 6)])
def test_dirichlet_eigenfunctions(p, q):
    """Appendix B: with homogeneous Dirichlet conditions the 5-point stencil has
    eigenvectors sin(i pi x) sin(j pi y) and eigenvalues
    (1/h^2)[4 - 2cos(i pi h) - 2cos(j pi h) - k^2 h^2].  Rectangular domain [0,1]x[0,1/2]
    (y-modes sin(q pi y / Ly)), variable k enters pointwise."""
    h = 1.0 / 16
    nx, ny = 15, 7            # interior nodes of [0,1] x [0,0.5]
    Ly = 0.5
    x = _nodes(nx, h, 1)
    y = _nodes(ny, h, 1)
    X, Y = np.meshgrid(x, y)
    u = np.sin(p * math.pi * X) * np.sin(q * math.pi * Y / Ly)
    lam_lap = (4 - 2 * math.cos(p * math.pi * h) - 2 * math.cos(q * math.pi * h / Ly)) / h**2
    k = random_k((ny, nx), seed=p * 10 + q)
    v = oracle.apply_A(u, k, h, "dirichlet")
    np.testing.assert_allclose(v, (lam_lap - k**2) * u, rtol=0, atol=1e-9 * np.abs(lam_lap))
    # constant k: exact eigenpair
    k0 = np.full((ny, nx), 20.0)
    v0 = oracle.apply_A(u, k0, h, "dirichlet")
    lam = (4 - 2 * math.cos(p * math.pi * h) - 2 * math.cos(q * math.pi * h / Ly) - 400.0 * h * h) / h**2
    np.testing.assert_allclose(v0, lam * u, atol=1e-9 * abs(lam_lap))


def _T1(n, h, k, bc):
    """1D second difference (textbook), Sommerfeld end rows from 1D ghost elimination
    u_{-1} = u_1 + 2 i h k u_0 (Eq. 2.8) -> (2 - 2ikh) u_0 - 2 u_1."""
    T = (2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)).astype(np.complex128)
    if bc == "sommerfeld":
        T[0, 0] = 2 - 2j * k * h
        T[0, 1] = -2
        T[-1, -1] = 2 - 2j * k * h
        T[-1, -2] = -2
    return T


@pytest.mark.parametrize("bc", ["dirichlet", "sommerfeld"])
@pytest.mark.parametrize("shape", [(5, 5), (6, 9), (9, 4)])
def test_kronecker_sum_assembly(bc, shape):
    """A = (I_y (x) T_x + T_y (x) I_x)/h^2 - k^2 I (constant k): the textbook Kronecker-sum
    form of the 5-point operator; the Sommerfeld corner gets 4 - 4ikh (Eq. 2.10)."""
    ny, nx = shape
    h, kval = 0.1, 3.7
    A = (np.kron(np.eye(ny), _T1(nx, h, kval, bc)) + np.kron(_T1(ny, h, kval, bc), np.eye(nx))) / h**2
    A -= kval**2 * np.eye(nx * ny)
    k = np.full(shape, kval)
    for seed in range(5):
        u = random_field(shape, seed)
        np.testing.assert_allclose(oracle.apply_A(u, k, h, bc).ravel(), A @ u.ravel(), rtol=1e-13, atol=1e-10)
    if bc == "sommerfeld":
        assert abs(A[0, 0] * h * h - (4 - kval**2 * h * h - 4j * kval * h)) < 1e-12


def test_sommerfeld_ghost_point_form():
    """Eq. 2.8: ghost u_{0,j} = u_{2,j} + 2 h i k_{1,j} u_{1,j}; then the plain 5-point
    Laplacian with ghosts, minus k^2, must equal the eliminated stencils (Eq. 2.9/2.10)."""
    ny, nx, h = 7, 9, 0.05
    k = random_k((ny, nx), 3)
    u = random_field((ny, nx), 4)
    g = np.zeros((ny + 2, nx + 2), dtype=np.complex128)
    g[1:-1, 1:-1] = u
    g[1:-1, 0] = u[:, 1] + 2j * h * k[:, 0] * u[:, 0]
    g[1:-1, -1] = u[:, -2] + 2j * h * k[:, -1] * u[:, -1]
    g[0, 1:-1] = u[1, :] + 2j * h * k[0, :] * u[0, :]
    g[-1, 1:-1] = u[-2, :] + 2j * h * k[-1, :] * u[-1, :]
    lap = (4 * g[1:-1, 1:-1] - g[1:-1, :-2] - g[1:-1, 2:] - g[:-2, 1:-1] - g[2:, 1:-1]) / h**2
    np.testing.assert_allclose(oracle.apply_A(u, k, h, "sommerfeld"), lap - k**2 * u, rtol=1e-12, atol=1e-8)


@pytest.mark.parametrize("bc", ["dirichlet", "sommerfeld"])
def test_cslp_shift(bc):
    """Eq. 3.1: M_{(1,0)} = A_h, and M_{(b1,b2)} - A_h = -(b1 - 1 + i b2) I(k^2)."""
    shape, h = (8, 11), 0.07
    k = random_k(shape, 7)
    u = random_field(shape, 8)
    A = oracle.apply_A(u, k, h, bc)
    np.testing.assert_array_equal(oracle.apply_M(u, k, h, bc, (1.0, 0.0)), A)
    for b1, b2 in [(1.0, 0.5), (0.8, -0.3)]:
        M = oracle.apply_M(u, k, h, bc, (b1, b2))
        np.testing.assert_allclose(M - A, -(b1 - 1 + 1j * b2) * k**2 * u, rtol=1e-12, atol=1e-9)


def test_interior_coefficient_example():
    """SPEC-style arithmetic example (Eq. 2.7): k=20, h=1/32 -> centre (4 - 0.390625)*1024 = 3696."""
    ap, aw, *_ = oracle.stencil_coefficients(np.full((3, 3), 20.0), 1 / 32, "dirichlet")
    assert ap[1, 1] == pytest.approx(3696.0, rel=1e-15)
    assert aw[1, 1] == pytest.approx(-1024.0)


def test_zero_and_linearity():
    shape, h = (6, 5), 0.2
    k = random_k(shape, 1)
    for bc in ("dirichlet", "sommerfeld"):
        assert not np.any(oracle.apply_A(np.zeros(shape, complex), k, h, bc))
        a, b = random_field(shape, 1), random_field(shape, 2)
        lhs = oracle.apply_A(2.0 * a - 3j * b, k, h, bc)
        rhs = 2.0 * oracle.apply_A(a, k, h, bc) - 3j * oracle.apply_A(b, k, h, bc)
        np.testing.assert_allclose(lhs, rhs, rtol=1e-12, atol=1e-9)
