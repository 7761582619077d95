"""Pins for oracle/multigrid.py (V-cycle) and oracle/krylov.py (FGMRES)."""
import numpy as np
import pytest

import oracle
from workloads import mp_problem, random_field, random_k
from tests.test_oracle_coarse import _A_dense
from tests.test_oracle_transfer import _interp_1d


def _M_dense(shape, h, kval, bc, beta):
    """M = A + (1 - beta1 - i beta2) k^2 I from the Kronecker-sum A (Eq. 3.1, reading R3)."""
    return _A_dense(shape, h, kval, bc) + (1 - beta[0] - 1j * beta[1]) * kval**2 * np.eye(shape[0] * shape[1])


@pytest.mark.parametrize("bc,shape", [("dirichlet", (7, 15)), ("sommerfeld", (9, 9))])
def test_two_grid_vcycle_equals_dense_operator(bc, shape):
    """With two levels and an exact coarse solve, one V(1,1) cycle from u = 0 is the dense
    two-grid operator  B = (I - w D^-1 M)[w D^-1 + P M_c^-1 R (I - M w D^-1)] + w D^-1
    (pre-smooth, residual, FW restriction, coarse solve, bilinear correction, post-smooth)."""
    h, kval, beta, w = 1 / 16, 9.0, (1.0, 0.5), 0.8
    M = _M_dense(shape, h, kval, bc, beta)
    cshape = oracle.coarse_shape(shape, bc)
    Mc = _M_dense(cshape, 2 * h, kval, bc, beta)
    Z = np.kron(_interp_1d(shape[0], bc), _interp_1d(shape[1], bc))
    R = Z.T / 4
    Dinv = np.diag(1.0 / np.diag(M))
    I = np.eye(M.shape[0])
    B = (I - w * Dinv @ M) @ (w * Dinv + Z @ np.linalg.solve(Mc, R @ (I - M @ (w * Dinv)))) + w * Dinv
    levels = oracle.build_hierarchy(np.full(shape, kval), h, bc, beta, max_levels=2)
    f = random_field(shape, 11)
    np.testing.assert_allclose(oracle.vcycle(levels, f).ravel(), B @ f.ravel(), rtol=1e-12, atol=1e-12 * np.abs(B @ f.ravel()).max())


def test_vcycle_linear_and_zero():
    shape, h = (31, 31), 1 / 32
    levels = oracle.build_hierarchy(random_k(shape, 2), h, "dirichlet")
    assert [L.shape for L in levels] == [(31, 31), (15, 15), (7, 7), (3, 3), (1, 1)]
    assert not np.any(oracle.vcycle(levels, np.zeros(shape, complex)))
    a, b = random_field(shape, 1), random_field(shape, 2)
    np.testing.assert_allclose(oracle.vcycle(levels, a - 2j * b),
                               oracle.vcycle(levels, a) - 2j * oracle.vcycle(levels, b), rtol=1e-12, atol=1e-14)


def test_jacobi_first_sweep():
    """R9: from u = 0 one damped Jacobi sweep is u = w D^-1 f; the exact solution is a fixed point."""
    shape, h = (5, 5), 0.1
    L = oracle.Level(shape, h, np.full(shape, 3.0), "sommerfeld", (1.0, 0.5))
    D = oracle.jacobi_diagonal(L)
    M = _M_dense(shape, h, 3.0, "sommerfeld", (1.0, 0.5))
    np.testing.assert_allclose(D.ravel(), np.diag(M), rtol=1e-15)
    u = random_field(shape, 1)
    f = L.M(u)
    np.testing.assert_allclose(u + 0.8 * (f - L.M(u)) / D, u, rtol=1e-15)


def test_fgmres_dense_exactness():
    """Full GMRES is exact in n steps: random dense 20x20 system, identity preconditioner."""
    rng = np.random.default_rng(0)
    A = rng.standard_normal((20, 20)) + 1j * rng.standard_normal((20, 20)) + 6 * np.eye(20)
    b = rng.standard_normal(20) + 0j
    hist = []
    x, its, conv = oracle.fgmres(lambda v: A @ v, lambda v: v, b, 1e-12, 40, history=hist)
    assert conv and its <= 20
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-10)
    assert all(hist[i + 1] <= hist[i] * (1 + 1e-12) for i in range(len(hist) - 1))
    x, its, conv = oracle.fgmres(lambda v: v, lambda v: v, b, 1e-12, 5)
    assert its == 1 and np.allclose(x, b)
    x, its, conv = oracle.fgmres(lambda v: A @ v, lambda v: v, np.zeros(20, complex), 1e-6, 5)
    assert its == 0 and not np.any(x)


@pytest.mark.parametrize("bc", ["dirichlet", "sommerfeld"])
@pytest.mark.parametrize("op", ["galerkin", "red_o2", "red_o4"])
def test_solver_matches_dense_solve(bc, op):
    """Brute force on a tiny grid: A-DEF1/CSLP FGMRES at tol 1e-11 reproduces the dense
    solution of the Kronecker-assembled A (relative error << 1e-6)."""
    p = mp_problem(12.0, 16, bc)
    A = _A_dense(p.shape, p.h, 12.0, bc)
    xd = np.linalg.solve(A, p.b.ravel())
    x, rep = oracle.solve(p, oracle.SolverParams(coarse_op=op, tol=1e-11, inner_tol=1e-3))
    assert rep["converged"] and rep["relres"] < 1e-10
    assert np.linalg.norm(x.ravel() - xd) / np.linalg.norm(xd) < 1e-8


def test_coarsest_n_stops_coarsening():
    """R7: coarsening stops at the first level with <= coarsest_n unknowns (§4)."""
    import numpy as np
    k = np.full((63, 63), 5.0)
    full = oracle.build_hierarchy(k, 1 / 64, "dirichlet")
    assert [L.shape for L in full][-1] == (1, 1)
    cut = oracle.build_hierarchy(k, 1 / 64, "dirichlet", coarsest_n=300)
    assert [L.shape for L in cut] == [(63, 63), (31, 31), (15, 15)]


def test_gcr_dense_exactness_and_minimal_residual():
    """GCR on a small dense complex system: converges to the dense solution; with the identity
    preconditioner its residuals equal GMRES's (both minimise ||b - Ax|| over the Krylov space,
    Eisenstat-Elman-Schultz), so the iteration counts agree with FGMRES's."""
    import numpy as np
    rng = np.random.default_rng(4)
    n = 30
    A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) + 8 * np.eye(n)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    mv = lambda v: A @ v
    ident = lambda v: v.copy()
    hg, hf = [], []
    x, its, conv = oracle.gcr(mv, ident, b, 1e-12, 200, history=hg)
    xf, itsf, convf = oracle.fgmres(mv, ident, b, 1e-12, 200, history=hf)
    assert conv and convf
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-9)
    np.testing.assert_allclose(hg[:6], hf[:6], rtol=1e-8)
    assert its == itsf


def test_gcr_outer_solver_matches_dense_solve():
    """The A-DEF1 preconditioned GCR (§6.3) solves the model problem to its tolerance."""
    import numpy as np
    from workloads import mp_problem
    p = mp_problem(10.0, 16, "sommerfeld")
    x, rep = oracle.solve(p, oracle.SolverParams(outer="gcr", inner_solver="direct", tol=1e-10))
    assert rep["converged"]
    r = p.b - oracle.apply_A(x, p.k, p.h, p.bc)
    assert np.linalg.norm(r) / np.linalg.norm(p.b) <= 1e-10


def test_tlkm_composition_dense():
    """Practical TLKM (reading R23) against its definition assembled from dense matrices:
    P = [I - M0^-1 A Z T^-1 Z^T + gamma Z T^-1 Z^T] M0^-1 with T = Z^T Z M1^-1 A_2h (PAPER.md
    Eq. 3.15-3.18 and :880), every factor built by applying the oracle's primitives to unit
    vectors -- pins the composition order (which operator is inverted where, the extra M^-1 on
    the deflation term, the shift gamma)."""
    import numpy as np
    from workloads import random_field, random_k
    shape, h, bc = (15, 15), 1 / 16, "dirichlet"
    k = random_k(shape, 3, 4, 12)
    s = oracle.Solver(k, h, bc, oracle.SolverParams(preconditioner="tlkm", coarse_op="red_o2", inner_solver="direct",
                                                    gamma=0.7))
    n0 = shape[0] * shape[1]
    cs = s.cshape
    n1 = cs[0] * cs[1]

    def dense(fn, nin, sin):
        cols = []
        for c in range(nin):
            e = np.zeros(nin, complex)
            e[c] = 1
            cols.append(fn(e.reshape(sin)).ravel())
        return np.array(cols).T
    M0 = dense(lambda v: s.vcycle(v, 0), n0, shape)
    M1 = dense(lambda v: s.vcycle(v, 1), n1, cs)
    A = dense(s.A, n0, shape)
    E = dense(s.E, n1, cs)
    Z = dense(s.Zp, n1, cs)
    Zt = dense(s.Zt, n0, shape)
    T = Zt @ Z @ M1 @ E
    Qt = Z @ np.linalg.solve(T, Zt)
    P = (np.eye(n0) - M0 @ A @ Qt + 0.7 * Qt) @ M0
    v = random_field(shape, 9)
    np.testing.assert_allclose(s.tlkm(v).ravel(), P @ v.ravel(), rtol=1e-9, atol=1e-9 * np.abs(P @ v.ravel()).max())


# ---------------------------------------------------------------- restarted FGMRES(m), reading R25

def _dense_system(n, seed, shift):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) + shift * np.eye(n)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return A, b


def test_restart_beyond_iterations_is_the_full_method():
    """FGMRES(m) with m >= the iterations the full method needs is the full method (bitwise)."""
    A, b = _dense_system(24, 5, 7.0)
    x0, it0, c0 = oracle.fgmres(lambda v: A @ v, lambda v: v, b, 1e-10, 200)
    x1, it1, c1 = oracle.fgmres(lambda v: A @ v, lambda v: v, b, 1e-10, 200, restart=it0)
    assert c0 and c1 and it0 == it1
    assert np.array_equal(x0, x1)


def test_restart_one_is_the_minimal_residual_iteration():
    """GMRES(1) is the minimal-residual iteration (Saad, Iterative Methods §5.3.2, closed form):
    alpha = (A r, r) / (A r, A r), x += alpha r, r -= alpha A r."""
    A, b = _dense_system(16, 6, 9.0)
    x, its, conv = oracle.fgmres(lambda v: A @ v, lambda v: v, b, 0.0, 7, restart=1)
    xm = np.zeros(16, complex)
    r = b.copy()
    for _ in range(7):
        ar = A @ r
        alpha = np.vdot(ar, r) / np.vdot(ar, ar)
        xm = xm + alpha * r
        r = r - alpha * ar
    assert its == 7 and not conv
    np.testing.assert_allclose(x, xm, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("m", [2, 3])
def test_flexible_restart_cycles_minimise_over_preconditioned_krylov(m):
    """With a fixed preconditioner P, each FGMRES(m) cycle from x minimises ||b - A(x + P K c)||
    over K = [r, (AP) r, ..., (AP)^{m-1} r] (right-preconditioned GMRES; Saad 1993 flexible
    GMRES reduces to it for constant P).  Reference: dense least squares per cycle."""
    A, b = _dense_system(20, 7, 5.0)
    rng = np.random.default_rng(8)
    P = np.eye(20) + 0.1 * (rng.standard_normal((20, 20)) + 1j * rng.standard_normal((20, 20)))
    ncyc = 4
    x, its, conv = oracle.fgmres(lambda v: A @ v, lambda v: P @ v, b, 0.0, m * ncyc, restart=m)
    xr = np.zeros(20, complex)
    for _ in range(ncyc):
        r = b - A @ xr
        K = [r]
        for _i in range(m - 1):
            K.append(A @ (P @ K[-1]))
        PK = P @ np.array(K).T
        c = np.linalg.lstsq(A @ PK, r, rcond=None)[0]
        xr = xr + PK @ c
    assert its == m * ncyc
    np.testing.assert_allclose(x, xr, rtol=1e-9, atol=1e-12)


def test_restarted_converges_to_dense_solution_with_original_norm():
    """A positive-real system (Hermitian part positive definite): GMRES(m) converges for every m
    (Elman 1982).  The stop is relative to the ORIGINAL ||b||: the true residual of the result
    meets tol * ||b||."""
    A, b = _dense_system(30, 9, 12.0)
    hist = []
    x, its, conv = oracle.fgmres(lambda v: A @ v, lambda v: v, b, 1e-9, 500, restart=3, history=hist)
    assert conv and its > 3
    assert np.linalg.norm(b - A @ x) <= 1e-9 * np.linalg.norm(b) * (1 + 1e-6)
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-7)
    assert len(hist) == its + 1 and hist[-1] <= 1e-9


def test_restarted_inner_solve_in_the_solver():
    """The restarted coarse solve is used by the solver (inner_restart) and still meets the
    outer tolerance; with inner_restart >= inner_maxit it is the unrestarted method bitwise."""
    p = mp_problem(12.0, 16, "sommerfeld")
    base = dict(vectors="high_order", inner_tol=1e-6, inner_maxit=40, tol=1e-8)
    x0, r0 = oracle.solve(p, oracle.SolverParams(**base))
    x1, r1 = oracle.solve(p, oracle.SolverParams(**base, inner_restart=40))
    assert np.array_equal(x0, x1) and r0["inner_iterations"] == r1["inner_iterations"]
    x2, r2 = oracle.solve(p, oracle.SolverParams(**base, inner_restart=4))
    assert r2["converged"] and r2["relres"] <= 1e-8
    assert max(r2["inner_iterations"]) > 4
    np.testing.assert_allclose(x2, x0, rtol=0, atol=1e-6 * np.abs(x0).max())


def test_gmres_left_minimises_preconditioned_residual():
    """Algorithm 1 as printed (oracle.gmres_left, reading R26): the k-th iterate minimises the
    PRECONDITIONED residual ||P(b - A x)|| over x in K_k(PA, Pb) (Saad 1993, left-preconditioned
    GMRES).  Reference: dense least squares over the explicit Krylov basis, for k = 1..5; and
    exactness in n steps, with the stop on ||P r|| / ||P b||."""
    A, b = _dense_system(20, 11, 5.0)
    rng = np.random.default_rng(12)
    P = np.eye(20) + 0.2 * (rng.standard_normal((20, 20)) + 1j * rng.standard_normal((20, 20)))
    for kk in range(1, 6):
        x, its, conv = oracle.gmres_left(lambda v: A @ v, lambda v: P @ v, b, 0.0, kk)
        K = [P @ b]
        for _i in range(kk - 1):
            K.append(P @ (A @ K[-1]))
        Kb = np.array(K).T
        c = np.linalg.lstsq(P @ A @ Kb, P @ b, rcond=None)[0]
        assert its == kk
        np.testing.assert_allclose(x, Kb @ c, rtol=1e-8, atol=1e-12)
    hist = []
    x, its, conv = oracle.gmres_left(lambda v: A @ v, lambda v: P @ v, b, 1e-12, 40, history=hist)
    assert conv and its <= 20
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-9)
    # the stopping quantity is the preconditioned relative residual
    assert np.linalg.norm(P @ (b - A @ x)) / np.linalg.norm(P @ b) <= 1e-12 * 1.01
    # exact preconditioner: one step
    x, its, conv = oracle.gmres_left(lambda v: A @ v, lambda v: np.linalg.solve(A, v), b, 1e-10, 5)
    assert its == 1 and conv
