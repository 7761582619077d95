"""GPU parity: libhelm.so (through its C ABI / ctypes binding) against the oracle, element by
element, on the same seeded inputs.  Tolerances (from BASELINE.json
north_star): a single operator apply within 1e-12 relative L2; outer iteration counts
within +-1; final solutions within 1e-6 relative L2."""
import numpy as np
import pytest
import torch

import oracle
from workloads import config_problem, mp_problem, random_field, random_k, wedge_problem

pytestmark = pytest.mark.gpu

OP_TOL = 1e-12


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def gpu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


class P:
    """A small problem description with an arbitrary k field."""

    def __init__(self, nx, ny, h, bc, k):
        self.nx, self.ny, self.h, self.bc, self.k = nx, ny, h, bc, k

    @property
    def shape(self):
        return (self.ny, self.nx)


GRIDS = [
    P(31, 31, 1 / 32, "dirichlet", np.full((31, 31), 20.0)),
    P(45, 37, 1 / 46, "dirichlet", random_k((37, 45), 1, 10, 60)),          # ragged, variable k
    P(33, 65, 1 / 64, "sommerfeld", random_k((65, 33), 2, 5, 40)),
    P(3, 3, 1 / 4, "dirichlet", np.full((3, 3), 2.0)),                       # smallest Dirichlet
    P(3, 5, 1 / 4, "sommerfeld", random_k((5, 3), 3, 1, 3)),                 # smallest Sommerfeld
    P(129, 257, 1 / 256, "sommerfeld", random_k((257, 129), 4, 10, 150)),
]
IDS = ["c0", "dir45x37", "som33x65", "dir3", "som3x5", "som129x257"]


@pytest.fixture(params=list(range(len(GRIDS))), ids=IDS)
def case(request, lib):
    p = GRIDS[request.param]
    H = lib.Helm(p.nx, p.ny, p.h, p.bc, p.k)
    yield p, H
    H.close()


def test_apply_A(case):
    p, H = case
    for seed in range(3):
        u = random_field(p.shape, seed)
        y = H.apply_A(gpu(u)).cpu().numpy()
        assert rel(y, oracle.apply_A(u, p.k, p.h, p.bc)) < OP_TOL


def test_levels_and_M(case):
    p, H = case
    levels = oracle.build_hierarchy(p.k, p.h, p.bc)
    assert [L.shape for L in levels] == [lv[:2] for lv in H.levels]
    for l, L in enumerate(levels):
        assert H.levels[l][2] == pytest.approx(L.h, rel=1e-15)
        u = random_field(L.shape, 10 + l)
        y = H.apply_M(l, gpu(u)).cpu().numpy()
        assert rel(y, oracle.apply_M(u, L.k, L.h, p.bc, (1.0, 0.5))) < OP_TOL


def test_transfers(case):
    p, H = case
    levels = oracle.build_hierarchy(p.k, p.h, p.bc)
    for l in range(len(levels) - 1):
        v = random_field(levels[l].shape, 20 + l)
        assert rel(H.restrict(l, gpu(v)).cpu().numpy(), oracle.restrict_fw(v, p.bc)) < 1e-14
        e = random_field(levels[l + 1].shape, 30 + l)
        assert rel(H.prolong(l, gpu(e)).cpu().numpy(), oracle.prolong_bilinear(e, levels[l].shape, p.bc)) < 1e-14


VARIANTS = [("bilinear", "galerkin"), ("bilinear", "red_o2"), ("bilinear", "red_o4"), ("bilinear", "red_o6"),
            ("bilinear", "red_cmpo4"), ("high_order", "galerkin"), ("high_order", "red_glk1"),
            ("high_order", "red_glk2"), ("high_order", "red_o2"), ("high_order", "red_o4"), ("high_order", "red_o6"),
            ("high_order", "red_cmpo4"), ("bilinear", "red_9pto2"), ("high_order", "red_9pto2")]


@pytest.mark.parametrize("vec,op", VARIANTS)
def test_coarse_operator_and_vectors(lib, vec, op):
    for p in GRIDS:
        H = lib.Helm(p.nx, p.ny, p.h, p.bc, p.k, {"coarse_op": op, "vectors": vec})
        cs = H.levels[1][:2]
        x = random_field(cs, 5)
        y = H.apply_E(gpu(x)).cpu().numpy()
        yo = oracle.apply_coarse_E(x, p.k, p.h, p.bc, op, vec)
        assert rel(y, yo) < OP_TOL, (vec, op, p.shape, p.bc)
        v = random_field(p.shape, 6)
        zt = oracle.restrict_bilinear_zt(v, p.bc) if vec == "bilinear" else oracle.restrict_high_order(v, p.bc)
        assert rel(H.apply_Zt(gpu(v)).cpu().numpy(), zt) < 1e-14
        z = oracle.prolong_bilinear(x, p.shape, p.bc) if vec == "bilinear" else \
            oracle.prolong_high_order(x, p.shape, p.bc)
        assert rel(H.apply_Z(gpu(x)).cpu().numpy(), z) < 1e-14
        H.close()


def test_vcycle(case):
    """Fused down/up kernels + single-CTA tail (default), every starting level."""
    p, H = case
    levels = oracle.build_hierarchy(p.k, p.h, p.bc)
    for l in range(len(levels)):
        f = random_field(levels[l].shape, 40 + l)
        u = H.vcycle(l, gpu(f)).cpu().numpy()
        assert rel(u, oracle.vcycle(levels, f, l)) < 1e-11, l


@pytest.mark.parametrize("nu,tail,col,pipe", [((1, 1), 65536, -1, 0), ((1, 1), 8192, -1, 0), ((2, 2), 8192, -1, 0),
                                              ((2, 2), 0, -1, 0), ((1, 0), 8192, -1, 0), ((3, 1), 0, -1, 0),
                                              ((1, 1), 0, 0, 0), ((1, 1), 0, 500, 0), ((1, 1), 0, 0, 1), ((1, 1), 0, 0, 24), ((1, 1), 0, 0, 4),
                                              ((1, 1), 0, 0, 6)])
def test_vcycle_variants(lib, nu, tail, col, pipe):
    """Generic sweep counts (unfused kernels), the per-level path (tail 0, the default), the
    thread-block-cluster tail (levels distributed over the cluster's shared memories) and the
    column-streaming legs (col_min_n: 0 = every level, 500 = the larger ones)."""
    for p in (GRIDS[1], GRIDS[2], GRIDS[5]):
        H = lib.Helm(p.nx, p.ny, p.h, p.bc, p.k, {"nu_pre": nu[0], "nu_post": nu[1], "tail_max_n": tail,
                                                  "col_min_n": col, "col_pipe": pipe})
        levels = oracle.build_hierarchy(p.k, p.h, p.bc)
        for l in range(min(3, len(levels))):
            f = random_field(levels[l].shape, 50 + l)
            u = H.vcycle(l, gpu(f)).cpu().numpy()
            assert rel(u, oracle.vcycle(levels, f, l, nu_pre=nu[0], nu_post=nu[1])) < 1e-11, (p.shape, l, nu, tail, col,
                                                                                                  pipe)
        H.close()


@pytest.mark.parametrize("vec,op", [("bilinear", "galerkin"), ("bilinear", "red_o4"), ("high_order", "galerkin"),
                                    ("high_order", "red_glk2")])
def test_deflate(lib, vec, op):
    """z = P_{A-DEF1} v with the inner coarse solve at a tight tolerance (1e-10), so both
    sides run to the same well-defined E^{-1} c."""
    for p in GRIDS[:3]:
        prm = {"coarse_op": op, "inner_tol": 1e-10, "inner_maxit": 400, "vectors": vec}
        H = lib.Helm(p.nx, p.ny, p.h, p.bc, p.k, prm)
        s = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(coarse_op=op, inner_tol=1e-10, inner_maxit=400,
                                                              vectors=vec))
        v = random_field(p.shape, 7)
        z, its = H.deflate(gpu(v))
        zo = s.adef1(v)
        assert rel(z.cpu().numpy(), zo) < 1e-8, (op, p.shape)
        assert abs(its - s.inner_its[-1]) <= 1
        H.close()


# (problem, vectors, coarse op, inner_tol, inner_maxit).  At the paper's outer tolerance 1e-6
# both sides must take the same outer iteration count (+-1) and the GPU solution must meet the
# true residual.  The solutions themselves are compared at a tight outer tolerance (1e-10,
# reading R16): two valid 1e-6 solutions of this indefinite system legitimately differ by
# cond(A) x 1e-6 (~7e-6 for c1_k50; the oracle's own MGS and CGS2 variants differ by that
# much), while at 1e-10 both are within ~1e-9 of the unique discrete solution.
SOLVE_CASES = [
    ("c0_tiny", "bilinear", "galerkin", 1e-1, 200), ("c0_tiny", "bilinear", "red_o2", 1e-1, 200),
    ("c0_tiny", "bilinear", "red_o4", 1e-1, 200), ("c0_tiny", "bilinear", "galerkin", 0.0, 20),
    ("mp_som_k20", "bilinear", "galerkin", 1e-1, 200), ("mp_som_k40", "bilinear", "red_o4", 0.0, 30),
    ("c1_k50", "bilinear", "galerkin", 0.0, 40), ("c1_k50", "bilinear", "red_o4", 0.0, 40),
    ("c1_k50", "high_order", "galerkin", 0.0, 60), ("c1_k50", "high_order", "red_glk2", 0.0, 60),
    ("c1_k50", "high_order", "galerkin", 1e-1, 200),
    ("mp_som_k40", "high_order", "galerkin", 1e-1, 200), ("mp_som_k40", "high_order", "red_glk1", 0.0, 30),
    ("wedge_f10", "bilinear", "galerkin", 0.0, 40), ("wedge_f10", "high_order", "red_glk2", 1e-1, 300),
    ("mp_som_k40", "high_order", "red_cmpo4", 1e-1, 200), ("mp_som_k40", "high_order", "red_o6", 0.0, 40),
    ("wedge_f10", "high_order", "red_cmpo4", 0.0, 40), ("c1_k50", "bilinear", "red_o6", 1e-1, 200),
    ("c1_k50", "high_order", "red_9pto2", 1e-1, 200), ("mp_som_k40", "bilinear", "red_9pto2", 0.0, 40),
]


def _problem(name):
    if name == "mp_som_k20":
        return mp_problem(20.0, 32, "sommerfeld")
    if name == "mp_som_k40":
        return mp_problem(40.0, 64, "sommerfeld")
    if name == "wedge_f10":
        return wedge_problem(10.0)
    return config_problem(name)


@pytest.mark.parametrize("name,vec,op,itol,imax", SOLVE_CASES)
def test_solve(lib, name, vec, op, itol, imax):
    p = _problem(name)
    H = lib.helm_setup(p, {"coarse_op": op, "vectors": vec, "inner_tol": itol, "inner_maxit": imax})
    x, rep = H.solve(gpu(p.b), tol=1e-6, maxit=400)
    so = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(coarse_op=op, vectors=vec, inner_tol=itol,
                                                           inner_maxit=imax, maxit=400))
    xo, rep_o = so.solve(p.b)
    assert rep["converged"] and rep_o["converged"]
    assert abs(rep["outer_iterations"] - rep_o["outer_iterations"]) <= 1, (rep, rep_o["outer_iterations"])
    x = x.cpu().numpy()
    # true residual of the GPU solution, measured by the oracle's operator
    assert rel(oracle.apply_A(x, p.k, p.h, p.bc), p.b) <= 1.05e-6
    xt, rep_t = H.solve(gpu(p.b), tol=1e-10, maxit=600)
    so_t = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(coarse_op=op, vectors=vec, inner_tol=itol,
                                                             inner_maxit=imax, maxit=600, tol=1e-10))
    xo_t, rep_ot = so_t.solve(p.b)
    assert rep_t["converged"] and rep_ot["converged"]
    assert rel(xt.cpu().numpy(), xo_t) < 1e-6
    H.close()


@pytest.mark.parametrize("name,vec,op,tail,coop,col", [("c0_tiny", "bilinear", "galerkin", 0, 0, -1),
                                                       ("mp_som_k40", "high_order", "red_glk2", 0, 0, 0),
                                                       ("wedge_f10", "high_order", "galerkin", 0, 1, 1 << 20),
                                                       ("c1_k50", "high_order", "galerkin", 65536, 0, 1 << 20)])
def test_graph_and_host_loop_agree(lib, name, vec, op, tail, coop, col):
    """The CUDA-graph solve (conditional while nodes) and the host-polled loop run the same
    kernels in the same order: identical iteration counts and bitwise-identical solutions
    (with the cluster tail, and with the cooperative one-kernel Gram-Schmidt step)."""
    p = _problem(name)
    prm = {"coarse_op": op, "vectors": vec, "inner_tol": 1e-1, "inner_maxit": 300, "tail_max_n": tail,
           "coop": coop, "col_min_n": col}
    Hg = lib.helm_setup(p, dict(prm, graph=1))
    He = lib.helm_setup(p, dict(prm, graph=0))
    xg, rg = Hg.solve(gpu(p.b), tol=1e-6, maxit=200)
    xe, re_ = He.solve(gpu(p.b), tol=1e-6, maxit=200)
    if coop:   # the cooperative step also matches the oracle (outer count and true residual)
        so = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(coarse_op=op, vectors=vec, inner_tol=1e-1,
                                                               inner_maxit=300, maxit=200))
        xo, ro = so.solve(p.b)
        assert abs(rg["outer_iterations"] - ro["outer_iterations"]) <= 1
        assert rel(oracle.apply_A(xg.cpu().numpy(), p.k, p.h, p.bc), p.b) <= 1.05e-6
    for key in ("outer_iterations", "inner_iterations_total", "inner_iterations_max", "converged"):
        assert rg[key] == re_[key], key
    assert torch.equal(xg, xe)
    assert rg["kernels"] == re_["kernels"] > 0
    xg2, rg2 = Hg.solve(gpu(p.b), tol=1e-6, maxit=200)      # graph replay
    assert torch.equal(xg2, xg)
    Hg.close()
    He.close()


def test_restarted_outer(lib):
    """Outer FGMRES(m) restarts (host loop of graph-captured cycles) still meet the tolerance."""
    p = config_problem("c1_k50")
    H = lib.helm_setup(p, {"vectors": "high_order", "restart": 4, "inner_tol": 1e-1, "inner_maxit": 200})
    x, rep = H.solve(gpu(p.b), tol=1e-6, maxit=200)
    assert rep["converged"] and rep["restarts"] >= 1
    assert rel(oracle.apply_A(x.cpu().numpy(), p.k, p.h, p.bc), p.b) <= 1.05e-6
    H.close()


def test_zero_rhs(lib):
    p = config_problem("c0_tiny")
    H = lib.helm_setup(p)
    x, rep = H.solve(torch.zeros(p.shape, dtype=torch.complex128, device="cuda"))
    assert rep["outer_iterations"] == 0 and rep["converged"] and not torch.any(x != 0)
    H.close()


def test_solve_host_matches_device(lib):
    p = config_problem("c0_tiny")
    H = lib.helm_setup(p)
    xd, rd = H.solve(gpu(p.b))
    xh, rh = H.solve_host(p.b)
    assert rd["outer_iterations"] == rh["outer_iterations"]
    np.testing.assert_array_equal(xd.cpu().numpy(), xh)
    H.close()


def test_invalid_arguments(lib):
    with pytest.raises(lib.HelmError):
        lib.Helm(4, 4, 0.2, "dirichlet", np.ones((4, 4)))          # even: not coarsenable
    p = config_problem("c0_tiny")
    with pytest.raises(lib.HelmError):
        lib.helm_setup(p, {"max_levels": 1})
    with pytest.raises(lib.HelmError):
        lib.helm_setup(p, {"vectors": "bilinear", "coarse_op": "red_glk2"})   # ReD-Glk needs APD vectors
    H = lib.helm_setup(p)
    b = gpu(p.b)
    with pytest.raises(lib.HelmError):
        H.solve(b, x=b)                                             # aliasing
    H.close()


def test_coarsest_n_hierarchy_and_solve(lib):
    """A predefined coarsest size (coarsest_n, §4; bench.py uses 512): same hierarchy as
    the oracle's, and the bench method (APD + Galerkin, inner CSLP-FGMRES to 1e-1 capped at 50)
    on c1_k50 agrees with the oracle (outer count +-1 at 1e-6, solutions at 1e-10)."""
    p = config_problem("c1_k50")
    prm = {"vectors": "high_order", "coarse_op": "galerkin", "inner_tol": 1e-1, "inner_maxit": 50,
           "coarsest_n": 100}
    H = lib.helm_setup(p, prm)
    levels = oracle.build_hierarchy(p.k, p.h, p.bc, coarsest_n=100)
    assert [L.shape for L in levels] == [lv[:2] for lv in H.levels]
    assert levels[-1].shape[0] * levels[-1].shape[1] <= 100 < levels[-2].shape[0] * levels[-2].shape[1]
    op = dict(vectors="high_order", coarse_op="galerkin", inner_tol=1e-1, inner_maxit=50, coarsest_n=100)
    x, rep = H.solve(gpu(p.b), tol=1e-6, maxit=400)
    xo, rep_o = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(maxit=400, **op)).solve(p.b)
    assert abs(rep["outer_iterations"] - rep_o["outer_iterations"]) <= 1
    xt, _ = H.solve(gpu(p.b), tol=1e-10, maxit=600)
    xot, _ = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(maxit=600, tol=1e-10, **op)).solve(p.b)
    assert rel(xt.cpu().numpy(), xot) < 1e-6
    H.close()


@pytest.mark.parametrize("name,vec,op,itol,imax", [("c0_tiny", "bilinear", "galerkin", 1e-1, 200),
                                                    ("mp_som_k40", "high_order", "galerkin", 1e-1, 200),
                                                    ("c1_k50", "high_order", "red_glk2", 0.0, 40)])
def test_solve_gcr(lib, name, vec, op, itol, imax):
    """GCR outer (§6.3) against the oracle's GCR: outer count +-1 at 1e-6, the true
    residual, solutions at 1e-10; graph and host-polled loops agree bitwise."""
    p = _problem(name)
    prm = {"coarse_op": op, "vectors": vec, "inner_tol": itol, "inner_maxit": imax, "outer": "gcr"}
    H = lib.helm_setup(p, prm)
    x, rep = H.solve(gpu(p.b), tol=1e-6, maxit=400)
    op_ = dict(coarse_op=op, vectors=vec, inner_tol=itol, inner_maxit=imax, outer="gcr")
    xo, rep_o = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(maxit=400, **op_)).solve(p.b)
    assert rep["converged"] and rep_o["converged"]
    assert abs(rep["outer_iterations"] - rep_o["outer_iterations"]) <= 1, (rep, rep_o["outer_iterations"])
    assert rel(oracle.apply_A(x.cpu().numpy(), p.k, p.h, p.bc), p.b) <= 1.05e-6
    xt, _ = H.solve(gpu(p.b), tol=1e-10, maxit=600)
    xot, _ = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(maxit=600, tol=1e-10, **op_)).solve(p.b)
    assert rel(xt.cpu().numpy(), xot) < 1e-6
    He = lib.helm_setup(p, dict(prm, graph=0))
    xe, re_ = He.solve(gpu(p.b), tol=1e-6, maxit=400)
    x2, rep2 = H.solve(gpu(p.b), tol=1e-6, maxit=400)
    assert re_["outer_iterations"] == rep2["outer_iterations"] and torch.equal(xe, x2)
    H.close()
    He.close()


@pytest.mark.parametrize("pipe", [1, 24, 0])
def test_column_legs_interior_segments(lib, pipe):
    """Grids large enough that whole column segments (256 / 128 rows, 28 columns) lie in the
    interior, so the branch-free interior forms of the cp.async legs run next to the boundary
    forms (col_min_n = 0: every level uses the column legs)."""
    for p in (P(255, 767, 1 / 256, "dirichlet", random_k((767, 255), 7, 10, 200)),
              P(257, 769, 1 / 256, "sommerfeld", random_k((769, 257), 8, 10, 200))):
        H = lib.Helm(p.nx, p.ny, p.h, p.bc, p.k, {"col_min_n": 0, "col_pipe": pipe})
        levels = oracle.build_hierarchy(p.k, p.h, p.bc)
        f = random_field(p.shape, 77)
        u = H.vcycle(0, gpu(f)).cpu().numpy()
        assert rel(u, oracle.vcycle(levels, f, 0)) < 1e-11, (p.shape, pipe)
        H.close()


@pytest.mark.parametrize("vec", ["bilinear", "high_order"])
def test_fused_E_dots_matches(lib, vec):
    """fuse_dots = 1 (E apply and pass 1 of the delayed CGS2 in one kernel) gives the same inner
    solve as the separate kernels: same inner iterations, solutions equal to rounding."""
    p = GRIDS[0]
    v = random_field(p.shape, 7)
    out = {}
    for fuse in (0, 1):
        H = lib.Helm(p.nx, p.ny, p.h, p.bc, p.k, {"coarse_op": "galerkin", "vectors": vec, "inner_tol": 1e-8,
                                                  "inner_maxit": 200, "fuse_dots": fuse})
        z, its = H.deflate(gpu(v))
        out[fuse] = (z.cpu().numpy(), its)
        H.close()
    assert out[0][1] == out[1][1]
    assert rel(out[1][0], out[0][0]) < 1e-10


@pytest.mark.parametrize("vec", ["bilinear", "high_order"])
def test_streaming_E_bitwise_tile_kernel(lib, vec):
    """The column-streaming str-Glk kernel (e_stream = 1, the default) performs the tile kernel's
    arithmetic in the same order (up to the compiler's FMA contraction, which differs between the
    two kernels): E x equal to 1e-14 relative on every parity grid, on a ragged grid
    wider than several 28-column warp bands and taller than several row segments, and on
    the configs[4] 2047^2 block (1023^2 coarse)."""
    grids = GRIDS + [P(255, 127, 1 / 256, "dirichlet", random_k((127, 255), 8, 10, 90)),
                     P(193, 97, 1 / 192, "sommerfeld", random_k((97, 193), 9, 5, 70))]
    big = config_problem("c4_weak_2049")
    grids.append(P(big.nx, big.ny, big.h, big.bc, big.k))
    for p in grids:
        ys = []
        for es in (0, 1):
            H = lib.Helm(p.nx, p.ny, p.h, p.bc, p.k, {"coarse_op": "galerkin", "vectors": vec, "e_stream": es})
            x = random_field(H.levels[1][:2], 11)
            ys.append(H.apply_E(gpu(x)).cpu().numpy())
            H.close()
        assert rel(ys[1], ys[0]) < 1e-14, (p.shape, p.bc, vec, rel(ys[1], ys[0]))



def test_tma_column_legs(lib):
    """The TMA-staged column legs (tma = 3: both legs; the default 1 stages the up leg only)
    against the oracle's V-cycle and bitwise against the per-lane cp.async legs (tma = 0): same arithmetic,
    only the staging differs.  Column legs on every level (col_min_n = 0), Dirichlet and
    Sommerfeld, ragged sizes spanning several 28-column warp bands and row segments, variable k;
    plus the configs[4] block with the default leg choice (column legs on the 2047^2 level)."""
    cases = [P(255, 127, 1 / 256, "dirichlet", random_k((127, 255), 12, 10, 90)),
             P(193, 97, 1 / 192, "sommerfeld", random_k((97, 193), 13, 5, 70)),
             P(61, 45, 1 / 60, "sommerfeld", random_k((45, 61), 14, 5, 30))]
    for p in cases:
        s = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams())
        u = random_field(p.shape, 15)
        outs = []
        for tma in (3, 0):
            H = lib.Helm(p.nx, p.ny, p.h, p.bc, p.k, {"col_min_n": 0, "tma": tma})
            outs.append(H.vcycle(0, gpu(u)).cpu().numpy())
            H.close()
        assert rel(outs[0], s.vcycle(u, 0)) < 1e-11, p.shape
        assert np.array_equal(outs[0], outs[1]), (p.shape, rel(outs[0], outs[1]))
    big = config_problem("c4_weak_2049")
    u = random_field(big.shape, 16)
    outs = []
    for tma in (3, 1, 0):
        H = lib.Helm(big.nx, big.ny, big.h, big.bc, big.k, {"tma": tma})
        outs.append(H.vcycle(0, gpu(u)).cpu().numpy())
        H.close()
    assert np.array_equal(outs[0], outs[2]) and np.array_equal(outs[1], outs[2]), rel(outs[0], outs[2])


@pytest.mark.parametrize("vec", ["bilinear", "high_order"])
def test_tlkm_apply_and_solve(lib, vec):
    """Practical TLKM (reading R23): one application at a tight coarse tolerance matches the
    oracle's; solves match its outer counts (+-1) and, at 1e-10, its solution."""
    for p in GRIDS[:3]:
        prm = {"precond": "tlkm", "coarse_op": "red_o2", "vectors": vec, "inner_tol": 1e-10, "inner_maxit": 600}
        H = lib.Helm(p.nx, p.ny, p.h, p.bc, p.k, prm)
        s = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(preconditioner="tlkm", coarse_op="red_o2", vectors=vec,
                                                              inner_tol=1e-10, inner_maxit=600))
        v = random_field(p.shape, 21)
        z, its = H.deflate(gpu(v))
        assert rel(z.cpu().numpy(), s.tlkm(v)) < 1e-8, p.shape
        H.close()
    for name in ("c0_tiny", "mp_som_k20"):
        pr = _problem(name)
        prm = {"precond": "tlkm", "coarse_op": "red_o2", "vectors": vec, "inner_tol": 1e-8, "inner_maxit": 600}
        H = lib.helm_setup(pr, prm)
        x, rep = H.solve(gpu(pr.b), tol=1e-6, maxit=300)
        so = oracle.Solver(pr.k, pr.h, pr.bc, oracle.SolverParams(preconditioner="tlkm", coarse_op="red_o2", vectors=vec,
                                                                  inner_tol=1e-8, inner_maxit=600, maxit=300))
        xo, ro = so.solve(pr.b)
        assert rep["converged"] and ro["converged"]
        assert abs(rep["outer_iterations"] - ro["outer_iterations"]) <= 1, (rep, ro["outer_iterations"])
        xt, _ = H.solve(gpu(pr.b), tol=1e-10, maxit=400)
        so_t = oracle.Solver(pr.k, pr.h, pr.bc, oracle.SolverParams(preconditioner="tlkm", coarse_op="red_o2",
                                                                    vectors=vec, inner_tol=1e-8, inner_maxit=600,
                                                                    maxit=400, tol=1e-10))
        xo_t, _ = so_t.solve(pr.b)
        assert rel(xt.cpu().numpy(), xo_t) < 1e-6
        H.close()


@pytest.mark.parametrize("name,vec,op,itol", [("c1_k50", "high_order", "galerkin", 0.5),
                                              ("mp_som_k40", "high_order", "galerkin", 0.3),
                                              ("c0_tiny", "bilinear", "red_o4", 0.1)])
def test_lagged_stepb_counts(lib, name, vec, op, itol):
    """helm_params.lag_stepb (the inner Arnoldi loop decision taken one iteration late from the
    corrected column, the discarded column dropped): the inner solves converge early here, and
    every inner solve must stop at the oracle's own count (per outer iteration; +-1 where the
    test is rounding-decided, reading R13), with the same outer count as lag_stepb = 0."""
    p = _problem(name)
    so = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(coarse_op=op, vectors=vec, inner_tol=itol,
                                                           inner_maxit=200, maxit=400))
    xo, rep_o = so.solve(p.b)
    its_o = rep_o["inner_iterations"]
    assert max(its_o) < 200   # the inner solves really converge (the lagged path is exercised)
    reps = {}
    for lag in (0, 1):
        H = lib.helm_setup(p, {"coarse_op": op, "vectors": vec, "inner_tol": itol, "inner_maxit": 200,
                               "lag_stepb": lag})
        x, rep = H.solve(gpu(p.b), tol=1e-6, maxit=400)
        assert rep["converged"]
        assert rel(oracle.apply_A(x.cpu().numpy(), p.k, p.h, p.bc), p.b) <= 1.05e-6
        reps[lag] = rep
        H.close()
    for lag in (0, 1):
        r = reps[lag]
        assert abs(r["outer_iterations"] - rep_o["outer_iterations"]) <= 1
        n = min(r["outer_iterations"], rep_o["outer_iterations"])
        assert abs(r["inner_iterations_total"] - sum(its_o[:r["outer_iterations"]])) <= max(2, n // 10), (r, its_o)
        assert r["inner_iterations_max"] <= max(its_o) + 1
    assert reps[0]["outer_iterations"] == reps[1]["outer_iterations"]


def test_dots_cluster_option(lib):
    """helm_params.dots_cluster (pass 1 summed over thread-block clusters, no reduction kernel;
    off by default): same outer / inner counts as the oracle (+-1, R13), true residual met."""
    p = _problem("c1_k50")
    prm = {"coarse_op": "galerkin", "vectors": "high_order", "inner_tol": 1e-1, "inner_maxit": 50}
    so = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(coarse_op="galerkin", vectors="high_order", inner_tol=1e-1,
                                                           inner_maxit=50, maxit=400))
    xo, rep_o = so.solve(p.b)
    H = lib.helm_setup(p, dict(prm, dots_cluster=1))
    x, rep = H.solve(gpu(p.b), tol=1e-6, maxit=400)
    assert rep["converged"] and abs(rep["outer_iterations"] - rep_o["outer_iterations"]) <= 1
    assert abs(rep["inner_iterations_total"] - sum(rep_o["inner_iterations"][:rep["outer_iterations"]])) <= 2
    assert rel(oracle.apply_A(x.cpu().numpy(), p.k, p.h, p.bc), p.b) <= 1.05e-6
    H.close()


def test_large_inner_basis_setup(lib):
    """A 3000-column inner basis (Tables 1-2 runs: coarse solve to 1e-8) sets up on one
    GPU: only the kernels the context can launch get their shared-memory limits raised (the
    peer transport's fused step kernels, the cluster pass 1 are not this context's)."""
    p = _problem("c0_tiny")
    H = lib.helm_setup(p, {"coarse_op": "galerkin", "vectors": "bilinear", "inner_tol": 1e-8, "inner_maxit": 3000})
    x, rep = H.solve(gpu(p.b), tol=1e-6, maxit=100)
    assert rep["converged"]
    assert rel(oracle.apply_A(x.cpu().numpy(), p.k, p.h, p.bc), p.b) <= 1.05e-6
    H.close()
