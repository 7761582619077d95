"""GPU parity on BASELINE.json configs[3] and configs[4] inputs, and at the bench method's own
setting (bench.DEFAULT_METHOD: APD vectors, str-Glk E, coarse CSLP-FGMRES(40) to 1e-1 capped at
160 steps, coarsest level <= 512 unknowns).

* Operators on the full configs[3] / configs[4] grids (whole-grid compare with the oracle, not
  windows): A within 1e-12, E = Z^T A Z within 1e-12, V-cycles from levels 0 and 1 within 1e-11,
  the deflation z = P v with a fixed coarse step count (inner_tol = 0, reading R15) within 1e-9.
* The bench method on a same-family smaller case (configs[1] k = 100, whose coarse solves also
  run at or near the step cap): outer count +-1 at 1e-6, true residual, solutions within
  1e-6 at 1e-10 (reading R16), and the 1e-6 operating point itself: the GPU's 1e-6 solution is
  no further from the 1e-10 solution than twice the oracle's own 1e-6 solution is.
* Algorithm 1's literal modified Gram-Schmidt (oracle orth="mgs") against the GPU's delayed
  CGS2 on the rounding-insensitive cases (fixed coarse step counts): counts +-1, solutions
  within 1e-6 at 1e-10 -- CGS2 shown equivalent to MGS rather than assumed (reading R13).
"""
import os

import numpy as np
import pytest
import torch

import oracle
from tests.test_gpu_parity import _problem, gpu, rel
from workloads import config_problem, random_field

pytestmark = pytest.mark.gpu


def _bench_method():
    import bench
    return dict(bench.DEFAULT_METHOD)


def _oracle_params(m, **kw):
    keys = ("vectors", "coarse_op", "inner_tol", "inner_maxit", "inner_restart", "coarsest_n", "restart")
    return oracle.SolverParams(**dict({k: m[k] for k in keys if k in m}, **kw))


def _host_gb():
    try:
        return os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE") / 2**30
    except (ValueError, OSError):
        return 0.0


def _operator_parity(lib, p, method, seeds=(1, 2), deflate_steps=6):
    """A, E, V-cycle (levels 0, 1) and z = P v on the whole grid of problem p."""
    H = lib.helm_setup(p, dict(method, inner_tol=0.0, inner_maxit=deflate_steps, inner_restart=0))
    s = oracle.Solver(p.k, p.h, p.bc, _oracle_params(method, inner_tol=0.0, inner_maxit=deflate_steps,
                                                     inner_restart=0))
    assert [L.shape for L in s.levels] == [lv[:2] for lv in H.levels]
    u = random_field(p.shape, seeds[0])
    assert rel(H.apply_A(gpu(u)).cpu().numpy(), s.A(u)) < 1e-12
    x = random_field(s.cshape, seeds[1])
    assert rel(H.apply_E(gpu(x)).cpu().numpy(), s.E(x)) < 1e-12
    assert rel(H.vcycle(0, gpu(u)).cpu().numpy(), s.vcycle(u, 0)) < 1e-11
    assert rel(H.vcycle(1, gpu(x)).cpu().numpy(), s.vcycle(x, 1)) < 1e-11
    z, its = H.deflate(gpu(u))
    zo = s.adef1(u)
    assert its == s.inner_its[-1] == deflate_steps
    assert rel(z.cpu().numpy(), zo) < 1e-9
    H.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["c3_marm_f40_2945", "c3_marm_f20_5889"])
def test_configs3_marmousi_operators(lib, name):
    """configs[3] (Marmousi-shaped, Sommerfeld, variable k) at full size."""
    _operator_parity(lib, config_problem(name), _bench_method())


def test_configs3_marmousi_red_glk2_E(lib):
    """The re-discretised ReD-Glk2 coarse operator on the configs[3] 2945 x 929 f = 40 input."""
    p = config_problem("c3_marm_f40_2945")
    m = dict(_bench_method(), coarse_op="red_glk2")
    H = lib.helm_setup(p, m)
    x = random_field(H.levels[1][:2], 3)
    yo = oracle.apply_coarse_E(x, p.k, p.h, p.bc, "red_glk2", "high_order")
    assert rel(H.apply_E(gpu(x)).cpu().numpy(), yo) < 1e-12
    H.close()


def test_configs4_weak_block_operators(lib):
    """configs[4]'s weak-scaling block (2047^2 unknowns, k = 1280, the bench workload)."""
    _operator_parity(lib, config_problem("c4_weak_2049"), _bench_method())


def test_configs4_strong_grid_operators(lib):
    """configs[4]'s strong-scaling grid (8191^2 unknowns, k = 1000): A, E and the V-cycle from
    levels 0 and 1 on the whole grid (the oracle needs ~20 GB of host memory here)."""
    if _host_gb() < 40:
        pytest.skip(f"host has {_host_gb():.0f} GB free; the whole-grid 8191^2 oracle needs ~40")
    p = config_problem("c4_strong_8193")
    m = _bench_method()
    H = lib.helm_setup(p, m)
    s = oracle.Solver(p.k, p.h, p.bc, _oracle_params(m))
    u = random_field(p.shape, 1)
    assert rel(H.apply_A(gpu(u)).cpu().numpy(), s.A(u)) < 1e-12
    assert rel(H.vcycle(0, gpu(u)).cpu().numpy(), s.vcycle(u, 0)) < 1e-11
    del u
    x = random_field(s.cshape, 2)
    assert rel(H.apply_E(gpu(x)).cpu().numpy(), s.E(x)) < 1e-12
    assert rel(H.vcycle(1, gpu(x)).cpu().numpy(), s.vcycle(x, 1)) < 1e-11
    H.close()
    torch.cuda.empty_cache()


def test_bench_method_same_family(lib):
    """bench.py's method on configs[1] k = 100 (159^2, coarse solves at or near the cap)."""
    p = config_problem("c1_k100")
    m = _bench_method()
    H = lib.helm_setup(p, m)
    x6, rep = H.solve(gpu(p.b), tol=1e-6, maxit=600)
    so = oracle.Solver(p.k, p.h, p.bc, _oracle_params(m, tol=1e-6, maxit=600))
    xo6, rep_o = so.solve(p.b)
    assert rep["converged"] and rep_o["converged"]
    assert abs(rep["outer_iterations"] - rep_o["outer_iterations"]) <= 1, (rep, rep_o["outer_iterations"])
    assert rep["inner_restarts"] > 0 and rep["inner_iterations_max"] > m["inner_restart"]
    x6 = x6.cpu().numpy()
    assert rel(oracle.apply_A(x6, p.k, p.h, p.bc), p.b) <= 1.05e-6
    x10, rep_t = H.solve(gpu(p.b), tol=1e-10, maxit=800)
    xo10, rep_ot = oracle.Solver(p.k, p.h, p.bc, _oracle_params(m, tol=1e-10, maxit=800)).solve(p.b)
    assert rep_t["converged"] and rep_ot["converged"]
    assert rel(x10.cpu().numpy(), xo10) < 1e-6
    # the 1e-6 operating point: no worse than twice the oracle's own distance to the 1e-10 solution
    d_gpu, d_or = rel(x6, xo10), rel(xo6, xo10)
    assert d_gpu <= 2.0 * d_or + 1e-9, (d_gpu, d_or)
    H.close()


# rounding-insensitive solves (fixed coarse step counts) against the literal MGS of Algorithm 1
MGS_CASES = [("c0_tiny", "bilinear", "galerkin", 20), ("c1_k50", "high_order", "galerkin", 60),
             ("mp_som_k40", "bilinear", "red_o4", 30), ("wedge_f10", "high_order", "red_glk2", 40)]


@pytest.mark.parametrize("name,vec,op,imax", MGS_CASES)
def test_solve_against_mgs_oracle(lib, name, vec, op, imax):
    p = _problem(name)
    prm = {"coarse_op": op, "vectors": vec, "inner_tol": 0.0, "inner_maxit": imax}
    H = lib.helm_setup(p, prm)
    op_ = dict(coarse_op=op, vectors=vec, inner_tol=0.0, inner_maxit=imax, orth="mgs")
    x, rep = H.solve(gpu(p.b), tol=1e-6, maxit=400)
    xo, rep_o = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(**op_, maxit=400)).solve(p.b)
    assert rep["converged"] and rep_o["converged"]
    assert abs(rep["outer_iterations"] - rep_o["outer_iterations"]) <= 1, (rep, rep_o["outer_iterations"])
    assert rel(oracle.apply_A(x.cpu().numpy(), p.k, p.h, p.bc), p.b) <= 1.05e-6
    xt, _ = H.solve(gpu(p.b), tol=1e-10, maxit=600)
    xot, rep_ot = oracle.Solver(p.k, p.h, p.bc, oracle.SolverParams(**op_, maxit=600, tol=1e-10)).solve(p.b)
    assert rep_ot["converged"]
    assert rel(xt.cpu().numpy(), xot) < 1e-6
    H.close()
