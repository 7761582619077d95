"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times:
sampled outputs the oracle computes one by one (operator applies on local windows), and
properties that hold at any size (true residual of the solve)."""
import numpy as np
import pytest
import torch

import oracle
from workloads import config_problem

pytestmark = pytest.mark.gpu


def _sample_points(ny, nx, rng, count=64):
    pts = [(0, 0), (0, nx - 1), (ny - 1, 0), (ny - 1, nx - 1), (ny // 2, nx // 2), (1, nx // 3), (ny - 2, 5)]
    pts += [(int(rng.integers(ny)), int(rng.integers(nx))) for _ in range(count)]
    return pts


def _window(a, j, i, r=1):
    j0, j1 = max(0, j - r), min(a.shape[0], j + r + 1)
    i0, i1 = max(0, i - r), min(a.shape[1], i + r + 1)
    return (j0, j1, i0, i1)


@pytest.mark.parametrize("name", ["c4_micro_16385", "c1_k400"])
def test_apply_A_sampled(lib, name):
    """The fine-grid operator at full size: each sampled output equals the oracle's
    Algorithm-2 apply on the 3x3 window around it (window edges coincide with the global
    boundary exactly when the sample sits on it)."""
    p_meta = config_problem(name) if name != "c4_micro_16385" else None
    if p_meta is None:
        n = 16383
        h = 1.0 / 16384
        k = torch.full((n, n), 0.625 * 16384, dtype=torch.float64, device="cuda")
        bc = "dirichlet"
    else:
        n, h, bc = p_meta.nx, p_meta.h, p_meta.bc
        k = torch.from_numpy(p_meta.k).cuda()
    H = lib.Helm(n, n, h, bc, k, {"inner_maxit": 8})
    g = torch.Generator(device="cuda").manual_seed(5)
    u = torch.complex(torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64),
                      torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64))
    y = H.apply_A(u)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    errs = []
    for (j, i) in _sample_points(n, n, rng):
        j0, j1, i0, i1 = _window(u, j, i)
        uw = u[j0:j1, i0:i1].cpu().numpy()
        kw = k[j0:j1, i0:i1].cpu().numpy()
        vo = oracle.apply_A(uw, kw, h, bc)[j - j0, i - i0]
        vg = y[j, i].item()
        errs.append(abs(vg - vo) / max(abs(vo), 1e-300))
    H.close()
    del u, y, k
    torch.cuda.empty_cache()
    assert max(errs) < 1e-12


def test_bench_workload_solve_residual(lib):
    """bench.py's workload (configs[1], k = 400, h = 1/640, APD + Galerkin E, bench.py's
    inner setting): the GPU solution's true relative residual, measured with the oracle's
    operator, meets 1e-6."""
    import bench
    p = config_problem("c1_k400")
    H = lib.helm_setup(p, bench.DEFAULT_METHOD)
    x, rep = H.solve(torch.from_numpy(p.b).cuda(), tol=1e-6, maxit=1000)
    assert rep["converged"]
    x = x.cpu().numpy()
    r = p.b - oracle.apply_A(x, p.k, p.h, p.bc)
    assert np.linalg.norm(r) / np.linalg.norm(p.b) <= 1.05e-6
    H.close()
