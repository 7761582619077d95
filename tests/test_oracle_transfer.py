"""Pins for oracle/transfer.py (bilinear Z = I_{2h}^h and full weighting I_h^{2h})."""
import numpy as np
import pytest

import oracle
from workloads import random_field


def _interp_1d(n_fine, bc):
    """Eq. 3.6 written on NODE indices: even fine node i copies coarse node i/2, odd fine
    node averages coarse nodes (i-1)/2 and (i+1)/2.  Dirichlet: unknown u <-> node u+1 and
    boundary nodes hold 0; Sommerfeld: unknown u <-> node u."""
    if bc == "dirichlet":
        nc = (n_fine - 1) // 2
        node_of_f = lambda i: i + 1
        unk_of_cnode = lambda c: c - 1 if 1 <= c <= nc else None
    else:
        nc = (n_fine + 1) // 2
        node_of_f = lambda i: i
        unk_of_cnode = lambda c: c if 0 <= c < nc else None
    P = np.zeros((n_fine, nc))
    for i in range(n_fine):
        node = node_of_f(i)
        if node % 2 == 0:
            src = [(node // 2, 1.0)]
        else:
            src = [((node - 1) // 2, 0.5), ((node + 1) // 2, 0.5)]
        for cn, w in src:
            u = unk_of_cnode(cn)
            if u is not None:
                P[i, u] += w
    return P


def _dense(fn, shape_in):
    n = shape_in[0] * shape_in[1]
    cols = []
    for c in range(n):
        e = np.zeros(n, dtype=np.complex128)
        e[c] = 1.0
        cols.append(fn(e.reshape(shape_in)).ravel())
    return np.array(cols).T


@pytest.mark.parametrize("bc,shape", [("dirichlet", (7, 15)), ("dirichlet", (3, 5)),
                                      ("sommerfeld", (9, 5)), ("sommerfeld", (3, 7))])
def test_prolongation_is_tensor_linear_interpolation(bc, shape):
    """Eq. 3.9 is the tensor product of the 1D rule Eq. 3.6: Z = P_y (x) P_x."""
    cshape = oracle.coarse_shape(shape, bc)
    Z = _dense(lambda e: oracle.prolong_bilinear(e, shape, bc), cshape)
    Zk = np.kron(_interp_1d(shape[0], bc), _interp_1d(shape[1], bc))
    np.testing.assert_array_equal(Z, Zk)


@pytest.mark.parametrize("bc,shape", [("dirichlet", (7, 15)), ("sommerfeld", (9, 5)), ("sommerfeld", (5, 5))])
def test_restriction_is_quarter_transpose(bc, shape):
    """§3.2.1 "Z^T will be the full-weighting restriction operator": the 1/16 full
    weighting (Eq. 3.8) equals Z^T / 4 exactly."""
    cshape = oracle.coarse_shape(shape, bc)
    Z = _dense(lambda e: oracle.prolong_bilinear(e, shape, bc), cshape)
    R = _dense(lambda v: oracle.restrict_fw(v, bc), shape)
    np.testing.assert_array_equal(R, Z.T / 4)


@pytest.mark.parametrize("bc,shape", [("dirichlet", (7, 15)), ("sommerfeld", (9, 5)), ("sommerfeld", (5, 5))])
def test_deflation_restriction_is_transpose(bc, shape):
    """Reading R10: the deflation restriction is Z^T (Eq. 3.7, (1/2)(u_{2i-1} + 2u_{2i} + u_{2i+1})
    in each direction) -- exactly the transpose of the bilinear interpolation, 4x Eq. 3.8."""
    cshape = oracle.coarse_shape(shape, bc)
    Z = _dense(lambda e: oracle.prolong_bilinear(e, shape, bc), cshape)
    R = _dense(lambda v: oracle.restrict_bilinear_zt(v, bc), shape)
    np.testing.assert_array_equal(R, Z.T)
    one = np.ones(shape, complex)
    np.testing.assert_allclose(oracle.restrict_bilinear_zt(one, bc)[1:-1, 1:-1], 4.0, atol=1e-15)


def test_constant_and_linear_reproduction():
    """Full weighting keeps constants at coarse points whose 9 taps are unknowns
    (weights sum to 1); bilinear interpolation reproduces linear functions."""
    bc, shape = "sommerfeld", (9, 13)
    one = np.ones(shape, complex)
    r = oracle.restrict_fw(one, bc)
    np.testing.assert_allclose(r[1:-1, 1:-1], 1.0, rtol=0, atol=1e-15)
    cshape = oracle.coarse_shape(shape, bc)
    Jc, Ic = np.meshgrid(np.arange(cshape[0]) * 2.0, np.arange(cshape[1]) * 2.0, indexing="ij")
    lin_c = 0.3 + 1.7 * Ic - 0.4 * Jc
    J, I = np.meshgrid(np.arange(shape[0]) * 1.0, np.arange(shape[1]) * 1.0, indexing="ij")
    np.testing.assert_allclose(oracle.prolong_bilinear(lin_c + 0j, shape, bc), 0.3 + 1.7 * I - 0.4 * J, atol=1e-13)


def test_coarse_shapes_and_index_map():
    """§4 coarse (i_c,j_c) <-> fine (2 i_c - 1, 2 j_c - 1) (1-based, boundary included)."""
    assert oracle.coarse_shape((31, 31), "dirichlet") == (15, 15)
    assert oracle.coarse_shape((33, 33), "sommerfeld") == (17, 17)
    assert oracle.coarse_shape((73, 121), "sommerfeld") == (37, 61)
    assert not oracle.coarsenable((10, 16), "sommerfeld")
    assert not oracle.coarsenable((4, 4), "dirichlet")
    k = np.arange(35.0).reshape(5, 7)
    np.testing.assert_array_equal(oracle.coarse_k(k, "sommerfeld"), k[0::2, 0::2])
    np.testing.assert_array_equal(oracle.coarse_k(k, "dirichlet"), k[1::2, 1::2][:2, :3])


def test_transfer_linearity():
    bc, shape = "dirichlet", (15, 7)
    a, b = random_field(shape, 1), random_field(shape, 2)
    np.testing.assert_allclose(oracle.restrict_fw(a + 2j * b, bc),
                               oracle.restrict_fw(a, bc) + 2j * oracle.restrict_fw(b, bc), atol=1e-14)
