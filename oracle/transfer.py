"""ORACLE (test infrastructure only) — inter-grid transfers (= deflation vectors Z, Z^T).

PAPER.md §3.2.1 Eq. 3.6 (1D linear interpolation), Eq. 3.8 (full-weighting restriction
stencil 1/16 [1 2 1; 2 4 2; 1 2 1]), Eq. 3.9 (bilinear interpolation stencil
1/4 [1 2 1; 2 4 2; 1 2 1]), "Z = I_{2h}^h", "Z^T will be the full-weighting restriction";
§4 "point (i_c, j_c) in the coarse grid corresponds to point (2 i_c - 1, 2 j_c - 1)".

Reading R4: taps that fall outside the unknown array are dropped without
renormalisation (Dirichlet: they are boundary nodes holding g = 0, so this is exact;
Sommerfeld: they lie outside the domain).  With this rule R = Z^T / 4 holds exactly.
"""
from __future__ import annotations

import numpy as np

from .operators import unknown_offset

FW = np.array([[1.0, 2.0, 1.0], [2.0, 4.0, 2.0], [1.0, 2.0, 1.0]]) / 16.0


def _coarse_n(n: int, bc: str):
    if n < 3 or n % 2 == 0:
        return None
    return (n - 1) // 2 if bc == "dirichlet" else (n + 1) // 2


def coarsenable(shape, bc: str) -> bool:
    ny, nx = shape
    return _coarse_n(nx, bc) is not None and _coarse_n(ny, bc) is not None


def coarse_shape(shape, bc: str):
    """Standard coarsening h -> 2h of a vertex-centred grid (§4)."""
    if not coarsenable(shape, bc):
        raise ValueError(f"grid {shape} ({bc}) is not coarsenable")
    ny, nx = shape
    return (_coarse_n(ny, bc), _coarse_n(nx, bc))


def coarse_k(k: np.ndarray, bc: str) -> np.ndarray:
    """Wavenumber on the coarse grid = value at the coincident fine node (re-discretisation, §5.1)."""
    o = unknown_offset(bc)
    nyc, nxc = coarse_shape(k.shape, bc)
    return np.ascontiguousarray(k[o::2, o::2][:nyc, :nxc])


def restrict_fw(v: np.ndarray, bc: str) -> np.ndarray:
    """Full weighting I_h^{2h} (Eq. 3.8): gather of the 9 fine taps around fine node (2I+o, 2J+o)."""
    o = unknown_offset(bc)
    ny, nx = v.shape
    nyc, nxc = coarse_shape(v.shape, bc)
    vp = np.zeros((ny + 2, nx + 2), dtype=np.complex128)
    vp[1:-1, 1:-1] = v
    out = np.zeros((nyc, nxc), dtype=np.complex128)
    for b in (-1, 0, 1):
        for a in (-1, 0, 1):
            r0 = o + 1 + b
            c0 = o + 1 + a
            out += FW[b + 1, a + 1] * vp[r0:r0 + 2 * nyc:2, c0:c0 + 2 * nxc:2]
    return out


def restrict_bilinear_zt(v: np.ndarray, bc: str) -> np.ndarray:
    """Z^T for the bilinear deflation vectors: PAPER.md Eq. 3.7, I_h^{2h} u_i =
    (1/2)(u_{2i-1} + 2 u_{2i} + u_{2i+1}), applied in both directions, i.e. the 9 taps
    (1/4, 1/2, 1/4) (x) (1/4, 1/2, 1/4) x 4 = [1 2 1; 2 4 2; 1 2 1]/4 around fine node (2I+o, 2J+o).
    It is the exact transpose of prolong_bilinear (taps outside the array dropped, R4) and 4x the
    full weighting of Eq. 3.8 that the CSLP V-cycle uses (reading R10)."""
    o = unknown_offset(bc)
    ny, nx = v.shape
    nyc, nxc = coarse_shape(v.shape, bc)
    vp = np.zeros((ny + 2, nx + 2), dtype=np.complex128)
    vp[1:-1, 1:-1] = v
    out = np.zeros((nyc, nxc), dtype=np.complex128)
    w1 = {-1: 0.5, 0: 1.0, 1: 0.5}
    for b in (-1, 0, 1):
        for a in (-1, 0, 1):
            r0 = o + 1 + b
            c0 = o + 1 + a
            out += (w1[a] * w1[b]) * vp[r0:r0 + 2 * nyc:2, c0:c0 + 2 * nxc:2]
    return out


def prolong_bilinear(e: np.ndarray, fine_shape, bc: str) -> np.ndarray:
    """Bilinear interpolation I_{2h}^h (Eq. 3.9 / Eq. 3.6 in each direction): coincident
    fine nodes copy, edge midpoints average 2 coarse values, cell centres average 4."""
    o = unknown_offset(bc)
    ny, nx = fine_shape
    nyc, nxc = coarse_shape(fine_shape, bc)
    if e.shape != (nyc, nxc):
        raise ValueError("coarse/fine shape mismatch")
    w = {-1: 0.5, 0: 1.0, 1: 0.5}
    fp = np.zeros((ny + 2, nx + 2), dtype=np.complex128)
    for b in (-1, 0, 1):
        for a in (-1, 0, 1):
            r0 = o + 1 + b
            c0 = o + 1 + a
            fp[r0:r0 + 2 * nyc:2, c0:c0 + 2 * nxc:2] += w[a] * w[b] * e
    return fp[1:-1, 1:-1].copy()


# ---------------------------------------------------------------------------------------
# Higher-order deflation vectors (APD, Dwarka & Vuik): PAPER.md Eq. 3.11a/b (1D), Eq. 3.12
# (2D matrix-free prolongation, four point classes), Eq. 3.13 (stencil
# 1/64 [1 4 6 4 1] (x) [1 4 6 4 1]), Eq. 3.14/3.15 (restriction with the same stencil).
# The restriction's weights sum to 4 (= 256/64): it is exactly Z_ho^T (not Z^T/4).
# Reading R4 applies: taps outside the unknown array are dropped.
# ---------------------------------------------------------------------------------------
def _ho_weights_1d(d):
    """Weight of coarse node c at fine node 2c + d (Eq. 3.11a read as a column of Z)."""
    return {0: 6.0 / 8.0, 1: 0.5, -1: 0.5, 2: 1.0 / 8.0, -2: 1.0 / 8.0}.get(d, 0.0)


def prolong_high_order(e: np.ndarray, fine_shape, bc: str) -> np.ndarray:
    """Eq. 3.12: coincident fine nodes get (1/64)(36 c + 6 (edge nbrs) + 1 (corner nbrs)),
    x-midpoints (1/16)(6,6 / 1,1 / 1,1), y-midpoints likewise, cell centres (1/4) x 4 —
    i.e. the tensor product of Eq. 3.11a, applied here as a scatter of the 1/64-stencil."""
    o = unknown_offset(bc)
    ny, nx = fine_shape
    nyc, nxc = coarse_shape(fine_shape, bc)
    fp = np.zeros((ny + 4, nx + 4), dtype=np.complex128)
    for b in range(-2, 3):
        for a in range(-2, 3):
            r0 = o + 2 + b
            c0 = o + 2 + a
            fp[r0:r0 + 2 * nyc:2, c0:c0 + 2 * nxc:2] += _ho_weights_1d(a) * _ho_weights_1d(b) * e
    return fp[2:-2, 2:-2].copy()


def restrict_high_order(v: np.ndarray, bc: str) -> np.ndarray:
    """Eq. 3.14: 25-tap gather (1/64)[1 4 6 4 1] (x) [1 4 6 4 1] around fine node (2I+o, 2J+o)."""
    o = unknown_offset(bc)
    ny, nx = v.shape
    nyc, nxc = coarse_shape(v.shape, bc)
    w1 = {-2: 1.0, -1: 4.0, 0: 6.0, 1: 4.0, 2: 1.0}
    vp = np.zeros((ny + 4, nx + 4), dtype=np.complex128)
    vp[2:-2, 2:-2] = v
    out = np.zeros((nyc, nxc), dtype=np.complex128)
    for b in range(-2, 3):
        for a in range(-2, 3):
            r0 = o + 2 + b
            c0 = o + 2 + a
            out += (w1[a] * w1[b] / 64.0) * vp[r0:r0 + 2 * nyc:2, c0:c0 + 2 * nxc:2]
    return out
