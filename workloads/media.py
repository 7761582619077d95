"""Problem inputs for the 2D Helmholtz model problems (§2).

Conventions (stated once, used by every consumer):

* Vertex-centred grid with nodes x_i = X0 + i*h, y_j = Y0 + j*h, i = 0..Nx, j = 0..Ny
  (§2.1).  Arrays are indexed ``a[j, i]`` (row = y, column = x, x contiguous),
  following §4 "the grid unknowns are stored as an array based on the grid ordering (i, j)".
* Dirichlet (Eq. 2.2, homogeneous g = 0): the unknowns are the INTERIOR nodes
  only, so an array has shape (Ny-1, Nx-1) and unknown (j, i) sits at node (j+1, i+1).
* First-order Sommerfeld (Eq. 2.3): every node is an unknown, shape (Ny+1, Nx+1).
* The point source delta(x-x0, y-y0) (Eq. 2.10) is discretised as the value
  1/h^2 at the nearest node (unit mass under the nodal quadrature weight h^2); ties snap
  to the lower index.
* k(x,y) = 2*pi*f / c(x,y) (Eq. 2.4), stored per unknown node as float64.

Nothing here implements the discrete operators; see oracle/ (reference) and
paper_2308_06152_b200/ (CUDA) for those.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class Problem:
    name: str
    bc: str                 # "dirichlet" | "sommerfeld"
    h: float
    nx: int                 # unknowns along x
    ny: int                 # unknowns along y
    x0: float               # physical x of unknown column 0
    y0: float               # physical y of unknown row 0
    k: np.ndarray           # (ny, nx) float64 wavenumber at unknown nodes
    b: np.ndarray           # (ny, nx) complex128 right-hand side
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def shape(self):
        return (self.ny, self.nx)

    @property
    def kh_max(self) -> float:
        return float(self.k.max() * self.h)


def _point_source(bc, h, nx, ny, x0, y0, xs, ys):
    b = np.zeros((ny, nx), dtype=np.complex128)
    i = int(math.floor((xs - x0) / h + 0.5 - 1e-12))
    j = int(math.floor((ys - y0) / h + 0.5 - 1e-12))
    i = min(max(i, 0), nx - 1)
    j = min(max(j, 0), ny - 1)
    b[j, i] = 1.0 / (h * h)
    return b, (j, i)


def mp_problem(k: float, n_cells: int, bc: str = "dirichlet", name: str | None = None) -> Problem:
    """Constant-wavenumber model problem MP-2a (Dirichlet) / MP-2b (Sommerfeld) on the
    unit square with a point source at (0.5, 0.5) (§2.2, Eq. 2.10).

    ``n_cells`` = 1/h; the paper's "Grid size (n_cells+1) x (n_cells+1)" counts nodes
    including the boundary (Table 1: "33 x 33, k=20, kh=0.625" <=> h = 1/32).
    """
    if n_cells % 2:
        raise ValueError("n_cells must be even so the source sits on the centre node")
    h = 1.0 / n_cells
    if bc == "dirichlet":
        nx = ny = n_cells - 1
        x0 = y0 = h
    elif bc == "sommerfeld":
        nx = ny = n_cells + 1
        x0 = y0 = 0.0
    else:
        raise ValueError(bc)
    kk = np.full((ny, nx), float(k))
    b, src = _point_source(bc, h, nx, ny, x0, y0, 0.5, 0.5)
    return Problem(name or f"mp_{bc}_k{k:g}_n{n_cells}", bc, h, nx, ny, x0, y0, kk, b,
                   {"k": float(k), "n_cells": n_cells, "source": src})


def strip_problem(k: float, n_cells: int, strips: int, name: str | None = None) -> Problem:
    """Weak-scaling family of the Dirichlet model problem (BASELINE configs[4], row-strip
    decomposition): the domain (0,1) x (0,strips) at the same h = 1/n_cells and k, i.e.
    `strips` unit squares stacked in y -- one per GPU -- with the point source at the centre
    (0.5, strips/2).  strips = 1 is mp_problem(k, n_cells)."""
    if n_cells % 2:
        raise ValueError("n_cells must be even")
    h = 1.0 / n_cells
    nx, ny = n_cells - 1, strips * n_cells - 1
    kk = np.full((ny, nx), float(k))
    b, src = _point_source("dirichlet", h, nx, ny, h, h, 0.5, 0.5 * strips)
    return Problem(name or f"strip{strips}_k{k:g}_n{n_cells}", "dirichlet", h, nx, ny, h, h, kk, b,
                   {"k": float(k), "n_cells": n_cells, "strips": strips, "source": src})


# --------------------------------------------------------------------------------------
# Wedge (§2.3, Eq. 2.14): Omega = (0,600) x (-1000,0), three layers with
# velocities 2000 / 1500 / 3000 m/s top to bottom separated by two sloping straight
# interfaces; source at (300, 0); Sommerfeld on all sides.  The interface geometry is
# NOT machine-readable from the paper's Figure 1; this recipe is ours:
#   interface 1: depth 400 m at x=0  -> 200 m at x=600
#   interface 2: depth 600 m at x=0  -> 700 m at x=600
# A node exactly on an interface takes the upper layer's velocity.
# --------------------------------------------------------------------------------------
WEDGE_GRIDS = {10.0: (73, 121), 20.0: (145, 241), 40.0: (289, 481)}


def wedge_velocity(x, depth):
    z1 = 400.0 - x / 3.0
    z2 = 600.0 + x / 6.0
    c = np.where(depth <= z1, 2000.0, np.where(depth <= z2, 1500.0, 3000.0))
    return c


def wedge_problem(f: float, nodes: tuple[int, int] | None = None) -> Problem:
    Nx1, Ny1 = nodes if nodes is not None else WEDGE_GRIDS[float(f)]
    h = 600.0 / (Nx1 - 1)
    if abs(1000.0 / (Ny1 - 1) - h) > 1e-9 * h:
        raise ValueError("anisotropic spacing")
    x = np.arange(Nx1) * h
    y = -1000.0 + np.arange(Ny1) * h
    X, Y = np.meshgrid(x, y)
    c = wedge_velocity(X, -Y)
    k = 2.0 * math.pi * f / c
    b, src = _point_source("sommerfeld", h, Nx1, Ny1, 0.0, -1000.0, 300.0, 0.0)
    return Problem(f"wedge_f{f:g}_{Nx1}x{Ny1}", "sommerfeld", h, Nx1, Ny1, 0.0, -1000.0,
                   k, b, {"f": float(f), "source": src})


# --------------------------------------------------------------------------------------
# Marmousi-shaped synthetic medium (§2.4 describes the real model: 9200 x 3000 m,
# "158 horizontal layers", highly heterogeneous).  The real data set is not available;
# this seeded generator produces a model of the same character:
#   ~150 dipping piecewise-smooth layers, velocity rising with depth 1500 -> 5500 m/s,
#   N(0, 150 m/s) per-layer jitter, ~10 random normal faults offsetting the layers.
# Domain 9192 m wide; the depth extent is (Ny-1)*h with h = 9192/(Nx-1) so spacing is
# isotropic (2945 x 929 nodes -> 9192 x 2897.5 m).
# --------------------------------------------------------------------------------------
MARMOUSI_GRIDS = [(2945, 929), (5889, 1857)]


def marmousi_velocity(X, D, width, depth, seed=2308):
    rng = np.random.default_rng(seed)
    n_layers = 150
    # layer top depths at x=0 and a per-layer dip (m per m), smooth undulation
    tops = np.sort(rng.uniform(0.0, depth, n_layers - 1))
    dips = rng.normal(0.08, 0.03, n_layers - 1)
    amp = rng.uniform(0.0, 30.0, n_layers - 1)
    wav = rng.uniform(800.0, 3000.0, n_layers - 1)
    phs = rng.uniform(0.0, 2 * math.pi, n_layers - 1)
    base = 1500.0 + 4000.0 * (np.arange(n_layers) / (n_layers - 1)) ** 1.3
    vel = np.clip(base + rng.normal(0.0, 150.0, n_layers), 1500.0, 5500.0)
    vel[0] = 1500.0
    # ~10 normal faults: dipping lines x = xf + (d) * tan(theta); hanging wall (x > line)
    # is displaced downward by `throw`.
    n_faults = 10
    xf = rng.uniform(0.1 * width, 0.9 * width, n_faults)
    tanth = rng.uniform(0.3, 0.9, n_faults) * rng.choice([-1.0, 1.0], n_faults)
    throw = rng.uniform(20.0, 150.0, n_faults)
    Deff = D.copy()
    for q in range(n_faults):
        hanging = X > xf[q] + D * tanth[q]
        Deff = np.where(hanging, Deff - throw[q], Deff)
    layer = np.zeros(X.shape, dtype=np.int64)
    for l in range(n_layers - 1):
        zb = tops[l] + dips[l] * (X - 0.5 * width) * 0.3 + amp[l] * np.sin(2 * math.pi * X / wav[l] + phs[l])
        layer += (Deff > zb).astype(np.int64)
    return vel[layer]


def marmousi_like_problem(f: float, nodes: tuple[int, int] = (2945, 929), seed: int = 2308) -> Problem:
    Nx1, Ny1 = nodes
    width = 9192.0
    h = width / (Nx1 - 1)
    depth = (Ny1 - 1) * h
    x = np.arange(Nx1) * h
    y = -depth + np.arange(Ny1) * h
    X, Y = np.meshgrid(x, y)
    c = marmousi_velocity(X, -Y, width, depth, seed)
    k = 2.0 * math.pi * f / c
    b, src = _point_source("sommerfeld", h, Nx1, Ny1, 0.0, -depth, width / 2.0, 0.0)
    return Problem(f"marmousi_like_f{f:g}_{Nx1}x{Ny1}", "sommerfeld", h, Nx1, Ny1, 0.0, -depth,
                   k, b, {"f": float(f), "source": src, "seed": seed})


# --------------------------------------------------------------------------------------
# Seeded random inputs for operator parity (not a workload of the paper; plain test data)
# --------------------------------------------------------------------------------------
def random_field(shape, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def random_k(shape, seed: int, kmin: float = 10.0, kmax: float = 40.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.uniform(kmin, kmax, shape)


# --------------------------------------------------------------------------------------
# BASELINE.json configs -> named problems
# --------------------------------------------------------------------------------------
CONFIG_NAMES = [
    "c0_tiny",                       # configs[0]
    "c1_k50", "c1_k100", "c1_k200", "c1_k400",   # configs[1] (kh = 0.625)
    "c2_wedge_f10", "c2_wedge_f20", "c2_wedge_f40",   # configs[2]
    "c3_marm_f10_2945", "c3_marm_f20_2945", "c3_marm_f40_2945",
    "c3_marm_f10_5889", "c3_marm_f20_5889", "c3_marm_f40_5889",   # configs[3]
    "c4_weak_2049", "c4_strong_8193", "c4_micro_16385",           # configs[4]
]


def config_problem(name: str) -> Problem:
    if name == "c0_tiny":
        return mp_problem(20.0, 32, "dirichlet", name)
    if name.startswith("c1_k"):
        k = float(name[4:])
        return mp_problem(k, int(round(k / 0.625)), "dirichlet", name)
    if name.startswith("c2_wedge_f"):
        return wedge_problem(float(name[len("c2_wedge_f"):]))
    if name.startswith("c3_marm_f"):
        f, n = name[len("c3_marm_f"):].split("_")
        nodes = (2945, 929) if n == "2945" else (5889, 1857)
        return marmousi_like_problem(float(f), nodes)
    if name == "c4_weak_2049":
        return mp_problem(0.625 * 2048, 2048, "dirichlet", name)
    if name == "c4_strong_8193":
        return mp_problem(1000.0, 8192, "dirichlet", name)
    if name == "c4_micro_16385":
        return mp_problem(0.625 * 16384, 16384, "dirichlet", name)
    raise KeyError(name)
