"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no stencils, transfers, smoothers or
Krylov steps).  It only builds the problem *inputs* the paper describes:

  * the vertex-centred grid description (§2.1, "Structural vertex-centered
    grids are used ... mesh width in x and y direction are both h"),
  * the wavenumber field k(x,y) = 2*pi*f / c(x,y) (Eq. 2.4),
  * the point-source right-hand side (Eq. 2.10, delta at (x0,y0)),
  * seeded random complex fields for operator parity tests.

Both `oracle/` and the CUDA path consume these arrays; neither imports the other.
"""
from .media import (  # noqa: F401
    Problem,
    mp_problem,
    strip_problem,
    wedge_problem,
    marmousi_like_problem,
    random_field,
    random_k,
    config_problem,
    CONFIG_NAMES,
)
