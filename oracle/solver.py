"""ORACLE (test infrastructure only) — A-DEF1 two-level deflation + CSLP, FGMRES outer.

PAPER.md §3.2.2 Eq. 3.21: P_{A-DEF1} = M^{-1}_{h,(beta1,beta2)} P_h + Q_h with
P_h = I - A_h Q_h, Q_h = I_{2h}^h A_{2h}^{-1} I_h^{2h}, Z = I_{2h}^h (bilinear).
§5.2 Eq. 5.3-5.5 give the matrix-free order: v1 = I_h^{2h} v (restriction),
v2 = A_{2h}^{-1} v1 (coarse-grid problem, Eq. 5.6, "by Krylov subspace methods ... CSLP
preconditioned"), v' = I_{2h}^h v2 (interpolation).
§6 preamble: "The (CSLP-preconditioned) GMRES is employed for approximating the inverse of
the coarse-grid operator"; §6.3: with a flexible outer method the coarse tolerance may be
loose (1e-1) while the outer solution still meets 1e-6.

Readings:
  R10 The deflation restriction is Z^T for both kinds of vectors: "Z^T will be the full-weighting
      restriction operator" names the operator, Eq. 3.7 fixes its scale (weights
      1/2, 1, 1/2 per direction, i.e. 4x the 1/16-normalised stencil of Eq. 3.8 that the CSLP
      V-cycle uses).  str-Glk is E = Z^T A Z (Q = Z E^{-1} Z^T is independent of that scale);
      the re-discretised operators replace E as printed (R21), so with them Q carries the
      factor 4 and P_h "is no longer a projection" -- which reproduces the ReD-O2
      counts of Tables 1-2 (the 1/16 scaling would make ReD-O2 as fast as str-Glk).
  R11 The coarse problem E e = c is solved by right-preconditioned FGMRES from e = 0 to the
      relative residual inner_tol, preconditioned by one CSLP V-cycle starting at level 1
      of the CSLP hierarchy (mesh 2h); inner_solver="direct" replaces it by a dense solve.
  R25 inner_restart = m > 0 makes that coarse solve FGMRES(m) (restarted from the current
      iterate every m steps, tolerance against ||c||, inner_maxit over all cycles); restart = m
      does the same for the outer FGMRES (oracle/krylov.py).
  R12 Outer FGMRES from u0 = 0 stops at ||b - A u||/||b|| <= tol (right preconditioning:
      the Arnoldi residual is the true residual).
  R15 inner_tol = 0 runs exactly inner_maxit inner iterations (a fixed polynomial
      preconditioner of E), the rounding-insensitive alternative to the tolerance stop.
  APD (vectors="high_order", §3.2.2 "When the higher-order deflation vector is employed, it
      will be denoted as Adapted Preconditioned Deflation"): Z = Eq. 3.12, Z^T = Eq. 3.14.

TLKM (preconditioner="tlkm"), §3.2.2 (:385-406) and Tables 1-2 (:856-901), in the
paper's practical form: P_TLKM = P~_{h,gamma} M^{-1} with P~_{h,gamma} = (I - A~ Q~) + gamma Q~,
A~ = M^{-1} A, Q~ = I_{2h}^h A~_{2h}^{-1} I_h^{2h}, gamma = 1 (:398), and the coarse matrix of
the practical method I_h^{2h} I_{2h}^h M_{2h}^{-1} A_{2h} (:880) with A_{2h} the configured coarse
operator (ReD-O2 in Tables 1-2) and M_{2h}^{-1} one CSLP V-cycle from level 1 (reading R23); the
coarse problem by unpreconditioned GMRES ("(GMRES)" column of Tables 1-2).  One application:
t = M^{-1} v, e = A~_{2h}^{-1} Z^T t, q = Z e, z = t - M^{-1} A q + gamma q.
"""
from __future__ import annotations

import dataclasses
import time

import numpy as np
import scipy.linalg

from .coarse import apply_coarse_E
from .krylov import fgmres, gcr, gmres_left
from .multigrid import build_hierarchy, vcycle
from .operators import apply_A
from .transfer import coarse_shape, prolong_bilinear, prolong_high_order, restrict_bilinear_zt, restrict_high_order


@dataclasses.dataclass
class SolverParams:
    beta: tuple = (1.0, 0.5)
    omega: float = 0.8
    nu_pre: int = 1
    nu_post: int = 1
    vectors: str = "bilinear"         # bilinear (A-DEF1) | high_order (APD)
    coarse_op: str = "galerkin"       # galerkin | red_o2 | red_o4 | red_o6 | red_cmpo4 | red_9pto2; red_glk1 | red_glk2 (high_order)
    inner_solver: str = "fgmres"      # fgmres | direct
    inner_tol: float = 1e-1           # 0 -> fixed inner_maxit iterations (reading R15)
    inner_maxit: int = 200
    inner_restart: int = 0            # coarse solve FGMRES(m); 0 = full basis (reading R25)
    restart: int = 0                  # outer FGMRES(m); 0 = full basis (reading R25)
    orth: str = "cgs2"                # cgs2 | mgs (reading R13)
    tol: float = 1e-6
    maxit: int = 600
    max_levels: int = 64
    coarsest_n: int = 0               # stop coarsening at the first level with <= coarsest_n unknowns (R7)
    outer: str = "fgmres"             # fgmres | gcr (§6.3) | gmres_left (Algorithm 1 as printed, reading R26)
    preconditioner: str = "adef1"     # adef1 (A-DEF1 / APD) | tlkm (practical TLKM, §3.2.2)
    gamma: float = 1.0                # TLKM shift


class Solver:
    def __init__(self, k, h, bc, params: SolverParams | None = None):
        self.k = np.asarray(k, dtype=np.float64)
        self.h = float(h)
        self.bc = bc
        self.p = params or SolverParams()
        self.levels = build_hierarchy(self.k, self.h, bc, self.p.beta, self.p.max_levels,
                                      coarsest_n=self.p.coarsest_n)
        if len(self.levels) < 2:
            raise ValueError("deflation needs a coarsenable fine grid")
        self.cshape = coarse_shape(self.k.shape, bc)
        self._Edense = None
        self._Elu = None
        self.inner_its = []

    # --- operators --------------------------------------------------------------------
    def A(self, u):
        return apply_A(u, self.k, self.h, self.bc)

    def E(self, x):
        return apply_coarse_E(x, self.k, self.h, self.bc, self.p.coarse_op, self.p.vectors)

    def Zt(self, v):
        return restrict_bilinear_zt(v, self.bc) if self.p.vectors == "bilinear" else restrict_high_order(v, self.bc)

    def Zp(self, e):
        if self.p.vectors == "bilinear":
            return prolong_bilinear(e, self.k.shape, self.bc)
        return prolong_high_order(e, self.k.shape, self.bc)

    def vcycle(self, f, level=0):
        return vcycle(self.levels, f, level, self.p.omega, self.p.nu_pre, self.p.nu_post)

    def E_dense(self):
        if self._Edense is None:
            n = self.cshape[0] * self.cshape[1]
            Ed = np.zeros((n, n), dtype=np.complex128)
            for c in range(n):
                e = np.zeros(n, dtype=np.complex128)
                e[c] = 1.0
                Ed[:, c] = self.E(e.reshape(self.cshape)).ravel()
            self._Edense = Ed
        return self._Edense

    def coarse_solve(self, c):
        """e ~= E^{-1} c (Eq. 5.6), reading R11."""
        if self.p.inner_solver == "direct":
            if self._Elu is None:
                self._Elu = scipy.linalg.lu_factor(self.E_dense())
            return scipy.linalg.lu_solve(self._Elu, c.ravel()).reshape(self.cshape)
        e, its, _ = fgmres(self.E, lambda v: self.vcycle(v, 1), c, self.p.inner_tol, self.p.inner_maxit,
                           orth=self.p.orth, restart=self.p.inner_restart)
        self.inner_its.append(its)
        return e

    def tlkm_coarse(self, x):
        """Coarse matrix of the practical TLKM: I_h^{2h} I_{2h}^h M_{2h}^{-1} A_{2h} x."""
        return self.Zt(self.Zp(self.vcycle(self.E(x), 1)))

    def tlkm(self, v):
        """P_TLKM v = P~_{h,gamma} M^{-1} v (Eq. 3.17-3.18, practical form, reading R23)."""
        t = self.vcycle(v, 0)
        c = self.Zt(t)
        if self.p.inner_solver == "direct":
            n = self.cshape[0] * self.cshape[1]
            Td = np.zeros((n, n), dtype=np.complex128)
            for col in range(n):
                u = np.zeros(n, dtype=np.complex128)
                u[col] = 1.0
                Td[:, col] = self.tlkm_coarse(u.reshape(self.cshape)).ravel()
            e = np.linalg.solve(Td, c.ravel()).reshape(self.cshape)
        else:
            e, its, _ = fgmres(self.tlkm_coarse, lambda w: w, c, self.p.inner_tol, self.p.inner_maxit,
                               orth=self.p.orth)
            self.inner_its.append(its)
        q = self.Zp(e)
        return t - self.vcycle(self.A(q), 0) + self.p.gamma * q

    def precond(self, v):
        return self.tlkm(v) if self.p.preconditioner == "tlkm" else self.adef1(v)

    def Q(self, v):
        """Q_h v = I_{2h}^h A_{2h}^{-1} I_h^{2h} v (Eq. 5.3-5.5)."""
        v1 = self.Zt(v)
        v2 = self.coarse_solve(v1)
        return self.Zp(v2)

    def adef1(self, v):
        """P_{A-DEF1} v = M^{-1}(v - A Q v) + Q v (Eq. 3.21)."""
        q = self.Q(v)
        t = v - self.A(q)
        return self.vcycle(t, 0) + q

    # --- solve ------------------------------------------------------------------------
    def solve(self, b, history=None):
        self.inner_its = []
        t0 = time.perf_counter()
        if self.p.outer == "gcr":
            x, its, conv = gcr(self.A, self.precond, np.asarray(b, dtype=np.complex128), self.p.tol, self.p.maxit,
                               history=history)
        elif self.p.outer == "gmres_left":
            x, its, conv = gmres_left(self.A, self.precond, np.asarray(b, dtype=np.complex128), self.p.tol,
                                      self.p.maxit, history=history)
        else:
            x, its, conv = fgmres(self.A, self.precond, np.asarray(b, dtype=np.complex128),
                                  self.p.tol, self.p.maxit, history=history, orth=self.p.orth, restart=self.p.restart)
        t1 = time.perf_counter()
        r = np.asarray(b) - self.A(x)
        relres = np.linalg.norm(r) / np.linalg.norm(b) if np.linalg.norm(b) > 0 else 0.0
        return x, {"outer_iterations": its, "converged": conv, "relres": float(relres),
                   "inner_iterations": list(self.inner_its), "seconds": t1 - t0}


def solve(problem, params: SolverParams | None = None, history=None):
    s = Solver(problem.k, problem.h, problem.bc, params)
    return s.solve(problem.b, history)
