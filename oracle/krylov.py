"""ORACLE (test infrastructure only) — flexible GMRES (right preconditioning).

PAPER.md §3.3 Algorithm 1 (Arnoldi with modified Gram-Schmidt: "h_{i,j} = (w, v_i);
w := w - h_{i,j} v_i; h_{j+1,j} := ||w||; v_{j+1} = w / h_{j+1,j}", then "minimize over
||beta e_1 - H_k y||") in its flexible form (§6.3 "Flexible GMRES algorithm, which also
allows for variable preconditioning"): the preconditioned vectors z_j = P v_j are stored
and the solution is u_k = u_0 + Z_k y_k.  The least-squares problem is solved with
complex Givens rotations; |g_{j+1}| is the residual norm ||b - A u_j||.

Inner product (w, v) = sum conj(v) w (np.vdot(v, w)).

Reading R13: Algorithm 1 writes the modified Gram-Schmidt loop.  The
default here is classical Gram-Schmidt applied twice (CGS2): the same projection in exact
arithmetic, and the form the GPU path uses (batched dot products).  With a loose,
tolerance-stopped inner solve the integer inner iteration counts are decided by rounding
(tests show MGS and CGS2 differ there), so both sides use CGS2; orth="mgs" keeps the
literal Algorithm-1 loop, and a pin checks that the two agree when the decisions are not
rounding-sensitive.

Restarts (reading R25): Algorithm 1 is written for a full Krylov basis ("for
j = 1, ..., m" followed by "if not converged, restart with u_0 = u_m" is the textbook GMRES(m)
of Saad & Schultz 1986 that Algorithm 1's "m" denotes).  `restart = m > 0` runs FGMRES(m):
cycles of at most m Arnoldi steps, each started from the current iterate with r = b - A x and
v_1 = r/||r||, the iterate updated x := x + Z_m y_m at the end of every cycle.  The stopping
test stays ||r||/||b|| <= tol against the ORIGINAL ||b||, and `maxit` counts iterations over
all cycles.  restart = 0 (or >= maxit) is the full method.
"""
from __future__ import annotations

import numpy as np


def fgmres(apply_A, apply_P, b: np.ndarray, tol: float, maxit: int, x0=None, history=None, orth="cgs2",
           restart: int = 0):
    """Solve A x = b.  Returns (x, iterations, converged).  restart = m > 0: FGMRES(m) (R25)."""
    if restart and restart < maxit:
        return _fgmres_restarted(apply_A, apply_P, b, tol, maxit, restart, x0, history, orth)
    return _fgmres_cycle(apply_A, apply_P, b, tol, maxit, x0, history, orth, np.linalg.norm(b.ravel()))


def _fgmres_restarted(apply_A, apply_P, b, tol, maxit, m, x0, history, orth):
    """FGMRES(m): cycles of <= m steps from the current iterate, tol against the original ||b||."""
    bnorm = np.linalg.norm(b.ravel())
    x = x0
    its_total = 0
    while True:
        x, its, conv = _fgmres_cycle(apply_A, apply_P, b, tol, min(m, maxit - its_total), x, history, orth, bnorm,
                                     first=its_total == 0)
        its_total += its
        if conv or its == 0 or its_total >= maxit:
            return x, its_total, conv


def _fgmres_cycle(apply_A, apply_P, b, tol, maxit, x0, history, orth, bnorm, first=True):
    """One FGMRES cycle of at most maxit steps from x0 (None = 0); relres against bnorm."""
    shape = b.shape
    bvec = b.ravel()
    x = np.zeros_like(bvec) if x0 is None else x0.ravel().astype(np.complex128).copy()
    if bnorm == 0.0:
        return x.reshape(shape), 0, True
    r = bvec - apply_A(x.reshape(shape)).ravel() if x0 is not None else bvec.copy()
    beta = np.linalg.norm(r)
    if history is not None and first:
        history.append(beta / bnorm)
    if beta / bnorm <= tol:
        return x.reshape(shape), 0, True
    V = [r / beta]
    Z = []
    H = np.zeros((maxit + 1, maxit), dtype=np.complex128)
    cs = np.zeros(maxit)
    sn = np.zeros(maxit, dtype=np.complex128)
    g = np.zeros(maxit + 1, dtype=np.complex128)
    g[0] = beta
    its = 0
    converged = False
    for j in range(maxit):
        z = apply_P(V[j].reshape(shape)).ravel()
        Z.append(z)
        w = apply_A(z.reshape(shape)).ravel()
        if orth == "mgs":
            for i in range(j + 1):                     # modified Gram-Schmidt (Algorithm 1)
                H[i, j] = np.vdot(V[i], w)
                w = w - H[i, j] * V[i]
        else:
            for _ in range(2):                         # classical Gram-Schmidt, twice (CGS2)
                hp = np.array([np.vdot(V[i], w) for i in range(j + 1)])
                for i in range(j + 1):
                    w = w - hp[i] * V[i]
                H[:j + 1, j] += hp
        H[j + 1, j] = np.linalg.norm(w)
        for i in range(j):                             # previous rotations
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -np.conj(sn[i]) * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        a, bb = H[j, j], H[j + 1, j]
        den = np.sqrt(abs(a) ** 2 + abs(bb) ** 2)
        if abs(a) == 0.0:
            cs[j], sn[j] = 0.0, 1.0
        else:
            cs[j] = abs(a) / den
            sn[j] = (a / abs(a)) * np.conj(bb) / den
        H[j, j] = cs[j] * a + sn[j] * bb
        H[j + 1, j] = 0.0
        g[j + 1] = -np.conj(sn[j]) * g[j]
        g[j] = cs[j] * g[j]
        its = j + 1
        res = abs(g[j + 1]) / bnorm
        if history is not None:
            history.append(res)
        if res <= tol:
            converged = True
            break
        hn = np.real(bb)
        if hn == 0.0:                                   # happy breakdown
            converged = True
            break
        V.append(w / hn)
    m = its
    y = np.zeros(m, dtype=np.complex128)
    for i in range(m - 1, -1, -1):                     # back substitution
        y[i] = (g[i] - np.dot(H[i, i + 1:m], y[i + 1:m])) / H[i, i]
    for i in range(m):
        x = x + y[i] * Z[i]
    return x.reshape(shape), its, converged


def gmres_left(apply_A, apply_P, b: np.ndarray, tol: float, maxit: int, x0=None, history=None):
    """Algorithm 1 as printed (§3.3): LEFT-preconditioned GMRES with modified
    Gram-Schmidt, "r_0 = P(b - A u_0), v_1 = r_0/||r_0||; for j: v~_j = A v_j, w := P v~_j;
    for i <= j: h_ij = (w, v_i), w := w - h_ij v_i; h_{j+1,j} = ||w||, v_{j+1} = w/h_{j+1,j}",
    then "minimize ||beta e_1 - H_k y||" and u_k = u_0 + V_k y_k.  The convergence test is on
    the PRECONDITIONED relative residual ||P r_k|| / ||P r_0|| ("the residual vectors
    computed by left preconditioning ... correspond to the preconditioned ... residuals"; :1065
    "we employ left preconditioning and use the preconditioned relative residual as the
    criterion for convergence").  P must be a fixed operator (an exact coarse solve or a fixed
    coarse step count).  The least-squares problem is solved directly (numpy lstsq) every step.
    Returns (x, iterations, converged)."""
    shape = b.shape
    bvec = b.ravel()
    x = np.zeros_like(bvec) if x0 is None else x0.ravel().astype(np.complex128).copy()
    r = bvec - apply_A(x.reshape(shape)).ravel()
    r0 = apply_P(r.reshape(shape)).ravel()
    beta = np.linalg.norm(r0)
    if history is not None:
        history.append(1.0)
    if beta == 0.0:
        return x.reshape(shape), 0, True
    V = [r0 / beta]
    H = np.zeros((maxit + 1, maxit), dtype=np.complex128)
    y = np.zeros(0, dtype=np.complex128)
    its, converged = 0, False
    for j in range(maxit):
        w = apply_P(apply_A(V[j].reshape(shape))).ravel()
        for i in range(j + 1):                             # modified Gram-Schmidt
            H[i, j] = np.vdot(V[i], w)
            w = w - H[i, j] * V[i]
        H[j + 1, j] = np.linalg.norm(w)
        e1 = np.zeros(j + 2, dtype=np.complex128)
        e1[0] = beta
        y = np.linalg.lstsq(H[:j + 2, :j + 1], e1, rcond=None)[0]
        res = np.linalg.norm(H[:j + 2, :j + 1] @ y - e1) / beta
        its = j + 1
        if history is not None:
            history.append(res)
        if res <= tol or H[j + 1, j] == 0.0:
            converged = True
            break
        V.append(w / H[j + 1, j])
    for i in range(its):
        x = x + y[i] * V[i]
    return x.reshape(shape), its, converged


def gcr(apply_A, apply_P, b: np.ndarray, tol: float, maxit: int, history=None):
    """Preconditioned generalised conjugate residual method ("the preconditioned
    Generalized Conjugate Residual method (GCR) [Eisenstat 1983] ... allows for variable
    preconditioning inherently"; §6.3 uses it as the outer method).  From x0 = 0:
        z_k = P r_k,  c_k = A z_k,
        c_k, z_k orthogonalised against c_0..c_{k-1} (classical Gram-Schmidt twice, the same
        coefficients applied to z_k), then scaled by 1/||c_k||,
        beta = (r_k, c_k),  x += beta z_k,  r -= beta c_k,
    until ||r|| / ||b|| <= tol.  Returns (x, iterations, converged)."""
    shape = b.shape
    bvec = b.ravel()
    bnorm = np.linalg.norm(bvec)
    x = np.zeros_like(bvec)
    if bnorm == 0.0:
        return x.reshape(shape), 0, True
    r = bvec.copy()
    if history is not None:
        history.append(1.0)
    C, Zs = [], []
    its, conv = 0, False
    for k in range(maxit):
        z = apply_P(r.reshape(shape)).ravel()
        c = apply_A(z.reshape(shape)).ravel()
        for _ in range(2):                                   # CGS2
            al = np.array([np.vdot(ci, c) for ci in C])
            for i in range(len(C)):
                c = c - al[i] * C[i]
                z = z - al[i] * Zs[i]
        nc = np.linalg.norm(c)
        its = k + 1
        if nc == 0.0:                                        # breakdown: P r in the kernel of A
            break
        c = c / nc
        z = z / nc
        beta = np.vdot(c, r)
        x = x + beta * z
        r = r - beta * c
        C.append(c)
        Zs.append(z)
        res = np.linalg.norm(r) / bnorm
        if history is not None:
            history.append(res)
        if res <= tol:
            conv = True
            break
    return x.reshape(shape), its, conv
