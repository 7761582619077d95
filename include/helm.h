/*
 * helm.h — C ABI of the B200 (sm_100a) hot path of arXiv:2308.06152:
 * matrix-free two-level deflation (A-DEF1 with bilinear vectors, APD with the higher-order
 * vectors) + CSLP-multigrid preconditioned FGMRES / GCR for the 2D finite-difference Helmholtz
 * equation  -Delta u - k(x,y)^2 u = b  (Eq. 2.1).  The whole solve runs on the device
 * (one CUDA graph; outer and inner Krylov loops are conditional while nodes).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Complex numbers are complex128 stored interleaved (re, im) as two doubles; a "field"
 *    is an array of nx*ny such numbers, row-major a[j*nx + i] with x (i) contiguous, the
 *    (i, j) grid ordering of PAPER.md §4.  Pointers named *_dev are DEVICE pointers
 *    (cudaMalloc / torch CUDA storage) owned by the caller; *_host are host pointers.
 *  - Unknowns: Dirichlet grids hold the interior nodes only (homogeneous data g = 0);
 *    Sommerfeld grids hold every node including the boundary (§2.1).
 *  - Level 0 is the fine grid; level l has mesh width 2^l h (standard vertex-centred
 *    coarsening, §4).  Level 1 is also the deflation coarse grid.
 *  - Operator entry points enqueue on the stream given to helm_setup (NULL = legacy default
 *    stream).  helm_solve / helm_solve_host run on a private stream ordered after that stream
 *    and synchronise before returning (they return scalars in helm_report).
 *  - Return value: 0 on success, a negative HELM_E* code on failure; helm_last_error()
 *    returns a thread-local message.  No entry point falls back to the CPU: if the device
 *    or the kernels are unavailable the call fails.
 *  - A helm_ctx is not thread-safe; use one per host thread / stream.
 */
#ifndef HELM_H
#define HELM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HELM_BC_DIRICHLET 0   /* PAPER.md Eq. 2.2 (homogeneous) */
#define HELM_BC_SOMMERFELD 1  /* PAPER.md Eq. 2.3, ghost elimination Eq. 2.8-2.10 */

#define HELM_COARSE_GALERKIN 0 /* str-Glk E = I_h^{2h} A_h I_{2h}^h applied as Z, A, Z^T fused (§3.2.1, §5.2.1) */
#define HELM_COARSE_RED_O2 1   /* second-order re-discretisation at 2h (§5.2.3) */
#define HELM_COARSE_RED_O4 2   /* fourth-order re-discretisation, Eq. 5.11 (§5.2.3) */
#define HELM_COARSE_RED_GLK1 3 /* ReD-Glk1, Eq. 5.12/5.14, 2nd order on two layers (§5.2.4) */
#define HELM_COARSE_RED_GLK2 4 /* ReD-Glk2, Eq. 5.12/5.14 with ghost points (§5.2.4) */
#define HELM_COARSE_RED_O6 5   /* sixth-order re-discretisation, Eq. 5.10 (§5.2.3) */
#define HELM_COARSE_RED_CMPO4 6 /* compact fourth-order re-discretisation, Eq. 5.19 (§5.2.5) */
#define HELM_COARSE_RED_9PTO2 7 /* nine-point eigenvalue-aligned re-discretisation, Appendix B */
/* The re-discretised operators (RED_O2/O4/O6/CMPO4) replace A_{2h} as printed for either kind of
 * deflation vectors (no factor 4 for the higher-order vectors; reading R21). */

#define HELM_OUTER_FGMRES 0 /* flexible GMRES, Algorithm 1 (flexible form, §6.3) */
#define HELM_OUTER_GCR 1    /* preconditioned GCR, PAPER.md:427 and §6.3 */

#define HELM_PRECOND_ADEF1 0 /* P = M^-1 (I - A Q) + Q, Eq. 3.21 */
#define HELM_PRECOND_TLKM 1  /* P = [(I - A~ Q~) + gamma Q~] M^-1, Eq. 3.15-3.18 (practical form) */

#define HELM_VECTORS_BILINEAR 0   /* A-DEF1: Z = Eq. 3.9, restriction Z^T (Eq. 3.7 per direction) */
#define HELM_VECTORS_HIGH_ORDER 1 /* APD: Z = Eq. 3.12, Z^T = Eq. 3.14 (§3.2.1, §3.2.2) */

#define HELM_OK 0
#define HELM_EINVAL -1   /* invalid argument (shape, parameter, null pointer) */
#define HELM_ECUDA -2    /* CUDA runtime error (no device, launch failure, OOM) */
#define HELM_ESHAPE -3   /* grid not coarsenable / coarsest grid too large */

typedef struct helm_ctx_s* helm_ctx;

/* Grid of unknowns (§2.1): nx*ny unknowns, uniform mesh width h, boundary kind. */
typedef struct {
  int nx, ny;
  double h;
  int bc; /* HELM_BC_* */
} helm_grid;

/* Method parameters (§3.1, §3.2.2, §6).  helm_default_params() fills the
 * configuration of BASELINE.json configs[0]: shift (1, 0.5), omega 0.8, V(1,1),
 * bilinear vectors, Galerkin E, inner CSLP-FGMRES to 1e-1 (cap 200).  inner_tol = 0 runs
 * exactly inner_maxit inner iterations (a fixed polynomial preconditioner of E). */
typedef struct {
  double beta1, beta2; /* CSLP shift M = -Delta - (beta1 + i beta2) k^2 (Eq. 3.1) */
  double omega;        /* damped-Jacobi relaxation (0.8, §3.1) */
  int nu_pre, nu_post; /* smoothing sweeps (1, 1) */
  int coarse_op;       /* HELM_COARSE_* */
  double inner_tol;    /* relative residual of the coarse solve E e = c (§6.3) */
  int inner_maxit;     /* cap on inner FGMRES iterations per coarse solve */
  int max_levels;      /* cap on multigrid levels (>= 2) */
  int restart;         /* outer FGMRES basis size; 0 = no restart (full FGMRES) */
  int max_coarsest;    /* largest coarsest grid (unknowns) solved by the dense inverse */
  int vectors;         /* HELM_VECTORS_*; RED_GLK1/RED_GLK2 need the higher-order vectors,
                          every other coarse_op works with both kinds */
  int graph;           /* 1 (default): helm_solve runs as one CUDA graph whose outer and inner
                          loops are conditional while nodes (no host sync inside a solve);
                          0: the same kernels with host-polled loops */
  int tail_max_n;      /* V-cycle levels with at most this many unknowns (and everything below
                          them) run in one thread-block-cluster kernel whose CTAs hold the
                          levels in distributed shared memory; 0 (default) runs every level with
                          the per-level fused kernels */
  int pdl;             /* 1 (default): launches carry programmatic stream serialization, so a
                          kernel's CTAs are scheduled while its predecessor drains */
  int coarsest_n;      /* coarsening stops at the first level with at most this many unknowns
                          (§4 "predefined coarsest grid size"; 0 = as far as possible) */
  int coop;            /* 1: for vectors up to 4M unknowns each delayed-CGS2 step is one cooperative
                          kernel (grid barriers between its phases) instead of three; measured
                          slower on B200 than the kernel chain, so 0 by default */
  int outer;           /* HELM_OUTER_FGMRES (default) or HELM_OUTER_GCR; the coarse solve is
                          always CSLP-preconditioned FGMRES */
  int col_min_n;       /* V-cycle levels with at least this many unknowns use the column-streaming
                          legs (registers + warp shuffles, no shared memory); smaller levels the
                          tiled legs; -1 disables (default 1 << 20) */
  int dist_levels;     /* decomposed contexts (helm_setup_dist): number of multigrid levels split
                          into row strips (0 = automatic: every level on which each rank owns at
                          least dist_min_rows rows, at most all but the coarsest); the levels below
                          are replicated on every rank.  Must be >= 2 (levels 0 and 1). */
  int dist_min_rows;   /* fewest rows a rank may own on a decomposed level (default 16, >= 6) */
  int col_pipe;        /* column-streaming legs: 0 = rows prefetched in registers; 1 (default) = rows
                          staged through a per-warp cp.async shared-memory ring, 4 rows in flight,
                          segments of 256 (down) / 128 (up) rows; 3, 4, 5, 14, 24: other depths /
                          segment lengths (measurement) */
  int fuse_dots;       /* 1: with str-Glk, the inner FGMRES applies E and pass 1 of the delayed CGS2
                          (the dots against the basis) in one kernel.  Measured slower on B200
                          than the two kernels early in round 1 (0.577 vs 0.568 s per bench
                          solve).  With the final round-1 step (lagged step B, one-wave pass 1)
                          it was 1.4 % faster (0.506 vs 0.513 s).  Round 2: the column-streaming E
                          kernel (e_stream) plus the separate dots kernel is faster still at the
                          configs[4] sizes (E 30 vs 83 us on 1023^2; the fused kernel keeps the
                          tile form), so 0 (default) */
  int precond;         /* HELM_PRECOND_ADEF1 (default; A-DEF1, or APD with the higher-order vectors)
                          or HELM_PRECOND_TLKM (practical two-level Krylov method, §3.2.2
                          and Tables 1-2: coarse matrix Z^T Z M_2h^-1 A_2h solved by unpreconditioned
                          FGMRES; two fine V-cycles per application; single-GPU contexts only) */
  double gamma;        /* TLKM shift (1) */
  int tail_cluster;    /* CTAs of the tail kernel (tail_max_n > 0): 0 = 16, else 8 (default); 1, 2,
                          4, 8 or 16 = exactly that many (1: one CTA, no cluster) */
  int lag_stepb;       /* inner solve (single GPU): the Arnoldi step's loop decision taken one
                          iteration late from the corrected column (the rotation leaves the serial
                          tail of every iteration; a converged inner solve runs one discarded
                          iteration).  Same iteration counts as the immediate test on the corrected
                          column.  1 = on, 0 = off */
  int dots_cluster;    /* inner / outer Arnoldi on one GPU: pass 1 of the delayed CGS2 sums its chunk
                          partials on chip over 8-CTA thread-block clusters (DSMEM) and the update
                          kernel adds the remaining 1/8 itself -- no reduction kernel.  Measured
                          slower on B200 (the cluster pass 1 costs +5-6 us over dots + reduction:
                          DESIGN.md §6b), so 0 (default) = the dots + reduction kernels; 1 = on */
  int inner_restart;   /* coarse solve as FGMRES(m) (reading R25): m > 0 restarts the inner
                          Arnoldi process from the current iterate every m steps (basis of m + 1
                          level-1 vectors, Gram-Schmidt cost O(m) per step), the tolerance stays
                          relative to ||c|| and inner_maxit counts steps over all cycles; 0 (default)
                          or m >= inner_maxit = one full cycle.  A-DEF1/APD only (TLKM: 0) */
  int e_stream;        /* str-Glk E on one GPU (not fused with the dots): 1 (default) = the
                          column-streaming kernel (fine fields in registers, neighbours by warp
                          shuffles; the tile kernel's arithmetic), 0 = the shared-memory
                          tile kernel */
  int tma;             /* column-streaming legs staged by the Tensor Memory Accelerator
                          (cp.async.bulk.tensor: one box of 116 columns x R rows per field and stage,
                          a CTA-wide full/empty mbarrier ring) when the level's fields are plain
                          device arrays; bit 1 = up leg, bit 2 = down leg; otherwise the per-lane
                          cp.async (LDGSTS) ring.  Default 1 (up leg only: measured faster there,
                          slower for the down leg) */
  int sstep;           /* coarse solve in s-step form (reading R28): 0 (default) = one basis
                          vector per step (delayed CGS2); 4, 6 or 8 = the basis generated s vectors
                          at a time (s V-cycles + E applies), orthogonalised as a block (one sweep
                          over the basis for all s dot products, Cholesky of the Pythagorean Gram
                          matrix, one update sweep), Hessenberg columns recovered from the block
                          factors.  The same GMRES(m) iterates in exact arithmetic (the V-cycle is a
                          fixed linear preconditioner within a coarse solve); per-step convergence
                          test and counts.  Decomposed contexts: one rank sum of the block's dot
                          products per s steps (instead of two per step).  A-DEF1/APD, the coarse
                          basis size (inner_restart, else inner_maxit) a multiple of s */
  int sstep_passes;    /* block Gram-Schmidt passes per block: 2 (default, BCGS-PIP2) or 1 */
  double sstep_shift;  /* shift sigma of the block basis w_i = sigma w_{i-1} - A w_{i-1} (default 0.5,
                          the centre of the CSLP-preconditioned spectrum's disc) */
} helm_params;

typedef struct {
  int outer_iterations;   /* FGMRES iterations to reach tol (PAPER.md "#iter") */
  int converged;          /* 1 if ||b - A x|| / ||b|| <= tol by the Arnoldi estimate */
  double relres;          /* final Arnoldi residual estimate / ||b|| */
  int inner_solves;       /* coarse solves performed (one per outer iteration) */
  long long inner_iterations_total;
  int inner_iterations_max;
  int restarts;
  double seconds;         /* host wall time of the solve (stream synchronised) */
  long long kernels;      /* kernels executed by the solve (graph replays counted per node run) */
  long long inner_restarts; /* restart cycles of the coarse solves (params.inner_restart), summed */
} helm_report;

void helm_default_params(helm_params* p);

/* Build the solver: copies k (nx*ny float64 wavenumbers at the unknowns, host or device
 * per k_on_device) to device memory, builds the multigrid hierarchy (coarse k sampled at
 * coincident nodes), the deflation coarse operator and the coarsest dense inverse.
 * `stream` is a cudaStream_t (may be NULL).  The context owns all internal workspace. */
int helm_setup(helm_ctx* out, const helm_grid* grid, const double* k, int k_on_device,
               const helm_params* params, void* stream);
void helm_destroy(helm_ctx ctx);

int helm_num_levels(helm_ctx ctx);
int helm_level_info(helm_ctx ctx, int level, int* nx, int* ny, double* h);

/* y = A_h x on level 0 (Algorithm 2, Eq. 2.7/2.9/2.10).  x, y: device fields. */
int helm_apply_A(helm_ctx ctx, const double* x_dev, double* y_dev);
/* y = M_l x, the CSLP operator of level l (Eq. 3.1, re-discretised on coarse levels). */
int helm_apply_M(helm_ctx ctx, int level, const double* x_dev, double* y_dev);
/* Full-weighting restriction level l -> l+1 (Eq. 3.8) and bilinear prolongation
 * level l+1 -> l (Eq. 3.9); for l = 0 these are Z^T/4 and Z of the deflation. */
int helm_restrict(helm_ctx ctx, int level, const double* fine_dev, double* coarse_dev);
int helm_prolong(helm_ctx ctx, int level, const double* coarse_dev, double* fine_dev);
/* y = E x on level 1, E the configured deflation coarse operator (§5.2). */
int helm_apply_E(helm_ctx ctx, const double* x_dev, double* y_dev);
/* u = one V(nu_pre, nu_post) cycle approximating M_l^{-1} f, starting at level l (§3.1). */
int helm_vcycle(helm_ctx ctx, int level, const double* f_dev, double* u_dev);
/* z = P_{A-DEF1} v = M^{-1}(v - A Q v) + Q v, Q = Z E^{-1} Z^T (Eq. 3.21, Eq. 5.3-5.5),
 * E^{-1} by CSLP-preconditioned FGMRES to inner_tol (writes the inner count to
 * *inner_its if non-NULL); with params.precond = HELM_PRECOND_TLKM the TLKM preconditioner. */
int helm_deflate(helm_ctx ctx, const double* v_dev, double* z_dev, int* inner_its);
/* Solve A x = b by A-DEF1/APD-preconditioned FGMRES (or GCR, params.outer) from x0 = 0 to
 * ||b - A x||/||b|| <= tol
 * (Algorithm 1 flexible form, Eq. 3.21).  The Arnoldi process, the Givens
 * least-squares update and both convergence tests run on the device; the whole solve is one
 * CUDA graph (params.graph = 1).  Orthogonalisation: classical Gram-Schmidt twice with the
 * second pass delayed one iteration (two sweeps over the basis per iteration; R13).  b, x: device fields (x may not
 * alias b).  rep may be NULL. */
int helm_solve(helm_ctx ctx, const double* b_dev, double* x_dev, double tol, int maxit, helm_report* rep);
/* Deflation vectors of the configured kind between level 0 and the coarse grid (level 1):
 * coarse = Z^T fine, fine = Z coarse (reading R10). */
int helm_apply_Zt(helm_ctx ctx, const double* fine_dev, double* coarse_dev);
int helm_apply_Z(helm_ctx ctx, const double* coarse_dev, double* fine_dev);
/* Same with host buffers: H2D copy of b, solve, D2H copy of x (end-to-end path). */
int helm_solve_host(helm_ctx ctx, const double* b_host, double* x_host, double tol, int maxit,
                    helm_report* rep);

/* Read a `bytes`-sized scratch buffer (> L2) on the context stream: L2 flush between timed steps
 * (reads, so the evicted lines are clean and the next kernel pays no write-backs). */
int helm_flush_l2(helm_ctx ctx, size_t bytes);
/* Number of kernels this context launched since creation (bench.py's gpu_launches); a graph
 * solve adds the kernels its replay executed. */
long long helm_launch_count(helm_ctx ctx);

/* Kernel timing for the roofline (bench.py): launches kernel `which` `reps` times on the
 * context stream at this context's sizes (level 0 / level `arg` / level 1 / inner basis), each bracketed by
 * CUDA events (after an L2 flush if `flush`), and returns the mean device time per launch and
 * the algorithmic bytes per launch.  `arg` = number of basis vectors for the
 * Gram-Schmidt kernels (1..inner_maxit).  Operates on internal scratch buffers only. */
#define HELM_KB_APPLY_A 0
#define HELM_KB_VC_DOWN 1    /* fused V-cycle down leg on level `arg` */
#define HELM_KB_VC_UP 2      /* fused V-cycle up leg on level `arg` */
#define HELM_KB_APPLY_E 3
#define HELM_KB_GS_DOTS 4    /* delayed-CGS2 pass 1 over `arg` basis vectors */
#define HELM_KB_GS_UPDATE 5  /* delayed-CGS2 pass 2 over `arg - 1` basis vectors */
int helm_bench_kernel(helm_ctx ctx, int which, int arg, int reps, int flush, double* us_per_launch,
                      double* bytes_per_launch);

/* Warm in-graph cost of a region of the path: `reps` back-to-back instances captured into one
 * CUDA graph (as inside a solve), replayed; returns the mean device time per instance.
 * HELM_GB_VCYCLE: one V-cycle from level `arg`; HELM_GB_APPLY_E: one E apply (level 1);
 * HELM_GB_APPLY_A: one A apply (level 0).  Internal scratch buffers only. */
#define HELM_GB_VCYCLE 0
#define HELM_GB_APPLY_E 1
#define HELM_GB_APPLY_A 2
#define HELM_GB_DCGS 3      /* one Arnoldi step of the inner FGMRES after the V-cycle, as the solve
                               runs it: E apply + pass 1 (fused by default), reduction + step A,
                               pass 2 + step B, from column `arg` (arg + reps < basis size).
                               Probe knobs (environment, this region only): HELM_GB_DCGS_MASK
                               selects its kernels (1 dots, 2 reduction, 4 update; default 7),
                               HELM_GB_UPD_FLAGS overrides the update kernel's flags */
#define HELM_GB_INNER_ITER 4 /* one whole inner FGMRES iteration (V-cycle from level 1, E apply,
                                delayed-CGS2 step) from column `arg`, without the loop node */
/* The kernels of the inner Arnoldi step one at a time, exactly as the solve launches them
 * (HELM_GB_DCGS is their sequence): */
#define HELM_GB_E_DOTS 5      /* w = E z_j with pass 1 of the delayed CGS2 (one fused kernel with
                                 str-Glk and fuse_dots; else the E apply and the dots kernel) */
#define HELM_GB_DCGS_REDUCE 6 /* reduction of the pass-1 partials + step A coefficients */
#define HELM_GB_DCGS_UPDATE 7 /* pass 2 (v_j, w') + step B (advances the column) */
#define HELM_GB_DCGS_DOTS 8   /* pass 1 alone (k_dcgs_dots) as the unfused step launches it */
#define HELM_GB_VC_DOWN 9     /* the fused V-cycle down leg of level `arg`, as the V-cycle launches it */
#define HELM_GB_VC_UP 10      /* the fused V-cycle up leg of level `arg` */
/* s-step coarse solve (params.sstep > 0; `arg` = the block's first column J, a multiple of s): */
#define HELM_GB_SS_DOTS 11    /* the block pass partials [Q_0..J, W]^H W (one sweep over the basis) */
#define HELM_GB_SS_REDUCE 12  /* their reduction + Cholesky of the Pythagorean Gram matrix */
#define HELM_GB_SS_UPDATE 13  /* W <- (W - Q C) R^-1 (one sweep over the basis) */
#define HELM_GB_SS_POWER 14   /* one step of the block basis: V-cycle from level 1 + E in residual mode */
#define HELM_GB_SS_E 15       /* E in residual mode alone, w = sigma f - E x */
#define HELM_GB_OUTER_DCGS 16 /* the outer FGMRES's delayed-CGS2 step at basis column `arg` (pass 1,
                                 reduction + step A, pass 2 + step B over the level-0 basis as the
                                 solve launches them; the operator applies are not included).  Needs
                                 an outer basis of more than arg + reps columns: call after a solve */
int helm_bench_graph(helm_ctx ctx, int which, int arg, int reps, double* us_per_region);

/* ---------------------------------------------------------------------------------------
 * Row-strip domain decomposition over ranks (DESIGN.md §7; §4, :463-469: the
 * (i, j)-ordered grid is distributed over processes by blocks with ghost layers, coarsening
 * stops at a predefined size).  Every rank holds the GLOBAL problem description; level l <= D
 * is split into nranks contiguous row strips (rank q owns global rows [row0, row0 + nrows) of
 * level l, see helm_dist_rows), stored with >= 6 ghost rows that are refreshed from the
 * neighbours before every kernel that reads them; the levels below D are replicated (each rank
 * completes its copy by an all-gather of the owned rows and runs the rest of the V-cycle and
 * the dense coarsest solve itself).  Dots and norms are summed over the ranks; every rank then
 * takes the same scalar steps.  Both outer methods (FGMRES, GCR); loops are host-polled
 * (params.graph is forced to 0).
 *
 * Transports:
 *  HELM_COMM_NCCL    one process per GPU; nccl_id = 128 bytes from helm_nccl_unique_id() on
 *                    rank 0, broadcast by the caller (e.g. torch.distributed); halos are grouped
 *                    ncclSend/ncclRecv, dots ncclAllReduce, the all-gather ncclBroadcast per
 *                    rank.  libnccl.so.2 is loaded at run time (the copy already in the process
 *                    if any, else $HELM_NCCL_LIB, else the default search path).
 *  HELM_COMM_THREADS nranks host threads of ONE process sharing one device (group from
 *                    helm_group_create(nranks)); each thread calls every entry point of its own
 *                    context in the same order.  Exchanges are device copies from the peers'
 *                    buffers ordered by CUDA events and host barriers: no kernel waits on
 *                    another rank, so this is safe on a single GPU.  It exercises the whole
 *                    decomposed path on one B200 (parity tests).
 *  HELM_COMM_PEER    one process per GPU of one NVLink/NVSwitch node, no NCCL: every rank's
 *                    exchange arena (halo rows, rank-sum and all-gather slots, epoch flags) is
 *                    mapped into its peers through CUDA IPC (helm_peer_handle on every rank,
 *                    gather the 64-byte handles, helm_peer_connect); an exchange is a producer
 *                    kernel that writes its slot and publishes an epoch flag and a consumer kernel
 *                    that waits for the peers' flags and reads their slots directly over NVLink
 *                    (peer.cuh).  Needs one GPU per rank (its kernels wait on other ranks');
 *                    waits give up after ~10 s and the solve returns HELM_ECUDA.
 * On a decomposed context helm_apply_A, helm_vcycle (level 0), helm_deflate, helm_solve and
 * helm_solve_host take and return THIS RANK'S OWNED ROWS of level 0 (nrows * nx values,
 * contiguous); the other per-level entry points and the benchmarks return HELM_EINVAL.
 * Errors: setup fails on every rank of a thread group if it fails on one; a rank that fails
 * later leaves its peers waiting (callers of thread groups must abort the process).
 * --------------------------------------------------------------------------------------- */
#define HELM_COMM_THREADS 0
#define HELM_COMM_NCCL 1
#define HELM_COMM_PEER 2
typedef struct helm_group_s* helm_group;
int helm_group_create(int nranks, helm_group* out);
void helm_group_destroy(helm_group g);
int helm_nccl_unique_id(unsigned char id[128]);

typedef struct {
  int kind;                     /* HELM_COMM_* */
  int rank, nranks;             /* 0 <= rank < nranks <= 16 */
  helm_group group;             /* HELM_COMM_THREADS */
  const unsigned char* nccl_id; /* HELM_COMM_NCCL: 128 bytes, identical on every rank */
  int flags;                    /* HELM_DIST_* bits, 0 for production */
} helm_dist;
/* HELM_COMM_PEER with nranks == 1: run the exchange kernels (halo, rank sums, all-gather, the
 * fused peer DCGS kernels) against the rank's own arena instead of skipping them -- a test
 * mode that exercises the peer transport on one GPU.  Without it a single rank exchanges
 * nothing (identical results, fewer launches). */
#define HELM_DIST_EXCHANGE_AT_ONE_RANK 1

/* As helm_setup, on the global grid and the global k (nx*ny, host or device), for rank
 * dist->rank of a decomposed solve.  Collective: every rank must call it. */
int helm_setup_dist(helm_ctx* out, const helm_grid* grid, const double* k, int k_on_device,
                    const helm_params* params, void* stream, const helm_dist* dist);
/* Peer transport: this rank's 64-byte CUDA IPC handle of its exchange arena; then, with the
 * handles of all ranks (nranks * 64 bytes, rank order), map the peers' arenas.  Both collective
 * in the sense that every rank must call them before its first exchange.  helm_peer_error: 1 if
 * a peer wait timed out. */
int helm_peer_handle(helm_ctx ctx, unsigned char out[64]);
int helm_peer_connect(helm_ctx ctx, const unsigned char* handles);
int helm_peer_error(helm_ctx ctx);
/* Host-only: the peer arena layout (bytes, flags, rank-sum slot, all-gather slot and its length,
 * then per decomposed level the up / down halo slots) -- identical on every rank by construction;
 * returns the number of entries (or a negative error). */
int helm_peer_layout(const helm_grid* grid, const helm_params* params, int nranks, size_t* out, int cap);
/* Global rows [*row0, *row0 + *nrows) of `level` owned by this rank (single-GPU context: all). */
int helm_dist_rows(helm_ctx ctx, int level, int* row0, int* nrows);
/* Host-only plan of the decomposition (no device needed): returns the number of levels L
 * (or a negative error), *D = deepest decomposed level, and table[(l * nranks + q) * 4 + i]
 * = {owned row begin, owned row end, stored row begin, stored row end} for l < min(L, cap). */
int helm_dist_plan(const helm_grid* grid, const helm_params* params, int nranks, int* D, int* table,
                   int cap_levels);

const char* helm_last_error(void);
const char* helm_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* HELM_H */
