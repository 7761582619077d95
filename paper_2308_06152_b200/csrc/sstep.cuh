// s-step form of the coarse solve's restarted GMRES (reading R28, §6d).
//
// The coarse problem E e = c is solved by CSLP(V-cycle)-preconditioned FGMRES(m) (PAPER.md:795
// §6 / :1065-1071 §6.3; readings R11, R25).  Inside one coarse solve the preconditioner -- one
// V-cycle from level 1 -- is a fixed linear operator M^{-1}, so the flexible method's iterates are
// those of right-preconditioned GMRES(m) on A = E M^{-1}: the same Krylov spaces K_j(A, r0), the
// same minimal-residual iterate after every step, e = e0 + M^{-1} Q y.  This file computes exactly
// those iterates with the Krylov basis generated s vectors at a time (s-step / communication-
// avoiding GMRES, Hoemmen 2010; Chronopoulos-Gear 1989):
//
//   powers : w_0 = q_J, w_i = sigma w_{i-1} - A w_{i-1}  (i = 1..s; one V-cycle + one E apply each,
//            the E kernel's residual mode y = sigma f - E x with f = w_{i-1})
//            =>  A W_{0..s-1} = W_{0..s} B,  B_ii = sigma, B_{i+1,i} = -1
//   orth   : [Q_{0..J}, W_{1..s}]^H W_{1..s} in ONE sweep over the basis (C = Q^H W and the Gram
//            matrix W^H W), C^H C subtracted (Pythagorean form), Cholesky R, and
//            W <- (W - Q C) R^{-1} in ONE more sweep  (block classical Gram-Schmidt, "BCGS-PIP");
//            optionally repeated once (passes = 2, "BCGS-PIP2")
//   hess   : with W_{0..s} = [Q, Q_new] Rf, the new Hessenberg columns H(:, J..J+s-1) follow from
//            A Q Rp = Q H Rp = [Q Q_new] Rf B  (Rp = Rf without its last row/column):
//            H_new Rbot = Rf B - H_old Rp_top, Rbot upper triangular (s x s)
//   Givens rotations of the new columns, |g_{j+1}| after every single column (the convergence
//   test and the iteration count are per step, as in the one-vector form).
//
// Bytes: the basis is read twice per block of s steps instead of twice per step (the delayed
// CGS2 of krylov.cuh), i.e. 2(J+1)/s + 3 vector transfers per step instead of 2J + 6.
// Reductions are deterministic (fixed chunks, fixed transpose-reduction trees, one warp per
// output in a second stage).
#pragma once
#include "krylov.cuh"
#include "vcycle.cuh"   // cp.async helpers

namespace helm {

constexpr int BG_THREADS = 256;                 // dots / update blocks
constexpr int BG_WARPS = BG_THREADS / 32;

template <int S>
struct BgsNV {   // doubles per dot row (2S, padded to a power of two for the transpose reduction)
  static constexpr int v = (2 * S <= 8) ? 8 : (2 * S <= 16 ? 16 : 32);
};

// Sum over the 32 lanes of NV per-lane values at once: after the transpose reduction lane L holds
// the full sum of value (L % NV).  NV - 1 + log2(32 / NV) shuffles instead of 5 NV.
template <int NV>
__device__ __forceinline__ double transpose_reduce(double (&v)[NV], int lane) {
#pragma unroll
  for (int half = NV / 2; half >= 1; half >>= 1) {
    const bool upper = (lane & half) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = upper ? v[i] : v[i + half];
      const double keep = upper ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  double r = v[0];
#pragma unroll
  for (int o = NV; o < 32; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}

// Pass partials of P = [Q_{0..J}, W]^H W, W = V[J+1 .. J+S]:  part[(c * NV + v) * gridDim.x + bx]
// for rows c in [blockIdx.y * crows, ...) of 0..J+S; v = 2t (real) / 2t+1 (imag) of column t.
// Block bx sums the elements [bx * chunk, (bx + 1) * chunk); each warp takes 32 * EPT elements
// at a time with W in registers and loops over the rows.
template <int S, int EPT>
__global__ void __launch_bounds__(BG_THREADS, 2) k_bgs_dots(const double2* __restrict__ V, long long ld,
                                                            const int* __restrict__ jptr, long long n, long long chunk,
                                                            int crows, double* __restrict__ part) {
  HELM_PDL_ENTRY();
  constexpr int NV = BgsNV<S>::v;
  extern __shared__ double bacc[];   // [BG_WARPS][crows][NV]
  const int J = *jptr;
  const int nrows = J + 1 + S;
  const int r0 = blockIdx.y * crows;
  if (r0 >= nrows) return;
  const int r1 = min(nrows, r0 + crows);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* acc = bacc + (size_t)warp * crows * NV;
  for (int i = lane; i < crows * NV; i += 32) acc[i] = 0.0;
  __syncwarp();
  const long long e0 = blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  const double2 zero = make_double2(0.0, 0.0);
  const double2* __restrict__ W = V + (long long)(J + 1) * ld;
  for (long long base = e0 + (long long)warp * 32 * EPT; base < e1; base += (long long)BG_WARPS * 32 * EPT) {
    double2 w[S][EPT];
    bool ok[EPT];
    long long ee[EPT];
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      ee[i] = base + lane + 32 * i;
      ok[i] = ee[i] < e1;
    }
#pragma unroll
    for (int t = 0; t < S; ++t)
#pragma unroll
      for (int i = 0; i < EPT; ++i) w[t][i] = ok[i] ? ldb<1>(W + (long long)t * ld + ee[i]) : zero;
    // rows of the existing basis
    const int qe = min(r1, J + 1);
    double2 qn[EPT];
    if (r0 < qe) {
#pragma unroll
      for (int i = 0; i < EPT; ++i) qn[i] = ok[i] ? ldb<1>(V + (long long)r0 * ld + ee[i]) : zero;
    }
    for (int c = r0; c < qe; ++c) {
      double2 q[EPT];
#pragma unroll
      for (int i = 0; i < EPT; ++i) q[i] = qn[i];
      if (c + 1 < qe) {   // next row's loads in flight during this row's arithmetic
#pragma unroll
        for (int i = 0; i < EPT; ++i) qn[i] = ok[i] ? ldb<1>(V + (long long)(c + 1) * ld + ee[i]) : zero;
      }
      double v[NV];
#pragma unroll
      for (int t = 0; t < S; ++t) {
        double2 a = zero;
#pragma unroll
        for (int i = 0; i < EPT; ++i) a = cadd(a, cconjmul(q[i], w[t][i]));
        v[2 * t] = a.x;
        v[2 * t + 1] = a.y;
      }
#pragma unroll
      for (int t = 2 * S; t < NV; ++t) v[t] = 0.0;
      const double r = transpose_reduce<NV>(v, lane);
      if (lane < NV) acc[(c - r0) * NV + lane] += r;
    }
    // rows of W itself (the Gram matrix W^H W): registers, no loads
#pragma unroll
    for (int u = 0; u < S; ++u) {
      const int c = J + 1 + u;
      if (c < r0 || c >= r1) continue;
      double v[NV];
#pragma unroll
      for (int t = 0; t < S; ++t) {
        double2 a = zero;
#pragma unroll
        for (int i = 0; i < EPT; ++i) a = cadd(a, cconjmul(w[u][i], w[t][i]));
        v[2 * t] = a.x;
        v[2 * t + 1] = a.y;
      }
#pragma unroll
      for (int t = 2 * S; t < NV; ++t) v[t] = 0.0;
      const double r = transpose_reduce<NV>(v, lane);
      if (lane < NV) acc[(c - r0) * NV + lane] += r;
    }
  }
  __syncthreads();
  const int nout = (r1 - r0) * NV;
  for (int i = threadIdx.x; i < nout; i += BG_THREADS) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < BG_WARPS; ++q) s += bacc[(size_t)q * crows * NV + i];
    part[((long long)r0 * NV + i) * gridDim.x + blockIdx.x] = s;
  }
}

// The pass partials on the CUDA cores from a cp.async shared-memory ring (default; DESIGN.md §6d:
// FP64 DMMA m8n8k4 forms of this sweep -- register fragments, or the same ring filled by cp.async
// or by bulk copies -- measured slower on B200: DMMA issues at ~1 per 40 cycles per SM
// sub-partition, ~14 TFLOP/s).
// Stage = SE elements x (J+1+S) rows (row stride 16 SE + 16 B: consecutive rows start 4 banks apart).
// Thread (rb, eg), rb < RB = ceil(rows / 2), eg < EG = 256 / RB: rows rb and rb + RB, elements
// eg, eg + EG, ... of every stage, all S columns in registers (2 S complex accumulators) for the
// whole kernel; one shared-memory reduction over eg at the end.
constexpr int BS_THREADS = 256;
// ring geometry: NS stages of SE elements (SE a multiple of 8), MINB resident blocks per SM
template <int NS_, int SE_, int MINB_>
struct BgsRing {
  static constexpr int NS = NS_, SE = SE_, MINB = MINB_;
  static constexpr int RS = SE * 16 + 16;   // bytes per staged row
  static size_t smem(int rows, int S) {
    return std::max((size_t)rows * RS * NS, (size_t)2 * BS_THREADS * S * sizeof(double2));
  }
};
template <int S, class RG>
__device__ __forceinline__ void bgs_dots_body(const double2* __restrict__ V, long long ld, int J, long long n,
                                              long long chunk, int rmax, double* __restrict__ part,
                                              unsigned char* ssm) {
  constexpr int NV = BgsNV<S>::v;
  const int nrows = J + 1 + S;
  const int RB = (nrows + 1) / 2, EG = BS_THREADS / RB;
  const int tid = threadIdx.x, rb = tid % RB, eg = tid / RB;
  const bool act = eg < EG;
  const int c0 = rb, c1 = rb + RB;
  const bool ok1 = c1 < nrows;
  constexpr int SE = RG::SE, NS = RG::NS;
  constexpr int RSd = RG::RS / 16;           // row stride in double2 (16 B of padding)
  const long long e0 = blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  const int nst = e1 > e0 ? (int)((e1 - e0 + SE - 1) / SE) : 0;
  const size_t stage_bytes = (size_t)rmax * RG::RS;   // >= nrows * RSd * 16
  auto issue = [&](int st) {
    if (st < nst) {
      const long long es = e0 + (long long)st * SE;
      const int cnt = (int)min((long long)SE, e1 - es);
      double2* base = reinterpret_cast<double2*>(ssm + (st % NS) * stage_bytes);
      for (int i = tid; i < nrows * SE; i += BS_THREADS) {
        const int r = i / SE, el = i % SE;
        const bool ok = el < cnt;
        cpa16(base + (size_t)r * RSd + el, V + (long long)r * ld + (ok ? es + el : 0), ok);
      }
    }
    cpa_commit();
  };
  for (int st = 0; st < NS - 1; ++st) issue(st);
  const double2 zero = make_double2(0.0, 0.0);
  double2 a0[S], a1[S];
#pragma unroll
  for (int t = 0; t < S; ++t) a0[t] = a1[t] = zero;
  for (int st = 0; st < nst; ++st) {
    issue(st + NS - 1);
    cpa_wait<NS - 1>();
    __syncthreads();
    const long long es = e0 + (long long)st * SE;
    const int cnt = (int)min((long long)SE, e1 - es);
    const double2* sb = reinterpret_cast<const double2*>(ssm + (st % NS) * stage_bytes);
    if (act) {
      const double2* q0p = sb + (size_t)c0 * RSd;
      const double2* q1p = sb + (size_t)c1 * RSd;
      const double2* wp = sb + (size_t)(J + 1) * RSd;
      for (int el = eg; el < cnt; el += EG) {
        const double2 q0 = q0p[el];
        const double2 q1 = ok1 ? q1p[el] : zero;
#pragma unroll
        for (int t = 0; t < S; ++t) {
          const double2 w = wp[(size_t)t * RSd + el];
          a0[t] = cadd(a0[t], cconjmul(q0, w));
          a1[t] = cadd(a1[t], cconjmul(q1, w));
        }
      }
    }
    __syncthreads();
  }
  cpa_wait<0>();
  __syncthreads();
  // sum over the element groups: [eg][row][t] in the (now free) stage memory
  double2* red = reinterpret_cast<double2*>(ssm);
  if (act) {
#pragma unroll
    for (int t = 0; t < S; ++t) {
      red[((size_t)eg * nrows + c0) * S + t] = a0[t];
      if (ok1) red[((size_t)eg * nrows + c1) * S + t] = a1[t];
    }
  }
  __syncthreads();
  for (int i = tid; i < nrows * S; i += BS_THREADS) {
    double2 sum = zero;
    for (int g = 0; g < EG; ++g) sum = cadd(sum, red[(size_t)g * nrows * S + i]);
    const int c = i / S, t = i % S;
    part[((long long)c * NV + 2 * t) * gridDim.x + blockIdx.x] = sum.x;
    part[((long long)c * NV + 2 * t + 1) * gridDim.x + blockIdx.x] = sum.y;
  }
}

// Blocks with few rows (J + 1 + S <= RSMALL) stage longer element runs (RGS), so the bytes in
// flight do not shrink with J; the rest RGL.  One kernel, the branch taken on the device-side J.
template <int S, class RGS, class RGL, int RSMALL>
__global__ void __launch_bounds__(BS_THREADS, RGL::MINB) k_bgs_dots_smem(const double2* __restrict__ V, long long ld,
                                                                  const int* __restrict__ jptr, long long n,
                                                                  long long chunk, int rmax, double* __restrict__ part) {
  HELM_PDL_ENTRY();
  extern __shared__ __align__(128) unsigned char ssm[];
  const int J = *jptr;
  if (J + 1 + S <= RSMALL) bgs_dots_body<S, RGS>(V, ld, J, n, chunk, RSMALL, part, ssm);
  else bgs_dots_body<S, RGL>(V, ld, J, n, chunk, rmax, part, ssm);
}

// Upper-triangular helpers on S x S row-major complex matrices (one thread).
// R has a real positive diagonal (a Cholesky factor): divisions become products with 1/R_uu.
template <int S>
__device__ void tri_inverse(const double2* R, double2* Ri) {   // Ri = R^{-1}, both upper
  double id[S];
#pragma unroll
  for (int u = 0; u < S; ++u) id[u] = 1.0 / R[u * S + u].x;
  for (int i = 0; i < S * S; ++i) Ri[i] = make_double2(0.0, 0.0);
#pragma unroll
  for (int t = 0; t < S; ++t) {
    Ri[t * S + t] = make_double2(id[t], 0.0);
#pragma unroll
    for (int u = t - 1; u >= 0; --u) {   // row u of column t: -(sum_{k=u+1..t} R_uk Ri_kt) / R_uu
      double2 s = make_double2(0.0, 0.0);
      for (int k = u + 1; k <= t; ++k) s = cfma(R[u * S + k], Ri[k * S + t], s);
      Ri[u * S + t] = cscale(-id[u], s);
    }
  }
}

// Sum of the pass partials (one warp per output double, fixed order), then in the last block:
// C = P(0..J, :), G = W^H W - C^H C, G = R^H R (Cholesky), R^{-1}; the accumulated factors of
// the block (W = Q Ctot + Q_new Rtot): pass 0 Ctot = C, Rtot = R; pass 1 Ctot += C Rtot,
// Rtot = R Rtot.  A non-positive Cholesky pivot (W numerically dependent on Q) marks st->sbrk.
// phase 3: both parts in one launch (the last block does the dense part); decomposed contexts
// launch phase 1 (sums), sum P over the ranks, then phase 2 (dense part, one block).
template <int S>
__global__ void __launch_bounds__(256) k_bgs_reduce(const double* __restrict__ part, int nparts, FgmState* st, int pass,
                                                    double* __restrict__ P, double2* __restrict__ Cm,
                                                    double2* __restrict__ Ri, double2* __restrict__ Ctot,
                                                    double2* __restrict__ Rtot, unsigned* __restrict__ ticket,
                                                    int phase) {
  HELM_PDL_ENTRY();
  constexpr int NV = BgsNV<S>::v;
  const int J = st->j;
  const int nrows = J + 1 + S;
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nout = (long long)nrows * NV;
  if ((phase & 1) && gw < nout && (gw % NV) < 2 * S) {
    const double* p = part + gw * nparts;
    double s = 0.0;
    for (int b = lane; b < nparts; b += 32) s += p[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) P[gw] = s;
  }
  if (!(phase & 2)) return;
  if (phase == 3 && !last_block(ticket)) return;
  __shared__ double2 G[S * S], R[S * S], Rin[S * S], Rt[S * S];
  __shared__ int brk;
  extern __shared__ double2 rsm[];   // the summed rows, complex: (J+1+S) x S
  for (int i = threadIdx.x; i < nrows * S; i += blockDim.x) {
    const int c = i / S, t = i % S;
    rsm[i] = make_double2(__ldcg(P + (long long)c * NV + 2 * t), __ldcg(P + (long long)c * NV + 2 * t + 1));
  }
  __syncthreads();
  auto Pc = [&](int c, int t) { return rsm[c * S + t]; };
  // G = W^H W - C^H C
  for (int i = threadIdx.x; i < S * S; i += blockDim.x) {
    const int u = i / S, t = i % S;
    double2 g = Pc(J + 1 + u, t);
    for (int c = 0; c <= J; ++c) g = csub(g, cconjmul(Pc(c, u), Pc(c, t)));
    G[i] = g;
  }
  for (int i = threadIdx.x; i < (J + 1) * S; i += blockDim.x) Cm[i] = Pc(i / S, i % S);
  __syncthreads();
  if (threadIdx.x == 0) {
    brk = 0;
    for (int i = 0; i < S * S; ++i) R[i] = make_double2(0.0, 0.0);
    for (int t = 0; t < S; ++t) {
      double d = G[t * S + t].x;
      for (int k = 0; k < t; ++k) d -= R[k * S + t].x * R[k * S + t].x + R[k * S + t].y * R[k * S + t].y;
      if (!(d > 1e-30 * fmax(G[t * S + t].x, 1e-300))) {   // breakdown (or NaN)
        brk = 1;
        d = fmax(G[t * S + t].x, 1e-300);
      }
      const double rtt = sqrt(d), irt = 1.0 / rtt;
      R[t * S + t] = make_double2(rtt, 0.0);
      for (int u = t + 1; u < S; ++u) {
        double2 s = G[t * S + u];
        for (int k = 0; k < t; ++k) s = csub(s, cconjmul(R[k * S + t], R[k * S + u]));
        R[t * S + u] = cscale(irt, s);
      }
    }
    tri_inverse<S>(R, Rin);
    if (brk) st->sbrk = 1;
    st->jblk = J;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < S * S; i += blockDim.x) Ri[i] = Rin[i];
  if (pass == 0) {
    for (int i = threadIdx.x; i < (J + 1) * S; i += blockDim.x) Ctot[i] = Cm[i];
    for (int i = threadIdx.x; i < S * S; i += blockDim.x) Rtot[i] = R[i];
  } else {
    for (int i = threadIdx.x; i < S * S; i += blockDim.x) Rt[i] = Rtot[i];
    __syncthreads();
    for (int i = threadIdx.x; i < (J + 1) * S; i += blockDim.x) {   // Ctot += C Rtot
      const int c = i / S, t = i % S;
      double2 s = Ctot[i];
      for (int u = 0; u <= t; ++u) s = cfma(Cm[c * S + u], Rt[u * S + t], s);
      Ctot[i] = s;
    }
    for (int i = threadIdx.x; i < S * S; i += blockDim.x) {   // Rtot = R Rtot (upper x upper)
      const int u = i / S, t = i % S;
      double2 s = make_double2(0.0, 0.0);
      for (int k = u; k <= t; ++k) s = cfma(R[u * S + k], Rt[k * S + t], s);
      Rtot[i] = s;
    }
  }
}

// New Hessenberg columns J..J+S-1 from the block's factors, their Givens rotations, the residual
// estimate after every column and the loop decision (one block).  H is the rotated (upper
// triangular) matrix the back substitution reads, Hr the raw Hessenberg matrix (column-major,
// ld m + 1).  Rotation k: (x_k, x_k+1) <- (c x_k + s x_k+1, -conj(s) x_k + c x_k+1).
struct BgsHessArgs {
  FgmState* st;
  const double2* Ctot;
  const double2* Rtot;
  const double* sig;
  double2* Hr;
  double2* H;
  double* cs;
  double2* sn;
  double2* g;
  int stage_h;
  cudaGraphConditionalHandle h;
  int use_h;
};

// One 256-thread block; hsm = its dynamic shared memory (sstep_hess_smem bytes):
// X: (J+1+S) x S column-major (ld m + 1 + S) | Ctot | Rtot | sn | cs [| raw H]
template <int S>
__device__ __forceinline__ void bgs_hess_body(const BgsHessArgs& a, double2* hsm) {
  FgmState* st = a.st;
  const double2* __restrict__ Ctot = a.Ctot;
  const double2* __restrict__ Rtot = a.Rtot;
  const double* __restrict__ sig = a.sig;
  double2* __restrict__ Hr = a.Hr;
  double2* __restrict__ H = a.H;
  double* __restrict__ cs = a.cs;
  double2* __restrict__ sn = a.sn;
  double2* __restrict__ g = a.g;
  const int stage_h = a.stage_h, use_h = a.use_h;
  const cudaGraphConditionalHandle h = a.h;
  const int J = st->j, m = st->m;
  const int ldh = m + 1, ldx = m + 1 + S;
  const int nr = J + 1 + S;
  const double sigma = *sig;
  const double2 zero = make_double2(0.0, 0.0);
  double2* sCt = hsm + (size_t)ldx * S;
  double2* sRt = sCt + (size_t)(m + 1) * S;
  double2* ssn = sRt + S * S;
  double* scs = reinterpret_cast<double*>(ssn + m);
  for (int i = threadIdx.x; i < (J + 1) * S; i += blockDim.x) sCt[i] = Ctot[i];
  for (int i = threadIdx.x; i < S * S; i += blockDim.x) sRt[i] = Rtot[i];
  for (int i = threadIdx.x; i < J; i += blockDim.x) {
    ssn[i] = sn[i];
    scs[i] = cs[i];
  }
  // the raw Hessenberg columns 0..J-1 (rows 0..J) when the caller sized the shared memory for them
  double2* sH = reinterpret_cast<double2*>(scs + m + (m & 1));
  const bool stageH = stage_h != 0;
  if (stageH)
    for (int i = threadIdx.x; i < J * (J + 1); i += blockDim.x) {
      const int k = i / (J + 1), r = i % (J + 1);
      sH[i] = Hr[(long long)k * ldh + r];
    }
  __syncthreads();
  Ctot = sCt;
  Rtot = sRt;
  // Rf(r, i), i = 0..S: column 0 = e_J; column i >= 1 = [Ctot(:, i-1); Rtot(:, i-1)]
  auto Rf = [&](int r, int i) -> double2 {
    if (i == 0) return r == J ? make_double2(1.0, 0.0) : zero;
    if (r <= J) return Ctot[r * S + (i - 1)];
    const int u = r - J - 1;
    return u < S ? Rtot[u * S + (i - 1)] : zero;
  };
  double2* X = hsm;
  // lhs = Rf B - [H_old Rp_top; 0]:  (Rf B)(:, i) = sigma Rf(:, i) - Rf(:, i + 1)
  for (int idx = threadIdx.x; idx < nr * S; idx += blockDim.x) {
    const int r = idx % nr, i = idx / nr;
    double2 v = csub(cscale(sigma, Rf(r, i)), Rf(r, i + 1));
    if (i > 0 && r <= J) {
      if (stageH) {
        for (int k = max(0, r - 1); k < J; ++k) v = csub(v, cmul(sH[k * (J + 1) + r], Ctot[k * S + (i - 1)]));
      } else {
#pragma unroll 8
        for (int k = max(0, r - 1); k < J; ++k) v = csub(v, cmul(Hr[(long long)k * ldh + r], Ctot[k * S + (i - 1)]));
      }
    }
    X[i * ldx + r] = v;
  }
  __syncthreads();
  // X Rbot = lhs, Rbot(u, i) = Rf(J + u, i): columns in order
  for (int i = 0; i < S; ++i) {
    const double2 d = Rf(J + i, i);
    for (int r = threadIdx.x; r < nr; r += blockDim.x) {
      double2 v = X[i * ldx + r];
      for (int u = 0; u < i; ++u) v = csub(v, cmul(X[u * ldx + r], Rf(J + u, i)));
      X[i * ldx + r] = cdiv(v, d);
    }
    __syncthreads();
  }
  // raw columns out; old rotations (0..J-1) applied to each new column by its own thread
  for (int idx = threadIdx.x; idx < nr * S; idx += blockDim.x) {
    const int r = idx % nr, i = idx / nr;
    Hr[(long long)(J + i) * ldh + r] = (r <= J + i + 1) ? X[i * ldx + r] : zero;
  }
  __syncthreads();
  if (threadIdx.x < S) {
    const int i = threadIdx.x;
    double2* x = X + i * ldx;
    for (int r = J + i + 2; r < nr; ++r) x[r] = zero;
    for (int k = 0; k < J; ++k) {
      const double c = scs[k];
      const double2 s = ssn[k];
      const double2 a = x[k], b = x[k + 1];
      x[k] = cadd(cscale(c, a), cmul(s, b));
      x[k + 1] = csub(cscale(c, b), cconjmul(s, a));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && st->sbrk) {   // numerically dependent block: stop this solve, keep columns 0..J-1
    st->sbrk = 0;
    st->sbrk_total += 1;
    st->its = st->maxit;
    st->ncols = J;
    st->j = J + S;
    st->done = 1;
    fgm_set_cond(st, h, use_h, 0);
    return;
  }
  if (threadIdx.x == 0) {
    int its = st->its, done = 0, conv = 0, acc = 0;
    double relres = st->relres;
    const double bn = st->bnorm, tol = st->tol;
    const int maxit = st->maxit;
    double2 gcur = g[J];
    for (int i = 0; i < S; ++i) {
      const int col = J + i;
      double2* x = X + i * ldx;
      for (int k = J; k < col; ++k) {   // this block's earlier rotations
        const double c = scs[k];
        const double2 s = ssn[k];
        const double2 a = x[k], b = x[k + 1];
        x[k] = cadd(cscale(c, a), cmul(s, b));
        x[k + 1] = csub(cscale(c, b), cconjmul(s, a));
      }
      const double2 a = x[col], b = x[col + 1];
      const double na = hypot(a.x, a.y), nb = hypot(b.x, b.y);
      const double t = hypot(na, nb);
      double c;
      double2 s;
      if (na == 0.0) {
        c = 0.0;
        s = make_double2(1.0, 0.0);
      } else {
        c = na / t;
        const double2 ph = cscale(1.0 / na, a);   // a / |a|
        s = cscale(1.0 / t, cmul(ph, make_double2(b.x, -b.y)));
      }
      x[col] = cadd(cscale(c, a), cmul(s, b));
      x[col + 1] = zero;
      cs[col] = c;
      sn[col] = s;
      scs[col] = c;
      ssn[col] = s;
      const double2 gc = gcur;
      gcur = make_double2(-(s.x * gc.x + s.y * gc.y), -(s.x * gc.y - s.y * gc.x));   // -conj(s) g_col
      g[col + 1] = gcur;
      g[col] = cscale(c, gc);
      ++its;
      ++acc;
      relres = bn > 0.0 ? hypot(gcur.x, gcur.y) / bn : 0.0;
      if (relres <= tol || nb == 0.0) {
        done = conv = 1;
        break;
      }
      if (its >= maxit) {
        done = 1;
        break;
      }
    }
    // rotated columns out (rows 0..col+1)
    for (int i = 0; i < acc; ++i) {
      const int col = J + i;
      for (int r = 0; r <= col + 1; ++r) H[(long long)col * ldh + r] = X[i * ldx + r];
    }
    st->its = its;
    st->ncols = J + acc;
    st->relres = relres;
    st->conv = conv;
    st->j = J + S;
    st->blocks += 1;
    if (J + S >= m) done = 1;   // basis full: the cycle ends (restart)
    st->done = done;
    fgm_set_cond(st, h, use_h, !done);
  }
}

// W <- (W - Q C) R^{-1} for W = V[J+1 .. J+S], Q = V[0 .. J] (in place: every element's outputs
// depend on that element's inputs only).  One element per thread per step.  Optionally the last
// block runs the Hessenberg step of the block instead (off the critical path).
#ifndef HELM_BGU_MINB
#define HELM_BGU_MINB 2
#endif
#ifndef HELM_BGU_UNROLL
#define HELM_BGU_UNROLL 4
#endif
template <int S>
__global__ void __launch_bounds__(BG_THREADS, HELM_BGU_MINB) k_bgs_update(double2* __restrict__ V, long long ld,
                                                              const int* __restrict__ jptr, long long n,
                                                              const double2* __restrict__ Cm,
                                                              const double2* __restrict__ Ri, int hess,
                                                              BgsHessArgs ha) {
  HELM_PDL_ENTRY();
  extern __shared__ double2 bsm[];   // C: (J+1) x S, then R^{-1}: S x S
  // hess: the last block runs the Hessenberg step of this s-step block (bgs_hess_body: it needs the
  // reduction's factors only) while the others stream the basis; it advances st->j at its end, so
  // jptr then points at the reduction's snapshot st->jblk.  The streaming blocks are all resident.
  const int nsb = hess ? (int)gridDim.x - 1 : (int)gridDim.x;
  if (hess && (int)blockIdx.x == nsb) {
    bgs_hess_body<S>(ha, bsm);
    return;
  }
  const int J = *jptr;
  double2* sC = bsm;
  double2* sR = bsm + (size_t)(J + 1) * S;
  for (int i = threadIdx.x; i < (J + 1) * S; i += blockDim.x) sC[i] = Cm[i];
  for (int i = threadIdx.x; i < S * S; i += blockDim.x) sR[i] = Ri[i];
  __syncthreads();
  double2* __restrict__ W = V + (long long)(J + 1) * ld;
  for (long long e = blockIdx.x * (long long)BG_THREADS + threadIdx.x; e < n; e += (long long)nsb * BG_THREADS) {
    double2 w[S];
#pragma unroll
    for (int t = 0; t < S; ++t) w[t] = W[(long long)t * ld + e];
    int c = 0;
    constexpr int UN = HELM_BGU_UNROLL;
    for (; c + UN <= J + 1; c += UN) {
      double2 q[UN];
#pragma unroll
      for (int k = 0; k < UN; ++k) q[k] = ldb<2>(V + (long long)(c + k) * ld + e);
#pragma unroll
      for (int k = 0; k < UN; ++k)
#pragma unroll
        for (int t = 0; t < S; ++t) {
          const double2 cc = sC[(c + k) * S + t];
          w[t] = cfma(make_double2(-q[k].x, -q[k].y), cc, w[t]);
        }
    }
    for (; c <= J; ++c) {
      const double2 q = ldb<2>(V + (long long)c * ld + e);
#pragma unroll
      for (int t = 0; t < S; ++t) w[t] = cfma(make_double2(-q.x, -q.y), sC[c * S + t], w[t]);
    }
#pragma unroll
    for (int t = S - 1; t >= 0; --t) {   // x_t = sum_{u <= t} w_u Ri_ut  (descending t: in place)
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u <= t; ++u) s = cfma(w[u], sR[u * S + t], s);
      W[(long long)t * ld + e] = s;
    }
  }
}

template <int S>
__global__ void __launch_bounds__(256) k_bgs_hess(BgsHessArgs a) {
  HELM_PDL_ENTRY();
  extern __shared__ double2 hsm[];
  bgs_hess_body<S>(a, hsm);
}

}  // namespace helm
