// Fused multigrid kernels for the CSLP V-cycle (§3.1: one pre-/post- damped-Jacobi
// sweep with omega = 0.8, full-weighting restriction Eq. 3.8, bilinear interpolation Eq. 3.9,
// coarsest-level solve; coarse operators re-discretised, §5.1).
//
// The unfused V-cycle of one level is five grid passes (Jacobi from u = 0, residual,
// restriction, interpolation + correction, post-Jacobi), ~208 B of HBM traffic per fine
// unknown.  Here each level is two tiled kernels:
//   k_vc_down: u = omega f / D ; r = f - M u ; f_c = I_h^{2h} r        (reads f, k; writes u, f_c)
//   k_vc_up:   u1 = u + I_{2h}^h e ; y = u1 + omega (f - M u1) / D (+ q)  (reads u, e, f, k; writes y)
// with the intermediate u / r / u1 tiles (and their halos) kept in shared memory: ~104 B per
// fine unknown and two launches instead of five.  Levels small enough for one SM run the
// whole remaining V-cycle (down to the dense coarsest solve) in a single CTA (k_vc_tail).
// Valid for nu_pre = nu_post = 1 (the paper's setting); other sweep counts use the generic
// kernels of kernels.cuh.
#pragma once
#include <cooperative_groups.h>
#include <cuda.h>

#include "kernels.cuh"

namespace cg = cooperative_groups;

#ifndef HELM_VC_MINB
#define HELM_VC_MINB 4   // 64-register cap: 4 CTAs/SM (c4 level-1 legs -4 us, profiles/r02_legs_probe.jsonl)
#endif
namespace helm {

__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }

__device__ __forceinline__ int floordiv2(int a) { return (a >= 0) ? (a >> 1) : -((-a + 1) >> 1); }

// Stencil apply with the 4 neighbours supplied explicitly (smem tiles).
__device__ __forceinline__ double2 stencil5(const Coef& c, double2 uc, double2 uw, double2 ue, double2 us, double2 un) {
  double2 v = cmul(c.ap, uc);
  if (c.aw != 0.0) v = cadd(v, cscale(c.aw, uw));
  if (c.ae != 0.0) v = cadd(v, cscale(c.ae, ue));
  if (c.as != 0.0) v = cadd(v, cscale(c.as, us));
  if (c.an != 0.0) v = cadd(v, cscale(c.an, un));
  return v;
}

// Interior points (all four neighbours inside the grid, no boundary row) share the multipliers
// aw = ae = as = an = -1/h^2; only the centre depends on k.  A CTA whose whole region is
// interior takes a branch-free path (uniform per CTA: no divergence).
__device__ __forceinline__ double2 interior_ap(double ih2, double kk, double sr, double si) {
  const double k2 = kk * kk;
  return make_double2(4.0 * ih2 - sr * k2, -si * k2);
}

__device__ __forceinline__ double2 interior_stencil(double ih2, double2 ap, double2 uc, double2 uw, double2 ue,
                                                    double2 us, double2 un) {
  // same operation order as stencil5 with nonzero multipliers
  double2 v = cmul(ap, uc);
  v = cadd(v, cscale(-ih2, uw));
  v = cadd(v, cscale(-ih2, ue));
  v = cadd(v, cscale(-ih2, us));
  v = cadd(v, cscale(-ih2, un));
  return v;
}

// ------------------------------------------------------------------ down leg
// CTA = TCX x TCY coarse points, 32 x 8 threads.  Fine footprint of the restriction: fine nodes
// 2I+o-1 .. 2I+o+1; the residual there needs u one node further out.  f (scaled) and k of the
// region are kept in shared memory for the residual phase.
template <int TCX, int TCY>
__global__ void __launch_bounds__(256, HELM_VC_MINB) k_vc_down(Geo F, Geo G, int o, DVec fv, const double* __restrict__ k,
                                                 double sr, double si, double omega, double2* __restrict__ u,
                                                 double2* __restrict__ fc) {
  constexpr int RX = 2 * TCX + 3, RY = 2 * TCY + 3;  // u region
  constexpr int QX = 2 * TCX + 1, QY = 2 * TCY + 1;  // r region
  __shared__ double2 su[RY * RX];
  __shared__ double2 sf[RY * RX];
  __shared__ double sk[RY * RX];
  __shared__ double2 sq[QY * QX];
  const int tx = threadIdx.x, ty = threadIdx.y;
  // f (and its device-side column index / scale) may be written by the kernel launched just
  // before this one: read after the PDL wait
  const double2* __restrict__ f = nullptr;
  double fs = 0.0;
  const int I0 = blockIdx.x * TCX, J0 = blockIdx.y * TCY;
  const int gx0 = 2 * I0 + o - 2, gy0 = 2 * J0 + o - 2;
  // fine points whose pre-smoothed u this CTA owns (a partition of the fine grid)
  const int xs = (I0 == 0) ? 0 : 2 * I0 + o - 1;
  const int xe = (I0 + TCX >= G.nx) ? F.nx : 2 * (I0 + TCX) + o - 1;
  const int ys = (J0 == 0) ? 0 : 2 * J0 + o - 1;
  const int ye = (J0 + TCY >= G.ny) ? F.ny : 2 * (J0 + TCY) + o - 1;
  const bool interior = gx0 >= 1 && gx0 + RX <= F.nx - 1 && gy0 >= 1 && gy0 + RY <= F.ny - 1;
  const double ih2 = 1.0 / (F.h * F.h);
  const int tid = ty * 32 + tx;
  // every global load of the tile is issued before the first use (NT per thread in flight)
#ifndef HELM_VC_DOWN_PRELOAD
#define HELM_VC_DOWN_PRELOAD 1
#endif
  constexpr int NT = HELM_VC_DOWN_PRELOAD ? (RX * RY + 255) / 256 : 1;
  for (int tb0 = 0; tb0 < RX * RY; tb0 += 256 * NT) {
  const int tid = ty * 32 + tx + tb0;
  double2 fl[NT];
  double kl[NT], dl[NT];
  // Small levels (latency-bound): k is set-up data, loaded -- and the reciprocal modulus of the
  // Jacobi diagonal formed -- before the PDL wait (f is the output of the kernel launched just
  // before this one).  Large levels wait first (the extra registers would spill).
  constexpr bool PRE = TCX * TCY <= 32;
  if (!PRE && tb0 == 0) {
    HELM_PDL_ENTRY();
    f = fv.get();
    fs = fv.scale();
  }
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const int t = tid + 256 * i;
    const int iy = t / RX, ix = t - iy * RX;   // compile-time divisor
    const int x = gx0 + ix, y = gy0 + iy;
    const bool in = t < RX * RY && (interior || (x >= 0 && x < F.nx && y >= 0 && y < F.ny));
    const size_t p = in ? (size_t)y * F.nx + x : 0;
    kl[i] = in ? k[p] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const int t = tid + 256 * i;
    const int iy = t / RX, ix = t - iy * RX;
    const int x = gx0 + ix, y = gy0 + iy;
    if (PRE) dl[i] = cdiv_den(interior ? interior_ap(ih2, kl[i], sr, si) : coef_at(F, x, y, kl[i], sr, si).ap);
  }
  if (PRE && tb0 == 0) {
    HELM_PDL_ENTRY();
    f = fv.get();
    fs = fv.scale();
  }
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const int t = tid + 256 * i;
    const int iy = t / RX, ix = t - iy * RX;
    const int x = gx0 + ix, y = gy0 + iy;
    const bool in = t < RX * RY && (interior || (x >= 0 && x < F.nx && y >= 0 && y < F.ny));
    const size_t p = in ? (size_t)y * F.nx + x : 0;
    fl[i] = in ? f[p] : czero();
  }
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const int t = tid + 256 * i;
    if (t < RX * RY) {
      const int iy = t / RX, ix = t - iy * RX;
      const int x = gx0 + ix, y = gy0 + iy;
      double2 uv = czero(), fvv = czero();
      double kk = 0.0;
      if (interior || (x >= 0 && x < F.nx && y >= 0 && y < F.ny)) {
        const size_t p = (size_t)y * F.nx + x;
        kk = kl[i];
        fvv = cscale(fs, fl[i]);
        const double2 ap = interior ? interior_ap(ih2, kk, sr, si) : coef_at(F, x, y, kk, sr, si).ap;
        uv = cscale(omega, PRE ? cdiv_d(fvv, ap, dl[i]) : cdiv(fvv, ap));   // reading R9: first sweep from u = 0
        if (x >= xs && x < xe && y >= ys && y < ye) u[p] = uv;
      }
      su[t] = uv;
      sf[t] = fvv;
      sk[t] = kk;
    }
  }
  }
  __syncthreads();
  for (int t = tid; t < QX * QY; t += 256) {
    {
      const int iy = t / QX, ix = t - iy * QX;
      const int x = gx0 + 1 + ix, y = gy0 + 1 + iy;
      const int q = (iy + 1) * RX + (ix + 1);
      double2 rv = czero();                      // reading R4: out-of-array taps dropped
      if (interior) {
        rv = csub(sf[q], interior_stencil(ih2, interior_ap(ih2, sk[q], sr, si), su[q], su[q - 1], su[q + 1],
                                          su[q - RX], su[q + RX]));
      } else if (x >= 0 && x < F.nx && y >= 0 && y < F.ny) {
        const Coef c = coef_at(F, x, y, sk[q], sr, si);
        rv = csub(sf[q], stencil5(c, su[q], su[q - 1], su[q + 1], su[q - RX], su[q + RX]));
      }
      sq[iy * QX + ix] = rv;
    }
  }
  __syncthreads();
  for (int t = tid; t < TCX * TCY; t += 256) {
    {
      const int jl = t / TCX, il = t - jl * TCX;
      const int I = I0 + il, J = J0 + jl;
      if (I >= G.nx || J >= G.ny) continue;
      const int ix = 2 * il + 1, iy = 2 * jl + 1;
      double2 s = czero();
#pragma unroll
      for (int b = -1; b <= 1; ++b)
#pragma unroll
        for (int a = -1; a <= 1; ++a) {
          const double w = (a == 0 ? 2.0 : 1.0) * (b == 0 ? 2.0 : 1.0) * (1.0 / 16.0);
          s = cadd(s, cscale(w, sq[(iy + b) * QX + ix + a]));
        }
      fc[(size_t)J * G.nx + I] = s;
    }
  }
}

// ------------------------------------------------------------------ up leg
// CTA = TX x TY fine points, 32 x 8 threads; u1 is formed on the tile plus a 1-node halo.
template <int TX, int TY>
__global__ void __launch_bounds__(256, HELM_VC_MINB) k_vc_up(Geo F, Geo G, int o, const double2* __restrict__ u,
                                               const double2* __restrict__ e, DVec fv,
                                               const double* __restrict__ k, double sr, double si, double omega,
                                               const double2* __restrict__ addq, DVec yv) {
  constexpr int RX = TX + 2, RY = TY + 2;
  constexpr int CX = TX / 2 + 3, CY = TY / 2 + 3;
  __shared__ double2 se[CY * CX];
  __shared__ double2 s1[RY * RX];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const double2* __restrict__ f = fv.get();
  const double fs = fv.scale();
  double2* __restrict__ y = yv.get();
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int cx0 = floordiv2(x0 - 1 - o), cy0 = floordiv2(y0 - 1 - o);
  const bool interior = x0 >= 2 && x0 + TX <= F.nx - 2 && y0 >= 2 && y0 + TY <= F.ny - 2 &&
                        cx0 >= 0 && cx0 + CX <= G.nx && cy0 >= 0 && cy0 + CY <= G.ny;
  const double ih2 = 1.0 / (F.h * F.h);
  const int tid = ty * 32 + tx;
  static_assert(TY == 8 && TX <= 32, "one output point per thread");
  // every global load of the tile is issued up front: the coarse correction e (NE per thread),
  // u on the tile + halo (NU per thread) and the output point's f, k (, q)
  // Only e is the output of the kernel launched just before this one (the coarser level's up leg
  // or the coarsest solve).  u (this level's down leg), f (this level's right-hand side, written
  // before the down leg), k and q (written before the V-cycle) come from kernels that completed
  // before that predecessor passed its own griddepcontrol.wait, i.e. before it let this grid be
  // scheduled: they are loaded before the PDL wait and their latency overlaps the predecessor.
  constexpr int NE = (CX * CY + 255) / 256, NU = (RX * RY + 255) / 256;
  double2 el[NE], ul[NU];
#pragma unroll
  for (int i = 0; i < NU; ++i) {
    const int t = tid + 256 * i;
    const int r = t / RX, c = t - r * RX;
    const int yy = y0 - 1 + r, x = x0 - 1 + c;
    ul[i] = (t < RX * RY && (interior || (x >= 0 && x < F.nx && yy >= 0 && yy < F.ny))) ? u[(size_t)yy * F.nx + x]
                                                                                          : czero();
  }
  const int ox_ = x0 + tx, oy_ = y0 + ty;
  const bool oin = tx < TX && ox_ < F.nx && oy_ < F.ny;
  const size_t po = oin ? (size_t)oy_ * F.nx + ox_ : 0;
  const double2 fo = oin ? f[po] : czero();
  const double ko = oin ? k[po] : 0.0;
  const double2 qo = (oin && addq) ? addq[po] : czero();
  const double2 apo = interior ? interior_ap(ih2, ko, sr, si) : coef_at(F, ox_, oy_, ko, sr, si).ap;
  const double dpo = cdiv_den(apo);
  HELM_PDL_ENTRY();
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    const int t = tid + 256 * i;
    const int r = t / CX, c = t - r * CX;
    const int J = cy0 + r, I = cx0 + c;
    el[i] = (t < CX * CY && (interior || (I >= 0 && I < G.nx && J >= 0 && J < G.ny))) ? e[(size_t)J * G.nx + I] : czero();
  }
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    const int t = tid + 256 * i;
    if (t < CX * CY) se[t] = el[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NU; ++i) {
    const int t = tid + 256 * i;
    if (t < RX * RY) {
      const int r = t / RX, c = t - r * RX;
      const int yy = y0 - 1 + r;
      const int rj = yy - o;
      const int Ja = floordiv2(rj);
      const bool oy = (rj & 1) != 0;
      const int ly = Ja - cy0;
      const int x = x0 - 1 + c;
      double2 v = czero();
      if (interior || (x >= 0 && x < F.nx && yy >= 0 && yy < F.ny)) {
        const int ri = x - o;
        const int Ia = floordiv2(ri);
        const bool ox = (ri & 1) != 0;
        const int lx = Ia - cx0;
        const double2* e0 = se + ly * CX + lx;
        // bilinear (Eq. 3.9): weights 1, 1/2 or 1/4 by parity, branch-free (the parities alternate
        // across the lanes of a warp): s = wy0 (wx0 e00 + wx1 e01) + wy1 (wx0 e10 + wx1 e11) with
        // power-of-two weights, so every product is exact and s equals the per-parity forms
        // e00, (e00/2 + e01/2), (e00/4 + e01/4) + (e10/4 + e11/4) bit for bit
        const double wx0 = ox ? 0.5 : 1.0, wx1 = ox ? 0.5 : 0.0;
        const double wy0 = oy ? 0.5 : 1.0, wy1 = oy ? 0.5 : 0.0;
        const double2 a = cadd(cscale(wx0, e0[0]), cscale(wx1, e0[1]));
        const double2 b = cadd(cscale(wx0, e0[CX]), cscale(wx1, e0[CX + 1]));
        const double2 s = cadd(cscale(wy0, a), cscale(wy1, b));
        v = cadd(s, ul[i]);
      }
      s1[t] = v;
    }
  }
  __syncthreads();
  if (oin) {
    const int r = ty, c = tx;
    const int q = (r + 1) * RX + (c + 1);
    double2 res;
    if (interior) {
      res = csub(cscale(fs, fo), interior_stencil(ih2, apo, s1[q], s1[q - 1], s1[q + 1], s1[q - RX], s1[q + RX]));
    } else {
      const Coef cf = coef_at(F, ox_, oy_, ko, sr, si);
      res = csub(cscale(fs, fo), stencil5(cf, s1[q], s1[q - 1], s1[q + 1], s1[q - RX], s1[q + RX]));
    }
    double2 v = cadd(s1[q], cscale(omega, cdiv_d(res, apo, dpo)));
    if (addq) v = cadd(v, qo);
    y[po] = v;
  }
}

// ------------------------------------------------------------------ column-streaming legs
// For large levels the tiled legs are limited by the L1/shared-memory pipe (every u/r value is
// staged and re-read from shared memory).  Here a warp owns 28 fine columns (lanes cover the
// 32 columns xo-2 .. xo+29: a 2-column halo each side) and streams down a segment of rows;
// x-neighbours come from warp shuffles, y-neighbours from registers (a ring of the last rows),
// so each f, k, u value is read from global memory once and shared memory is not used.
constexpr int COL_OWN = 28;   // fine columns owned per warp
constexpr int COL_SEG = 64;   // fine rows owned per warp

__device__ __forceinline__ double2 shfl_up2(double2 v, int d) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
}
__device__ __forceinline__ double2 shfl_dn2(double2 v, int d) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
}

// Down leg, column-streaming form (same arithmetic as k_vc_down):
//   u = omega f / D,  r = f - M u,  f_c = I_h^{2h} r.
// Grid: x = ceil(nx / 28) warp-columns (4 warps per block along x), y = ceil(ny / 64) segments.
__global__ void __launch_bounds__(128) k_vc_down_col(Geo F, Geo G, int o, DVec fv, const double* __restrict__ k,
                                                     double sr, double si, double omega, double2* __restrict__ u,
                                                     double2* __restrict__ fc) {
  HELM_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int wcol = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int xo = wcol * COL_OWN;
  if (xo >= F.nx) return;
  const int x = xo - 2 + lane;
  const bool xin = (x >= 0 && x < F.nx);
  const bool xown = (lane >= 2 && lane < 2 + COL_OWN && x < F.nx);
  const int ya = blockIdx.y * COL_SEG;
  const int yb = min(F.ny, ya + COL_SEG);
  const double2* __restrict__ f = fv.get();
  const double fs = fv.scale();
  // coarse column of this lane's fine column (restriction centre when even relative index)
  const int ri = x - o;
  const bool xcentre = ((ri & 1) == 0) && ri >= 0 && (ri >> 1) < G.nx && xown;
  const int I = ri >> 1;
  // rings: u at rows y-2, y-1, y; f, k at row y-1; r at rows y-3, y-2, y-1
  double2 um2 = czero(), um1 = czero(), fm1 = czero(), rm3 = czero(), rm2 = czero();
  double km1 = 0.0;
  // software pipeline: f and k of rows y and y+1 are loaded one and two iterations ahead
  auto ldf = [&](int yy, double2& fo, double& ko) {
    if (xin && yy >= 0 && yy < F.ny) {
      const size_t p = (size_t)yy * F.nx + x;
      fo = f[p];
      ko = k[p];
    } else {
      fo = czero();
      ko = 0.0;
    }
  };
  double2 fA, fB;
  double kA, kB;
  ldf(ya - 2, fA, kA);
  ldf(ya - 1, fB, kB);
  for (int y = ya - 2; y <= yb + 1; ++y) {
    const bool yin = (y >= 0 && y < F.ny);
    const double2 fraw = fA;
    const double k0 = kA;
    fA = fB;
    kA = kB;
    ldf(y + 2, fB, kB);
    double2 f0 = czero(), u0 = czero();
    if (xin && yin) {
      f0 = cscale(fs, fraw);
      const Coef c = coef_at(F, x, y, k0, sr, si);
      u0 = cscale(omega, cdiv(f0, c.ap));   // reading R9: first sweep from u = 0
      if (xown && y >= ya && y < yb) u[(size_t)y * F.nx + x] = u0;
    }
    // residual at row y-1 (needs u rows y-2, y-1, y)
    const int yr = y - 1;
    const double2 uw = shfl_up2(um1, 1), ue = shfl_dn2(um1, 1);
    double2 r = czero();                      // reading R4: out-of-array taps dropped
    if (xin && yr >= 0 && yr < F.ny && lane >= 1 && lane <= 30) {
      const Coef c = coef_at(F, x, yr, km1, sr, si);
      r = csub(fm1, stencil5(c, um1, uw, ue, um2, u0));
    }
    // restriction for the coarse row whose centre is fine row y-2 (needs r rows y-3, y-2, y-1)
    const int yc = y - 2;
    const int rj = yc - o;
    {
      const double2 a0 = shfl_up2(rm3, 1), a2 = shfl_dn2(rm3, 1);
      const double2 b0 = shfl_up2(rm2, 1), b2 = shfl_dn2(rm2, 1);
      const double2 c0 = shfl_up2(r, 1), c2 = shfl_dn2(r, 1);
      if (xcentre && yc >= ya && yc < yb && ((rj & 1) == 0) && rj >= 0 && (rj >> 1) < G.ny) {
        double2 s = czero();
        // same tap order as k_vc_down: b = -1, 0, 1 outer; a = -1, 0, 1 inner
        s = cadd(s, cscale(1.0 / 16.0, a0));
        s = cadd(s, cscale(2.0 / 16.0, rm3));
        s = cadd(s, cscale(1.0 / 16.0, a2));
        s = cadd(s, cscale(2.0 / 16.0, b0));
        s = cadd(s, cscale(4.0 / 16.0, rm2));
        s = cadd(s, cscale(2.0 / 16.0, b2));
        s = cadd(s, cscale(1.0 / 16.0, c0));
        s = cadd(s, cscale(2.0 / 16.0, r));
        s = cadd(s, cscale(1.0 / 16.0, c2));
        fc[(size_t)(rj >> 1) * G.nx + I] = s;
      }
    }
    rm3 = rm2;
    rm2 = r;
    um2 = um1;
    um1 = u0;
    fm1 = f0;
    km1 = k0;
  }
}

// ---- cp.async-pipelined column legs: the rows ahead are staged in a per-warp shared-memory
// ring by asynchronous copies (LDGSTS; each lane copies and later reads only its own slots, so
// no barrier), PF rows in flight per warp without holding them in registers.
__device__ __forceinline__ void cpa16(void* smem, const void* g, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(pred ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cpa8(void* smem, const void* g, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g), "r"(pred ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Down leg (same arithmetic and tap order as k_vc_down_col), f and k staged PF rows ahead.
// INT: every node the warp touches is interior (all four neighbours in the grid, no boundary
// row), so the multipliers are the branch-free interior ones (identical values and operation
// order); the restriction's shuffles run only on the rows that end a coarse row.
template <int PF, int SEG, bool INT>
__device__ __forceinline__ void down_cpa_body(const Geo& F, const Geo& G, int o, const double2* __restrict__ f,
                                              double fs, const double* __restrict__ k, double sr, double si,
                                              double omega, double2* __restrict__ u, double2* __restrict__ fc,
                                              double2 (*rf)[32], double (*rk)[32], int lane, int xo, int ya, int yb) {
  const int x = xo - 2 + lane;
  const bool xin = (x >= 0 && x < F.nx);
  const bool xown = (lane >= 2 && lane < 2 + COL_OWN && x < F.nx);
  const int ri = x - o;
  const bool xcentre = ((ri & 1) == 0) && ri >= 0 && (ri >> 1) < G.nx && xown;
  const int I = ri >> 1;
  const double ih2 = 1.0 / (F.h * F.h);
  const int y0 = ya - 2, y1 = yb + 1;   // rows consumed
  auto issue = [&](int yy) {
    const int slot = (yy - y0) % PF;
    const bool ok = xin && yy >= 0 && yy < F.ny && yy <= y1;
    const size_t p = ok ? (size_t)yy * F.nx + x : 0;
    cpa16(&rf[slot][lane], f + p, ok);
    cpa8(&rk[slot][lane], k + p, ok);
    cpa_commit();
  };
#pragma unroll
  for (int q = 0; q < PF; ++q) issue(y0 + q);
  double2 um2 = czero(), um1 = czero(), fm1 = czero(), rm3 = czero(), rm2 = czero();
  double km1 = 0.0;
  for (int y = y0; y <= y1; ++y) {
    cpa_wait<PF - 1>();
    const int slot = (y - y0) % PF;
    const double2 fraw = rf[slot][lane];
    const double k0 = rk[slot][lane];
    issue(y + PF);   // refills this lane's slot (already read)
    double2 f0 = czero(), u0 = czero();
    if (INT || (xin && y >= 0 && y < F.ny)) {
      f0 = cscale(fs, fraw);
      const double2 ap = INT ? interior_ap(ih2, k0, sr, si) : coef_at(F, x, y, k0, sr, si).ap;
      u0 = cscale(omega, cdiv(f0, ap));   // reading R9: first sweep from u = 0
      if (xown && y >= ya && y < yb) u[(size_t)y * F.nx + x] = u0;
    }
    const int yr = y - 1;
    const double2 uw = shfl_up2(um1, 1), ue = shfl_dn2(um1, 1);
    double2 r = czero();
    if (lane >= 1 && lane <= 30) {
      if (INT) {
        r = csub(fm1, interior_stencil(ih2, interior_ap(ih2, km1, sr, si), um1, uw, ue, um2, u0));
      } else if (xin && yr >= 0 && yr < F.ny) {
        const Coef c = coef_at(F, x, yr, km1, sr, si);
        r = csub(fm1, stencil5(c, um1, uw, ue, um2, u0));
      }
    }
    const int yc = y - 2;
    const int rj = yc - o;
    if (((rj & 1) == 0) && yc >= ya && yc < yb && rj >= 0 && (rj >> 1) < G.ny) {   // warp-uniform
      const double2 a0 = shfl_up2(rm3, 1), a2 = shfl_dn2(rm3, 1);
      const double2 b0 = shfl_up2(rm2, 1), b2 = shfl_dn2(rm2, 1);
      const double2 c0 = shfl_up2(r, 1), c2 = shfl_dn2(r, 1);
      if (xcentre) {
        double2 s = czero();
        s = cadd(s, cscale(1.0 / 16.0, a0));
        s = cadd(s, cscale(2.0 / 16.0, rm3));
        s = cadd(s, cscale(1.0 / 16.0, a2));
        s = cadd(s, cscale(2.0 / 16.0, b0));
        s = cadd(s, cscale(4.0 / 16.0, rm2));
        s = cadd(s, cscale(2.0 / 16.0, b2));
        s = cadd(s, cscale(1.0 / 16.0, c0));
        s = cadd(s, cscale(2.0 / 16.0, r));
        s = cadd(s, cscale(1.0 / 16.0, c2));
        fc[(size_t)(rj >> 1) * G.nx + I] = s;
      }
    }
    rm3 = rm2;
    rm2 = r;
    um2 = um1;
    um1 = u0;
    fm1 = f0;
    km1 = k0;
  }
  cpa_wait<0>();
}

template <int PF, int SEG = COL_SEG>
__global__ void __launch_bounds__(128) k_vc_down_cpa(Geo F, Geo G, int o, DVec fv, const double* __restrict__ k,
                                                     double sr, double si, double omega, double2* __restrict__ u,
                                                     double2* __restrict__ fc) {
  HELM_PDL_ENTRY();
  __shared__ double2 rf[4][PF][32];
  __shared__ double rk[4][PF][32];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int xo = (blockIdx.x * 4 + wq) * COL_OWN;
  if (xo >= F.nx) return;
  const int ya = blockIdx.y * SEG;
  const int yb = min(F.ny, ya + SEG);
  const bool interior = xo - 2 >= 1 && xo + 29 <= F.nx - 2 && ya - 3 >= 1 && yb + 1 <= F.ny - 2;
  if (interior)
    down_cpa_body<PF, SEG, true>(F, G, o, fv.get(), fv.scale(), k, sr, si, omega, u, fc, rf[wq], rk[wq], lane, xo,
                                 ya, yb);
  else
    down_cpa_body<PF, SEG, false>(F, G, o, fv.get(), fv.scale(), k, sr, si, omega, u, fc, rf[wq], rk[wq], lane, xo,
                                  ya, yb);
}

// Up leg, column-streaming form (same arithmetic as k_vc_up):
//   u1 = u + I_{2h}^h e,  y = u1 + omega (f - M u1)/D (+ q).
__global__ void __launch_bounds__(128) k_vc_up_col(Geo F, Geo G, int o, const double2* __restrict__ u,
                                                   const double2* __restrict__ e, DVec fv,
                                                   const double* __restrict__ k, double sr, double si, double omega,
                                                   const double2* __restrict__ addq, DVec yv) {
  HELM_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int wcol = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int xo = wcol * COL_OWN;
  if (xo >= F.nx) return;
  const int x = xo - 2 + lane;
  const bool xin = (x >= 0 && x < F.nx);
  const bool xown = (lane >= 2 && lane < 2 + COL_OWN && x < F.nx);
  const int ya = blockIdx.y * COL_SEG;
  const int yb = min(F.ny, ya + COL_SEG);
  const double2* __restrict__ f = fv.get();
  const double fs = fv.scale();
  double2* __restrict__ yo = yv.get();
  const int ri = x - o;
  const int Ia = floordiv2(ri);
  const bool ox = (ri & 1) != 0;
  const bool i0in = Ia >= 0 && Ia < G.nx, i1in = (Ia + 1) >= 0 && (Ia + 1) < G.nx;
  // bilinear interpolation of e at fine (x, y): weights 1, 1/2, 1/4 by parity (Eq. 3.9),
  // same operation order as k_vc_up (coarse values come from L1: adjacent lanes share them)
  auto interp = [&](int yy) -> double2 {
    const int rj = yy - o;
    const int Ja = floordiv2(rj);
    const bool oy = (rj & 1) != 0;
    auto ev = [&](int J, int Ii, bool iin) -> double2 {
      return (iin && J >= 0 && J < G.ny) ? e[(size_t)J * G.nx + Ii] : czero();
    };
    const double2 e00 = ev(Ja, Ia, i0in);
    if (!ox && !oy) return e00;
    if (ox && !oy) return cadd(cscale(0.5, e00), cscale(0.5, ev(Ja, Ia + 1, i1in)));
    if (!ox && oy) return cadd(cscale(0.5, e00), cscale(0.5, ev(Ja + 1, Ia, i0in)));
    return cadd(cadd(cscale(0.25, e00), cscale(0.25, ev(Ja, Ia + 1, i1in))),
                cadd(cscale(0.25, ev(Ja + 1, Ia, i0in)), cscale(0.25, ev(Ja + 1, Ia + 1, i1in))));
  };
  double2 v1m2 = czero(), v1m1 = czero();   // u1 at rows y-2, y-1
  auto ldu = [&](int yy) -> double2 { return (xin && yy >= 0 && yy < F.ny) ? u[(size_t)yy * F.nx + x] : czero(); };
  auto ldo = [&](int yy, double2& fo, double& ko, double2& qo) {
    if (xown && yy >= ya && yy < yb) {
      const size_t p = (size_t)yy * F.nx + x;
      fo = f[p];
      ko = k[p];
      qo = addq ? addq[p] : czero();
    } else {
      fo = czero();
      ko = 0.0;
      qo = czero();
    }
  };
  double2 uA = ldu(ya - 1);
  double2 fO, qO;
  double kO;
  ldo(ya - 2, fO, kO, qO);
  for (int y = ya - 1; y <= yb; ++y) {
    const bool yin = (y >= 0 && y < F.ny);
    const double2 ucur = uA;
    uA = ldu(y + 1);
    const double2 fcur = fO, qcur = qO;
    const double kcur = kO;
    ldo(y, fO, kO, qO);
    double2 v10 = czero();
    if (xin && yin) v10 = cadd(interp(y), ucur);
    // post-smoothing at row y-1 (needs u1 rows y-2, y-1, y)
    const int yr = y - 1;
    const double2 uw = shfl_up2(v1m1, 1), ue = shfl_dn2(v1m1, 1);
    if (xown && yr >= ya && yr < yb) {
      const size_t p = (size_t)yr * F.nx + x;
      const Coef c = coef_at(F, x, yr, kcur, sr, si);
      const double2 res = csub(cscale(fs, fcur), stencil5(c, v1m1, uw, ue, v1m2, v10));
      double2 out = cadd(v1m1, cscale(omega, cdiv(res, c.ap)));
      if (addq) out = cadd(out, qcur);
      yo[p] = out;
    }
    v1m2 = v1m1;
    v1m1 = v10;
  }
}

// Up leg (same arithmetic as k_vc_up_col): u staged PF rows ahead, f, k (and q) staged with it.
// INT as in the down leg (branch-free interior multipliers for the post-smoothing).
template <int PF, int SEG, bool INT>
__device__ __forceinline__ void up_cpa_body(const Geo& F, const Geo& G, int o, const double2* __restrict__ u,
                                            const double2* __restrict__ e, const double2* __restrict__ f, double fs,
                                            const double* __restrict__ k, double sr, double si, double omega,
                                            const double2* __restrict__ addq, double2* __restrict__ yo,
                                            double2 (*ru)[32], double2 (*rf)[32], double2 (*rq)[32], double (*rk)[32],
                                            int lane, int xo, int ya, int yb) {
  const int x = xo - 2 + lane;
  const bool xin = (x >= 0 && x < F.nx);
  const bool xown = (lane >= 2 && lane < 2 + COL_OWN && x < F.nx);
  const double ih2 = 1.0 / (F.h * F.h);
  const int ri = x - o;
  const int Ia = floordiv2(ri);
  const bool ox = (ri & 1) != 0;
  const bool i0in = Ia >= 0 && Ia < G.nx, i1in = (Ia + 1) >= 0 && (Ia + 1) < G.nx;
  auto interp = [&](int yy) -> double2 {
    const int rj = yy - o;
    const int Ja = floordiv2(rj);
    const bool oy = (rj & 1) != 0;
    auto ev = [&](int J, int Ii, bool iin) -> double2 {
      return (iin && J >= 0 && J < G.ny) ? e[(size_t)J * G.nx + Ii] : czero();
    };
    const double2 e00 = ev(Ja, Ia, i0in);
    if (!ox && !oy) return e00;
    if (ox && !oy) return cadd(cscale(0.5, e00), cscale(0.5, ev(Ja, Ia + 1, i1in)));
    if (!ox && oy) return cadd(cscale(0.5, e00), cscale(0.5, ev(Ja + 1, Ia, i0in)));
    return cadd(cadd(cscale(0.25, e00), cscale(0.25, ev(Ja, Ia + 1, i1in))),
                cadd(cscale(0.25, ev(Ja + 1, Ia, i0in)), cscale(0.25, ev(Ja + 1, Ia + 1, i1in))));
  };
  const int y0 = ya - 1, y1 = yb;   // rows of u consumed; f, k, q of row y are used one row later
  auto issue = [&](int yy) {
    const int slot = (yy - y0) % PF;
    const bool uok = xin && yy >= 0 && yy < F.ny && yy <= y1;
    const bool ook = xown && yy >= ya && yy < yb;
    const size_t pu = uok ? (size_t)yy * F.nx + x : 0;
    const size_t po = ook ? (size_t)yy * F.nx + x : 0;
    cpa16(&ru[slot][lane], u + pu, uok);
    cpa16(&rf[slot][lane], f + po, ook);
    cpa8(&rk[slot][lane], k + po, ook);
    if (addq) cpa16(&rq[slot][lane], addq + po, ook);
    cpa_commit();
  };
#pragma unroll
  for (int q = 0; q < PF; ++q) issue(y0 + q);
  double2 v1m2 = czero(), v1m1 = czero();
  double2 fcur = czero(), qcur = czero();
  double kcur = 0.0;
  double2 e0 = czero(), e1 = czero();   // INT: e at (Ja, Ia), (Ja + 1, Ia)
  int eJ = -1 << 30;
  for (int y = y0; y <= y1; ++y) {
    cpa_wait<PF - 1>();
    const int slot = (y - y0) % PF;
    const double2 ucur = ru[slot][lane];
    const double2 fnew = rf[slot][lane];
    const double knew = rk[slot][lane];
    const double2 qnew = addq ? rq[slot][lane] : czero();
    issue(y + PF);
    double2 v10 = czero();
    if (INT) {
      // coarse rows Ja, Ja + 1 of this fine row: each coarse value is loaded once (kept while
      // two fine rows use it) and column Ia + 1 comes from the next lane (whose base column
      // it is when ri is odd; lanes 0 and 31 only feed halo lanes, which store nothing)
      const int rj = y - o;
      const int Ja = floordiv2(rj);
      const bool oy = (rj & 1) != 0;
      if (Ja != eJ) {
        if (Ja == eJ + 1) {
          e0 = e1;
        } else {
          e0 = (Ja >= 0 && Ja < G.ny && i0in) ? e[(size_t)Ja * G.nx + Ia] : czero();
        }
        e1 = (Ja + 1 < G.ny && Ja + 1 >= 0 && i0in) ? e[(size_t)(Ja + 1) * G.nx + Ia] : czero();
        eJ = Ja;
      }
      const double2 e01 = shfl_dn2(e0, 1), e11 = shfl_dn2(e1, 1);
      double2 ip;
      if (!ox && !oy) ip = e0;
      else if (ox && !oy) ip = cadd(cscale(0.5, e0), cscale(0.5, e01));
      else if (!ox && oy) ip = cadd(cscale(0.5, e0), cscale(0.5, e1));
      else ip = cadd(cadd(cscale(0.25, e0), cscale(0.25, e01)), cadd(cscale(0.25, e1), cscale(0.25, e11)));
      v10 = cadd(ip, ucur);
    } else if (xin && y >= 0 && y < F.ny) {
      v10 = cadd(interp(y), ucur);
    }
    const int yr = y - 1;
    const double2 uw = shfl_up2(v1m1, 1), ue = shfl_dn2(v1m1, 1);
    if (xown && yr >= ya && yr < yb) {
      const size_t p = (size_t)yr * F.nx + x;
      double2 res, ap;
      if (INT) {
        ap = interior_ap(ih2, kcur, sr, si);
        res = csub(cscale(fs, fcur), interior_stencil(ih2, ap, v1m1, uw, ue, v1m2, v10));
      } else {
        const Coef c = coef_at(F, x, yr, kcur, sr, si);
        ap = c.ap;
        res = csub(cscale(fs, fcur), stencil5(c, v1m1, uw, ue, v1m2, v10));
      }
      double2 out = cadd(v1m1, cscale(omega, cdiv(res, ap)));
      if (addq) out = cadd(out, qcur);
      yo[p] = out;
    }
    v1m2 = v1m1;
    v1m1 = v10;
    fcur = fnew;
    kcur = knew;
    qcur = qnew;
  }
  cpa_wait<0>();
}

template <int PF, int SEG = COL_SEG>
__global__ void __launch_bounds__(128) k_vc_up_cpa(Geo F, Geo G, int o, const double2* __restrict__ u,
                                                   const double2* __restrict__ e, DVec fv,
                                                   const double* __restrict__ k, double sr, double si, double omega,
                                                   const double2* __restrict__ addq, DVec yv) {
  HELM_PDL_ENTRY();
  __shared__ double2 ru[4][PF][32];
  __shared__ double2 rf[4][PF][32];
  __shared__ double2 rq[4][PF][32];
  __shared__ double rk[4][PF][32];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int xo = (blockIdx.x * 4 + wq) * COL_OWN;
  if (xo >= F.nx) return;
  const int ya = blockIdx.y * SEG;
  const int yb = min(F.ny, ya + SEG);
  const bool interior = xo - 2 >= 1 && xo + 29 <= F.nx - 2 && ya - 2 >= 1 && yb <= F.ny - 2;
  if (interior)
    up_cpa_body<PF, SEG, true>(F, G, o, u, e, fv.get(), fv.scale(), k, sr, si, omega, addq, yv.get(), ru[wq], rf[wq],
                               rq[wq], rk[wq], lane, xo, ya, yb);
  else
    up_cpa_body<PF, SEG, false>(F, G, o, u, e, fv.get(), fv.scale(), k, sr, si, omega, addq, yv.get(), ru[wq],
                                rf[wq], rq[wq], rk[wq], lane, xo, ya, yb);
}

// ---- TMA column legs: the rows ahead are staged by the Tensor Memory Accelerator
// (cp.async.bulk.tensor, one instruction per row and field issued by lane 0; completion on a
// per-slot mbarrier with the transaction byte count).  The tensor maps describe each field as a
// 2D float64 array (complex128 = 2 doubles); a warp's row segment is one 32-column box whose
// out-of-grid columns / rows the TMA unit fills with zeros -- the same values the LDGSTS legs
// substitute.  Same arithmetic and tap order as the cp.async legs (down_cpa_body / up_cpa_body).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_row(void* dst, const CUtensorMap* map, int x, int y, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// k is float64 with rows of odd length, whose byte stride is not a multiple of 16 (a TMA
// requirement): the legs read a copy with an even row stride (Level.kp), mapped in 2D like the
// complex fields (zero fill outside the grid).
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// CTA-wide staging: the 4 warps of a CTA own 4 x 28 consecutive columns; one box of TMA_W = 116
// columns (2 halo columns each side) x R rows per field and stage, S stages in flight.  full[s]
// completes when the stage's bytes landed (transaction count), empty[s] when every active warp
// has read it; thread 0 refills a stage after its empty barrier.  (A dedicated producer warp was
// measured slower: 0.61 / 0.56 of HBM on 16383^2, its 160-thread CTAs hold fewer warps per SM.)  Warp w reads column 28 w + lane
// of the box, i.e. the same fine column as lane `lane` of the per-warp legs.
constexpr int TMA_W = 4 * COL_OWN + 4;
// stage sizes padded to 128 bytes (TMA destinations); R even keeps the complex stages aligned
template <int R>
struct TmaStage {
  static_assert(R % 2 == 0, "R even");
  static constexpr int C = R * TMA_W;                 // complex values per stage (R * 1856 B)
  static constexpr int K = (R * TMA_W + 15) / 16 * 16;   // doubles per stage, 128-B multiple
};

template <int R, int S, int SEG>
__global__ void __launch_bounds__(128) k_vc_down_tma(Geo F, Geo G, int o, const __grid_constant__ CUtensorMap mf,
                                                     const __grid_constant__ CUtensorMap mk, double fs, double sr,
                                                     double si, double omega, double2* __restrict__ u,
                                                     double2* __restrict__ fc) {
  HELM_PDL_ENTRY();
  using ST = TmaStage<R>;
  __shared__ alignas(128) double2 rf[S * ST::C];
  __shared__ alignas(128) double rk[S * ST::K];
  __shared__ unsigned long long full[S], empty[S];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int xc = blockIdx.x * 4 * COL_OWN;
  const int nact = min(4, (F.nx - xc + COL_OWN - 1) / COL_OWN);   // warps with columns
  const int ya = blockIdx.y * SEG;
  const int yb = min(F.ny, ya + SEG);
  const int y0 = ya - 2, y1 = yb + 1;   // rows consumed
  const int nst = (y1 - y0 + R) / R;    // stages
  if (threadIdx.x == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], nact);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int t) {   // thread 0: stage t into slot t % S
    const int q = t % S;
    mbar_expect_tx(&full[q], R * TMA_W * 24);
    tma_row(rf + q * ST::C, &mf, 2 * (xc - 2), y0 + t * R, &full[q]);
    tma_row(rk + q * ST::K, &mk, xc - 2, y0 + t * R, &full[q]);
  };
  if (threadIdx.x == 0)
    for (int t = 0; t < S && t < nst; ++t) issue(t);
  if (wq >= nact) return;   // no columns (after the barrier set-up; not counted in empty)
  const int xo = xc + wq * COL_OWN;
  const int x = xo - 2 + lane;
  const int col = wq * COL_OWN + lane;
  const bool xin = (x >= 0 && x < F.nx);
  const bool xown = (lane >= 2 && lane < 2 + COL_OWN && x < F.nx);
  const int ri = x - o;
  const bool xcentre = ((ri & 1) == 0) && ri >= 0 && (ri >> 1) < G.nx && xown;
  const int I = ri >> 1;
  const bool INT = xo - 2 >= 1 && xo + 29 <= F.nx - 2 && ya - 3 >= 1 && yb + 1 <= F.ny - 2;
  const double ih2 = 1.0 / (F.h * F.h);
  double2 um2 = czero(), um1 = czero(), fm1 = czero(), rm3 = czero(), rm2 = czero();
  double km1 = 0.0;
  for (int y = y0; y <= y1; ++y) {
    const int t = (y - y0) / R, r = (y - y0) - t * R, q = t % S;
    if (r == 0) mbar_wait(&full[q], (t / S) & 1);
    const double2 fraw = rf[q * ST::C + r * TMA_W + col];
    const double k0 = rk[q * ST::K + r * TMA_W + col];
    if (r == R - 1 || y == y1) {   // this warp is done with stage t
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[q]);
      if (threadIdx.x == 0 && t + S < nst) {   // thread 0 refills the slot once every warp left it
        mbar_wait(&empty[q], (t / S) & 1);
        issue(t + S);
      }
    }
    double2 f0 = czero(), u0 = czero();
    if (INT || (xin && y >= 0 && y < F.ny)) {
      f0 = cscale(fs, fraw);
      const double2 ap = INT ? interior_ap(ih2, k0, sr, si) : coef_at(F, x, y, k0, sr, si).ap;
      u0 = cscale(omega, cdiv(f0, ap));   // reading R9: first sweep from u = 0
      if (xown && y >= ya && y < yb) u[(size_t)y * F.nx + x] = u0;
    }
    const int yr = y - 1;
    const double2 uw = shfl_up2(um1, 1), ue = shfl_dn2(um1, 1);
    double2 rr = czero();
    if (lane >= 1 && lane <= 30) {
      if (INT) {
        rr = csub(fm1, interior_stencil(ih2, interior_ap(ih2, km1, sr, si), um1, uw, ue, um2, u0));
      } else if (xin && yr >= 0 && yr < F.ny) {
        const Coef c = coef_at(F, x, yr, km1, sr, si);
        rr = csub(fm1, stencil5(c, um1, uw, ue, um2, u0));
      }
    }
    const int yc = y - 2;
    const int rj = yc - o;
    if (((rj & 1) == 0) && yc >= ya && yc < yb && rj >= 0 && (rj >> 1) < G.ny) {   // warp-uniform
      const double2 a0 = shfl_up2(rm3, 1), a2 = shfl_dn2(rm3, 1);
      const double2 b0 = shfl_up2(rm2, 1), b2 = shfl_dn2(rm2, 1);
      const double2 c0 = shfl_up2(rr, 1), c2 = shfl_dn2(rr, 1);
      if (xcentre) {
        double2 sacc = czero();
        sacc = cadd(sacc, cscale(1.0 / 16.0, a0));
        sacc = cadd(sacc, cscale(2.0 / 16.0, rm3));
        sacc = cadd(sacc, cscale(1.0 / 16.0, a2));
        sacc = cadd(sacc, cscale(2.0 / 16.0, b0));
        sacc = cadd(sacc, cscale(4.0 / 16.0, rm2));
        sacc = cadd(sacc, cscale(2.0 / 16.0, b2));
        sacc = cadd(sacc, cscale(1.0 / 16.0, c0));
        sacc = cadd(sacc, cscale(2.0 / 16.0, rr));
        sacc = cadd(sacc, cscale(1.0 / 16.0, c2));
        fc[(size_t)(rj >> 1) * G.nx + I] = sacc;
      }
    }
    rm3 = rm2;
    rm2 = rr;
    um2 = um1;
    um1 = u0;
    fm1 = f0;
    km1 = k0;
  }
}

// Up leg with CTA-wide TMA staging of u, f, k (and q) of each row.
template <int R, int S, int SEG, bool Q>
__global__ void __launch_bounds__(128) k_vc_up_tma(Geo F, Geo G, int o, const __grid_constant__ CUtensorMap mu,
                                                   const double2* __restrict__ e, const __grid_constant__ CUtensorMap mf,
                                                   double fs, const __grid_constant__ CUtensorMap mk, double sr,
                                                   double si, double omega, const __grid_constant__ CUtensorMap mq,
                                                   DVec yv) {
  HELM_PDL_ENTRY();
  using ST = TmaStage<R>;
  __shared__ alignas(128) double2 ru[S * ST::C];
  __shared__ alignas(128) double2 rf[S * ST::C];
  __shared__ alignas(128) double2 rq[Q ? S * ST::C : 8];
  __shared__ alignas(128) double rk[S * ST::K];
  __shared__ unsigned long long full[S], empty[S];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int xc = blockIdx.x * 4 * COL_OWN;
  const int nact = min(4, (F.nx - xc + COL_OWN - 1) / COL_OWN);
  const int ya = blockIdx.y * SEG;
  const int yb = min(F.ny, ya + SEG);
  const int y0 = ya - 1, y1 = yb;   // rows of u consumed; f, k, q of row y are used one row later
  const int nst = (y1 - y0 + R) / R;
  if (threadIdx.x == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], nact);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int t) {
    const int q = t % S;
    mbar_expect_tx(&full[q], R * TMA_W * (Q ? 56 : 40));
    tma_row(ru + q * ST::C, &mu, 2 * (xc - 2), y0 + t * R, &full[q]);
    tma_row(rf + q * ST::C, &mf, 2 * (xc - 2), y0 + t * R, &full[q]);
    tma_row(rk + q * ST::K, &mk, xc - 2, y0 + t * R, &full[q]);
    if (Q) tma_row(rq + q * ST::C, &mq, 2 * (xc - 2), y0 + t * R, &full[q]);
  };
  if (threadIdx.x == 0)
    for (int t = 0; t < S && t < nst; ++t) issue(t);
  if (wq >= nact) return;
  double2* __restrict__ yo = yv.get();
  const int xo = xc + wq * COL_OWN;
  const int x = xo - 2 + lane;
  const int col = wq * COL_OWN + lane;
  const bool xin = (x >= 0 && x < F.nx);
  const bool xown = (lane >= 2 && lane < 2 + COL_OWN && x < F.nx);
  const double ih2 = 1.0 / (F.h * F.h);
  const int ri = x - o;
  const int Ia = floordiv2(ri);
  const bool ox = (ri & 1) != 0;
  const bool i0in = Ia >= 0 && Ia < G.nx, i1in = (Ia + 1) >= 0 && (Ia + 1) < G.nx;
  const bool INT = xo - 2 >= 1 && xo + 29 <= F.nx - 2 && ya - 2 >= 1 && yb <= F.ny - 2;
  auto interp = [&](int yy) -> double2 {
    const int rj = yy - o;
    const int Ja = floordiv2(rj);
    const bool oy = (rj & 1) != 0;
    auto ev = [&](int J, int Ii, bool iin) -> double2 {
      return (iin && J >= 0 && J < G.ny) ? e[(size_t)J * G.nx + Ii] : czero();
    };
    const double2 e00 = ev(Ja, Ia, i0in);
    if (!ox && !oy) return e00;
    if (ox && !oy) return cadd(cscale(0.5, e00), cscale(0.5, ev(Ja, Ia + 1, i1in)));
    if (!ox && oy) return cadd(cscale(0.5, e00), cscale(0.5, ev(Ja + 1, Ia, i0in)));
    return cadd(cadd(cscale(0.25, e00), cscale(0.25, ev(Ja, Ia + 1, i1in))),
                cadd(cscale(0.25, ev(Ja + 1, Ia, i0in)), cscale(0.25, ev(Ja + 1, Ia + 1, i1in))));
  };
  double2 v1m2 = czero(), v1m1 = czero();
  double2 fcur = czero(), qcur = czero();
  double kcur = 0.0;
  double2 e0 = czero(), e1 = czero();
  int eJ = -1 << 30;
  for (int y = y0; y <= y1; ++y) {
    const int t = (y - y0) / R, r = (y - y0) - t * R, q = t % S;
    if (r == 0) mbar_wait(&full[q], (t / S) & 1);
    const double2 ucur = ru[q * ST::C + r * TMA_W + col];
    const double2 fnew = rf[q * ST::C + r * TMA_W + col];
    const double knew = rk[q * ST::K + r * TMA_W + col];
    const double2 qnew = Q ? rq[q * ST::C + r * TMA_W + col] : czero();
    if (r == R - 1 || y == y1) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[q]);
      if (threadIdx.x == 0 && t + S < nst) {
        mbar_wait(&empty[q], (t / S) & 1);
        issue(t + S);
      }
    }
    double2 v10 = czero();
    if (INT) {
      const int rj = y - o;
      const int Ja = floordiv2(rj);
      const bool oy = (rj & 1) != 0;
      if (Ja != eJ) {
        if (Ja == eJ + 1) {
          e0 = e1;
        } else {
          e0 = (Ja >= 0 && Ja < G.ny && i0in) ? e[(size_t)Ja * G.nx + Ia] : czero();
        }
        e1 = (Ja + 1 < G.ny && Ja + 1 >= 0 && i0in) ? e[(size_t)(Ja + 1) * G.nx + Ia] : czero();
        eJ = Ja;
      }
      const double2 e01 = shfl_dn2(e0, 1), e11 = shfl_dn2(e1, 1);
      double2 ip;
      if (!ox && !oy) ip = e0;
      else if (ox && !oy) ip = cadd(cscale(0.5, e0), cscale(0.5, e01));
      else if (!ox && oy) ip = cadd(cscale(0.5, e0), cscale(0.5, e1));
      else ip = cadd(cadd(cscale(0.25, e0), cscale(0.25, e01)), cadd(cscale(0.25, e1), cscale(0.25, e11)));
      v10 = cadd(ip, ucur);
    } else if (xin && y >= 0 && y < F.ny) {
      v10 = cadd(interp(y), ucur);
    }
    const int yr = y - 1;
    const double2 uw = shfl_up2(v1m1, 1), ue = shfl_dn2(v1m1, 1);
    if (xown && yr >= ya && yr < yb) {
      const size_t p = (size_t)yr * F.nx + x;
      double2 res, ap;
      if (INT) {
        ap = interior_ap(ih2, kcur, sr, si);
        res = csub(cscale(fs, fcur), interior_stencil(ih2, ap, v1m1, uw, ue, v1m2, v10));
      } else {
        const Coef c = coef_at(F, x, yr, kcur, sr, si);
        ap = c.ap;
        res = csub(cscale(fs, fcur), stencil5(c, v1m1, uw, ue, v1m2, v10));
      }
      double2 out = cadd(v1m1, cscale(omega, cdiv(res, ap)));
      if (Q) out = cadd(out, qcur);
      yo[p] = out;
    }
    v1m2 = v1m1;
    v1m1 = v10;
    fcur = fnew;
    kcur = knew;
    qcur = qnew;
  }
}

// ------------------------------------------------------------------ cluster tail
// The remaining levels lt..last of a V-cycle (small grids) run in ONE thread-block cluster of
// CS CTAs (CS = 16 on B200, one CTA per SM): every level's arrays (f, u, two scratch fields and
// k) are partitioned by rows across the cluster's shared memories; a stencil tap in a row owned
// by another CTA is read through distributed shared memory (DSMEM); stages are separated by
// cluster barriers.  Only the input f, the output u (+ q) and the dense coarsest inverse touch
// global memory.  CS = 1 degenerates to a single-CTA tail.
struct LevelDesc {
  Geo g;
  int o;
  const double* k;
};

__host__ __device__ inline int tail_rpc(int ny, int cs) { return (ny + cs - 1) / cs; }

// Shared-memory bytes per CTA for levels lt..last with a cluster of cs CTAs.
__host__ __device__ inline size_t tail_smem_bytes(const LevelDesc* Ls, int lt, int last, int cs) {
  size_t b = 0;
  for (int l = lt; l <= last; ++l) {
    const size_t n = (size_t)tail_rpc(Ls[l].g.ny, cs) * Ls[l].g.nx;
    b += n * 4 * sizeof(double2) + ((n * sizeof(double) + 15) / 16) * 16;   // keep 16-byte alignment
  }
  return b + (size_t)Ls[last].g.nx * Ls[last].g.ny * sizeof(double2);   // + the gathered coarsest rhs
}

struct TailLevel {
  Geo g;
  int o;
  int rpc;          // rows per CTA
  int r0, r1;       // rows owned by this CTA
  double* k;
  double2 *f, *u, *s, *t;
};

constexpr int TAIL_MAX_LEVELS = 24;

// Pointer to element (i, j) of a level array whose local (this CTA's) base is `base`.
__device__ __forceinline__ double2* tail_at(cg::cluster_group& cl, const TailLevel& L, double2* base, int i, int j,
                                            unsigned rank) {
  const int owner = j / L.rpc;
  double2* p = base + (size_t)(j - owner * L.rpc) * L.g.nx + i;
  return (owner == (int)rank) ? p : cl.map_shared_rank(p, owner);
}

// Stencil of the level operator at (i, j) reading `arr` through DSMEM where needed.
__device__ __forceinline__ double2 tail_stencil(cg::cluster_group& cl, const TailLevel& L, double2* arr, int i, int j,
                                                unsigned rank, const Coef& c) {
  const double2* row = arr + (size_t)(j - L.r0) * L.g.nx;   // own row
  double2 v = cmul(c.ap, row[i]);
  if (c.aw != 0.0) v = cadd(v, cscale(c.aw, row[i - 1]));
  if (c.ae != 0.0) v = cadd(v, cscale(c.ae, row[i + 1]));
  if (c.as != 0.0) v = cadd(v, cscale(c.as, *tail_at(cl, L, arr, i, j - 1, rank)));
  if (c.an != 0.0) v = cadd(v, cscale(c.an, *tail_at(cl, L, arr, i, j + 1, rank)));
  return v;
}

__device__ __forceinline__ void tail_jacobi(cg::cluster_group& cl, const TailLevel& L, double2* u, const double2* f,
                                            double2* out, double sr, double si, double omega, unsigned rank) {
  const int nx = L.g.nx;
  const int n = (L.r1 - L.r0) * nx;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    const int i = p % nx, j = L.r0 + p / nx;
    const Coef c = coef_at(L.g, i, j, L.k[p], sr, si);
    const double2 r = csub(f[p], tail_stencil(cl, L, u, i, j, rank, c));
    out[p] = cadd(u[p], cscale(omega, cdiv(r, c.ap)));
  }
}

__global__ void __launch_bounds__(1024) k_vc_tail(const LevelDesc* __restrict__ Ls, int lt, int last, DVec fv,
                                                  DVec uv, const double2* __restrict__ addq, double sr, double si,
                                                  double omega, int nu_pre, int nu_post,
                                                  const double2* __restrict__ Minv) {
  HELM_PDL_ENTRY();
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  const int cs = (int)cl.num_blocks();
  extern __shared__ double2 tsm[];
  __shared__ TailLevel T[TAIL_MAX_LEVELS];
  __shared__ int curi[TAIL_MAX_LEVELS];   // 0: pre-smoothed iterate in s, 1: in t
  __shared__ double2* s_gat;               // the whole coarsest rhs, gathered into this CTA
  double2* const uout = uv.get();
  const double2* const fin = fv.get();
  const double fsc = fv.scale();
  const int nl = last - lt + 1;
  if (threadIdx.x == 0) {
    char* p = reinterpret_cast<char*>(tsm);
    for (int q = 0; q < nl; ++q) {
      const LevelDesc D = Ls[lt + q];
      const int rpc = tail_rpc(D.g.ny, cs);
      const size_t n = (size_t)rpc * D.g.nx;
      T[q].g = D.g;
      T[q].o = D.o;
      T[q].rpc = rpc;
      T[q].r0 = min(D.g.ny, (int)rank * rpc);
      T[q].r1 = min(D.g.ny, ((int)rank + 1) * rpc);
      T[q].f = reinterpret_cast<double2*>(p); p += n * sizeof(double2);
      T[q].u = reinterpret_cast<double2*>(p); p += n * sizeof(double2);
      T[q].s = reinterpret_cast<double2*>(p); p += n * sizeof(double2);
      T[q].t = reinterpret_cast<double2*>(p); p += n * sizeof(double2);
      T[q].k = reinterpret_cast<double*>(p); p += ((n * sizeof(double) + 15) / 16) * 16;
    }
    s_gat = reinterpret_cast<double2*>(p);
  }
  __syncthreads();
  for (int q = 0; q < nl; ++q) {
    const TailLevel& L = T[q];
    const int n = (L.r1 - L.r0) * L.g.nx;
    const double* kg = Ls[lt + q].k + (size_t)L.r0 * L.g.nx;
    for (int p = threadIdx.x; p < n; p += blockDim.x) L.k[p] = kg[p];
  }
  {
    const TailLevel& L = T[0];
    const int n = (L.r1 - L.r0) * L.g.nx;
    const double2* fg = fin + (size_t)L.r0 * L.g.nx;
    for (int p = threadIdx.x; p < n; p += blockDim.x) L.f[p] = cscale(fsc, fg[p]);
  }
  cl.sync();
  // ---- down
  for (int q = 0; q < nl - 1; ++q) {
    const TailLevel L = T[q];
    const TailLevel G = T[q + 1];
    const int nx = L.g.nx;
    const int n = (L.r1 - L.r0) * nx;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
      const int i = p % nx, j = L.r0 + p / nx;
      const Coef c = coef_at(L.g, i, j, L.k[p], sr, si);
      L.s[p] = cscale(omega, cdiv(L.f[p], c.ap));
    }
    cl.sync();
    double2* cur = L.s;
    for (int sw = 1; sw < nu_pre; ++sw) {
      double2* nxt = (cur == L.s) ? L.t : L.s;
      tail_jacobi(cl, L, cur, L.f, nxt, sr, si, omega, rank);
      cl.sync();
      cur = nxt;
    }
    double2* rb = (cur == L.s) ? L.t : L.s;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
      const int i = p % nx, j = L.r0 + p / nx;
      const Coef c = coef_at(L.g, i, j, L.k[p], sr, si);
      rb[p] = csub(L.f[p], tail_stencil(cl, L, cur, i, j, rank, c));
    }
    cl.sync();
    const int ncx = G.g.nx;
    const int nc = (G.r1 - G.r0) * ncx;
    for (int P = threadIdx.x; P < nc; P += blockDim.x) {
      const int I = P % ncx, J = G.r0 + P / ncx;
      const int ci = 2 * I + L.o, cj = 2 * J + L.o;
      double2 s = czero();
      for (int b = -1; b <= 1; ++b) {
        const int jj = cj + b;
        if (jj < 0 || jj >= L.g.ny) continue;
        const double2* rowp = tail_at(cl, L, rb, 0, jj, rank);
        for (int a = -1; a <= 1; ++a) {
          const int ii = ci + a;
          if (ii < 0 || ii >= nx) continue;
          const double w = (a == 0 ? 2.0 : 1.0) * (b == 0 ? 2.0 : 1.0) * (1.0 / 16.0);
          s = cadd(s, cscale(w, rowp[ii]));
        }
      }
      G.f[P] = s;
    }
    if (threadIdx.x == 0) curi[q] = (cur == L.s) ? 0 : 1;
    cl.sync();
  }
  // ---- coarsest: dense inverse (reading R8), one warp per owned row; the rhs is first gathered
  // from the cluster into this CTA's shared memory (one distributed-shared-memory pass)
  {
    const TailLevel Cl = T[nl - 1];
    const int n = Cl.g.nx * Cl.g.ny;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int rb0 = Cl.r0 * Cl.g.nx, rb1 = Cl.r1 * Cl.g.nx;
    double2* fl = s_gat;
    for (int c = threadIdx.x; c < n; c += blockDim.x) fl[c] = *tail_at(cl, Cl, Cl.f, c % Cl.g.nx, c / Cl.g.nx, rank);
    __syncthreads();
    for (int r = rb0 + warp; r < rb1; r += nw) {
      double2 s = czero();
      const double2* __restrict__ mrow = Minv + (size_t)r * n;
#pragma unroll 4
      for (int c = lane; c < n; c += 32) s = cfma(mrow[c], fl[c], s);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, off);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
      }
      if (lane == 0) {
        if (nl == 1) uout[r] = addq ? cadd(s, addq[r]) : s;
        else Cl.u[r - rb0] = s;
      }
    }
    cl.sync();
  }
  // ---- up
  for (int q = nl - 2; q >= 0; --q) {
    const TailLevel L = T[q];
    const TailLevel G = T[q + 1];
    const bool top = (q == 0);
    double2* cur = curi[q] ? L.t : L.s;
    double2* ob = curi[q] ? L.s : L.t;
    const int nx = L.g.nx;
    const int n = (L.r1 - L.r0) * nx;
    double2* u1 = (nu_post == 0) ? L.u : ob;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
      const int i = p % nx, j = L.r0 + p / nx;
      const int ri = i - L.o, rj = j - L.o;
      const int Ia = floordiv2(ri), Ja = floordiv2(rj);
      const bool ox = (ri & 1) != 0, oy = (rj & 1) != 0;
      double2 s = czero();
      for (int bj = 0; bj <= (oy ? 1 : 0); ++bj) {
        const int J = Ja + bj;
        if (J < 0 || J >= G.g.ny) continue;
        const double wy = oy ? 0.5 : 1.0;
        const double2* crow = tail_at(cl, G, G.u, 0, J, rank);
        for (int ai = 0; ai <= (ox ? 1 : 0); ++ai) {
          const int I = Ia + ai;
          if (I < 0 || I >= G.g.nx) continue;
          const double wx = ox ? 0.5 : 1.0;
          s = cadd(s, cscale(wx * wy, crow[I]));
        }
      }
      u1[p] = cadd(s, cur[p]);
    }
    cl.sync();
    double2* src = u1;
    for (int sw = 0; sw < nu_post; ++sw) {
      double2* dst = (sw == nu_post - 1) ? L.u : ((src == ob) ? cur : ob);
      tail_jacobi(cl, L, src, L.f, dst, sr, si, omega, rank);
      cl.sync();
      src = dst;
    }
    if (top) {
      double2* ug = uout + (size_t)L.r0 * nx;
      const double2* qg = addq ? addq + (size_t)L.r0 * nx : nullptr;
      for (int p = threadIdx.x; p < n; p += blockDim.x) ug[p] = qg ? cadd(L.u[p], qg[p]) : L.u[p];
    }
  }
}

}  // namespace helm
