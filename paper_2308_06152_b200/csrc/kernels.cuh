// Device kernels of the B200 (sm_100a) hot path.  complex128 is stored as interleaved
// double2 (re, im); grids are row-major a[j*nx + i] (x contiguous), the (i, j) grid
// ordering of PAPER.md §4.  Every kernel here is bandwidth-bound stencil / BLAS-1 work:
// no tensor cores.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace helm {

// Programmatic dependent launch (PDL): every kernel first waits until the grids it depends on
// have completed and their writes are visible (a no-op when launched without the attribute),
// then lets its own dependents be scheduled (they block in the same wait until this grid ends).
#define HELM_PDL_ENTRY()                                      \
  do {                                                        \
    asm volatile("griddepcontrol.wait;" ::: "memory");        \
    asm volatile("griddepcontrol.launch_dependents;" :::);    \
  } while (0)

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
// conj(a) * b
__device__ __forceinline__ double2 cconjmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}
__device__ __forceinline__ double cdiv_den(double2 b) { return 1.0 / fma(b.x, b.x, b.y * b.y); }
// a / b with d = cdiv_den(b) computed beforehand (the same operations as cdiv)
__device__ __forceinline__ double2 cdiv_d(double2 a, double2 b, double d) {
  return make_double2(fma(a.x, b.x, a.y * b.y) * d, fma(a.y, b.x, -a.x * b.y) * d);
}
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) { return cdiv_d(a, b, cdiv_den(b)); }
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // a*b + c
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

enum { BC_DIRICHLET = 0, BC_SOMMERFELD = 1 };

// A field pointer that may be indexed by a device-resident counter: address = p + (*idx) * stride.
// Krylov kernels captured once into a CUDA graph read the current basis slot (V[j], Z[j]) this
// way, so one graph serves every iteration of the device-controlled FGMRES loop.
// An optional device-resident scale `sc` is applied by the kernels that read the field through
// it (value = *sc * p[i]): the FGMRES basis vector v~_{j+1} = w'/||w'|| is consumed without a
// separate normalisation pass.
struct DVec {
  double2* p;
  const int* idx;
  long long stride;
  const double* sc;
  __host__ __device__ DVec(double2* p_ = nullptr) : p(p_), idx(nullptr), stride(0), sc(nullptr) {}
  __host__ __device__ DVec(const double2* p_) : p(const_cast<double2*>(p_)), idx(nullptr), stride(0), sc(nullptr) {}
  __host__ __device__ DVec(double2* p_, const int* i, long long s, const double* scale = nullptr)
      : p(p_), idx(i), stride(s), sc(scale) {}
  __device__ __forceinline__ double2* get() const { return idx ? p + (long long)(*idx) * stride : p; }
  __device__ __forceinline__ double scale() const { return sc ? *sc : 1.0; }
};


// Geometry of one grid level.
struct Geo {
  int nx, ny;
  double h;
  int bc;
};

// Multipliers of PAPER.md Algorithm 2 at unknown (i, j) for the operator
//   -Delta_h - s I(k^2),  s = sr + i si   (s = 1: A_h, Eq. 2.7; s = beta: CSLP M_h, Eq. 3.1)
// with Dirichlet (zero boundary neighbours) or first-order Sommerfeld ghost elimination
// (Eq. 2.8-2.10: outward multiplier 0, inward -2/h^2, centre -2ik/h per boundary side).
struct Coef {
  double2 ap;
  double aw, ae, as, an;
};

__device__ __forceinline__ Coef coef_at(const Geo& g, int i, int j, double kk, double sr, double si) {
  const double ih2 = 1.0 / (g.h * g.h);
  Coef c;
  const double k2 = kk * kk;
  c.ap = make_double2(4.0 * ih2 - sr * k2, -si * k2);
  c.aw = (i > 0) ? -ih2 : 0.0;
  c.ae = (i < g.nx - 1) ? -ih2 : 0.0;
  c.as = (j > 0) ? -ih2 : 0.0;
  c.an = (j < g.ny - 1) ? -ih2 : 0.0;
  if (g.bc == BC_SOMMERFELD) {
    const double t = 2.0 * kk / g.h;
    if (i == 0)        { c.ae = -2.0 * ih2; c.ap.y -= t; }
    if (i == g.nx - 1) { c.aw = -2.0 * ih2; c.ap.y -= t; }
    if (j == 0)        { c.an = -2.0 * ih2; c.ap.y -= t; }
    if (j == g.ny - 1) { c.as = -2.0 * ih2; c.ap.y -= t; }
  }
  return c;
}

__device__ __forceinline__ double2 stencil_apply(const Geo& g, const double2* __restrict__ u, int i, int j,
                                                 const Coef& c) {
  const size_t p = (size_t)j * g.nx + i;
  double2 v = cmul(c.ap, u[p]);
  if (c.aw != 0.0) v = cadd(v, cscale(c.aw, u[p - 1]));
  if (c.ae != 0.0) v = cadd(v, cscale(c.ae, u[p + 1]));
  if (c.as != 0.0) v = cadd(v, cscale(c.as, u[p - g.nx]));
  if (c.an != 0.0) v = cadd(v, cscale(c.an, u[p + g.nx]));
  return v;
}

// ------------------------------------------------------------------ operator kernels
// mode 0: y = Op u ;  mode 1: y = f - Op u (residual).  Linear indexing: each warp touches
// 512 contiguous, 512-byte-aligned bytes of u, k and y (rows of odd length would misalign a
// 2D tiling); the y-neighbours u[p -+ nx] come from L2 (the rows are re-read by the CTAs of
// the adjacent rows shortly after), so HBM sees u, k and y once: 40 (56) B per unknown.
template <int MODE>
__global__ void __launch_bounds__(256) k_apply_op(Geo g, DVec uv, DVec fv, DVec yv, const double* __restrict__ k,
                                                  double sr, double si) {
  HELM_PDL_ENTRY();
  const unsigned n = (unsigned)g.nx * (unsigned)g.ny;
  const unsigned p = blockIdx.x * 256u + threadIdx.x;
  if (p >= n) return;
  const double2* __restrict__ u = uv.get();
  const double2* __restrict__ f = fv.get();
  double2* __restrict__ y = yv.get();
  const int j = (int)(p / (unsigned)g.nx);
  const int i = (int)(p - (unsigned)j * (unsigned)g.nx);
  const double kk = k[p];
  double2 v;
  if (i > 0 && i < g.nx - 1 && j > 0 && j < g.ny - 1) {
    // interior: constant off-diagonal multipliers, no boundary branches (same operation order)
    const double ih2 = 1.0 / (g.h * g.h);
    const double k2 = kk * kk;
    v = cmul(make_double2(4.0 * ih2 - sr * k2, -si * k2), u[p]);
    v = cadd(v, cscale(-ih2, u[p - 1]));
    v = cadd(v, cscale(-ih2, u[p + 1]));
    v = cadd(v, cscale(-ih2, u[p - g.nx]));
    v = cadd(v, cscale(-ih2, u[p + g.nx]));
  } else {
    const Coef c = coef_at(g, i, j, kk, sr, si);
    v = stencil_apply(g, u, i, j, c);
  }
  if (MODE == 1) v = csub(cscale(fv.scale(), f[p]), v);
  y[p] = v;
}

// u = omega * f / D   (first damped-Jacobi sweep from u = 0)
__global__ void k_jacobi0(Geo g, DVec fv, double2* __restrict__ u,
                          const double* __restrict__ k, double sr, double si, double omega) {
  HELM_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.nx || j >= g.ny) return;
  const double2* __restrict__ f = fv.get();
  const size_t p = (size_t)j * g.nx + i;
  Coef c = coef_at(g, i, j, k[p], sr, si);
  u[p] = cscale(omega, cdiv(cscale(fv.scale(), f[p]), c.ap));
}

// unew = u + omega * (f - M u) / D  (+ optional add of `q`, used to fuse z = M^-1 t + q)
__global__ void k_jacobi(Geo g, const double2* __restrict__ u, DVec fv,
                         DVec unewv, const double* __restrict__ k, double sr, double si,
                         double omega, const double2* __restrict__ addq) {
  HELM_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.nx || j >= g.ny) return;
  const double2* __restrict__ f = fv.get();
  double2* __restrict__ unew = unewv.get();
  const size_t p = (size_t)j * g.nx + i;
  Coef c = coef_at(g, i, j, k[p], sr, si);
  double2 r = csub(cscale(fv.scale(), f[p]), stencil_apply(g, u, i, j, c));
  double2 v = cadd(u[p], cscale(omega, cdiv(r, c.ap)));
  if (addq) v = cadd(v, addq[p]);
  unew[p] = v;
}

// Full weighting (Eq. 3.8), gather at fine node (2I+o, 2J+o); out-of-array taps dropped.
__global__ void k_restrict(Geo gf, Geo gc, int o, const double2* __restrict__ v, double2* __restrict__ vc) {
  HELM_PDL_ENTRY();
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  const int J = blockIdx.y * blockDim.y + threadIdx.y;
  if (I >= gc.nx || J >= gc.ny) return;
  const int ci = 2 * I + o, cj = 2 * J + o;
  double2 s = make_double2(0.0, 0.0);
#pragma unroll
  for (int b = -1; b <= 1; ++b) {
    const int jj = cj + b;
    if (jj < 0 || jj >= gf.ny) continue;
#pragma unroll
    for (int a = -1; a <= 1; ++a) {
      const int ii = ci + a;
      if (ii < 0 || ii >= gf.nx) continue;
      const double w = (a == 0 ? 2.0 : 1.0) * (b == 0 ? 2.0 : 1.0) * (1.0 / 16.0);
      s = cadd(s, cscale(w, v[(size_t)jj * gf.nx + ii]));
    }
  }
  vc[(size_t)J * gc.nx + I] = s;
}

// Bilinear interpolation (Eq. 3.9) as a gather at each fine node:
//   y = P e  (MODE 0)  or  y = base + P e  (MODE 1)
template <int MODE>
__global__ void k_prolong(Geo gf, Geo gc, int o, const double2* __restrict__ e, const double2* __restrict__ base,
                          DVec yv, const double2* __restrict__ addq) {
  HELM_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= gf.nx || j >= gf.ny) return;
  const int ri = i - o, rj = j - o;           // position relative to coarse node 0
  // coarse candidates: I0 = floor(ri/2) and I0+1 when ri is odd
  double2 s = make_double2(0.0, 0.0);
  const int I0 = (ri >= 0) ? (ri >> 1) : -1;   // ri = -1 only for Dirichlet i = 0
  const int J0 = (rj >= 0) ? (rj >> 1) : -1;
  const bool oddx = (ri & 1) != 0, oddy = (rj & 1) != 0;
  for (int bj = 0; bj <= (oddy ? 1 : 0); ++bj) {
    const int J = J0 + bj;
    if (J < 0 || J >= gc.ny) continue;
    const double wy = oddy ? 0.5 : 1.0;
    for (int ai = 0; ai <= (oddx ? 1 : 0); ++ai) {
      const int I = I0 + ai;
      if (I < 0 || I >= gc.nx) continue;
      const double wx = oddx ? 0.5 : 1.0;
      s = cadd(s, cscale(wx * wy, e[(size_t)J * gc.nx + I]));
    }
  }
  const size_t p = (size_t)j * gf.nx + i;
  if (MODE == 1) s = cadd(s, base[p]);
  if (addq) s = cadd(s, addq[p]);
  yv.get()[p] = s;
}

// Coarse wavenumber sampled at coincident fine nodes (re-discretisation, §5.1).
__global__ void k_sample_k(Geo gf, Geo gc, int o, const double* __restrict__ kf, double* __restrict__ kc) {
  HELM_PDL_ENTRY();
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  const int J = blockIdx.y * blockDim.y + threadIdx.y;
  if (I >= gc.nx || J >= gc.ny) return;
  kc[(size_t)J * gc.nx + I] = kf[(size_t)(2 * J + o) * gf.nx + (2 * I + o)];
}

// ------------------------------------------------------------------ deflation vectors Z, Z^T
// 1D weight of coarse node c at fine node 2c + o + d (a column of Z):
//   bilinear (R = 1): Eq. 3.6/3.9      w(0) = 1,   w(+-1) = 1/2
//   high order (R = 2): Eq. 3.11a/3.12 w(0) = 3/4, w(+-1) = 1/2, w(+-2) = 1/8
// The deflation restriction is Z^T for both (Eq. 3.7 per direction / Eq. 3.14; reading R10) --
// 4x the 1/16-normalised full weighting the V-cycle uses for the bilinear vectors.
template <int R>
__device__ __forceinline__ double zw(int d) {
  if (R == 1) return d == 0 ? 1.0 : ((d == 1 || d == -1) ? 0.5 : 0.0);
  return d == 0 ? 0.75 : ((d == 1 || d == -1) ? 0.5 : ((d == 2 || d == -2) ? 0.125 : 0.0));
}

// vc = Z^T v  (gather of the (2R+1)^2 fine taps; out-of-array taps dropped, reading R4)
template <int R>
__global__ void k_restrict_z(Geo gf, Geo gc, int o, DVec vv, double2* __restrict__ vc) {
  HELM_PDL_ENTRY();
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  const int J = blockIdx.y * blockDim.y + threadIdx.y;
  if (I >= gc.nx || J >= gc.ny) return;
  const double2* __restrict__ v = vv.get();
  const double vs = vv.scale();
  const int ci = 2 * I + o, cj = 2 * J + o;
  double2 s = make_double2(0.0, 0.0);
#pragma unroll
  for (int b = -R; b <= R; ++b) {
    const int jj = cj + b;
    if (jj < 0 || jj >= gf.ny) continue;
    const double wy = zw<R>(b);
#pragma unroll
    for (int a = -R; a <= R; ++a) {
      const int ii = ci + a;
      if (ii < 0 || ii >= gf.nx) continue;
      s = cadd(s, cscale(wy * zw<R>(a), v[(size_t)jj * gf.nx + ii]));
    }
  }
  vc[(size_t)J * gc.nx + I] = cscale(vs, s);
}

// y = Z e (MODE 0) or y = base + Z e (MODE 1), gather at each fine node.
template <int R, int MODE>
__global__ void k_prolong_z(Geo gf, Geo gc, int o, const double2* __restrict__ e, const double2* __restrict__ base,
                            double2* __restrict__ y) {
  HELM_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= gf.nx || j >= gf.ny) return;
  const int ri = i - o, rj = j - o;
  // coarse nodes c with |ri - 2c| <= R  ->  c in [ceil((ri-R)/2), floor((ri+R)/2)]
  const int clo = (ri - R + 1 + 2 * 64) / 2 - 64, chi = (ri + R + 2 * 64) / 2 - 64;
  const int rlo = (rj - R + 1 + 2 * 64) / 2 - 64, rhi = (rj + R + 2 * 64) / 2 - 64;
  double2 s = make_double2(0.0, 0.0);
  for (int J = max(rlo, 0); J <= min(rhi, gc.ny - 1); ++J) {
    const double wy = zw<R>(rj - 2 * J);
    for (int I = max(clo, 0); I <= min(chi, gc.nx - 1); ++I)
      s = cadd(s, cscale(wy * zw<R>(ri - 2 * I), e[(size_t)J * gc.nx + I]));
  }
  const size_t p = (size_t)j * gf.nx + i;
  if (MODE == 1) s = cadd(s, base[p]);
  y[p] = s;
}

// ------------------------------------------------------------------ Galerkin coarse operator
// y = E x = Z^T A Z x (§3.2.1 "A_{2h} = I_h^{2h} A_h I_{2h}^h"; str-Glk §5.2.1,
// Eq. 5.7a-c: interpolation, fine-grid operator, restriction) applied matrix-free in ONE kernel:
// for a tile of TCX x TCY coarse outputs, x (coarse, with halo) -> t = Z x on the fine footprint
// plus one node -> s = A t on the footprint -> y = Z^T s, all in shared memory.  HBM traffic
// per coarse unknown: x 16 + k 4 x 8 + y 16 B (the paper's three passes, or a stored 25-point
// stencil, would move ~10x more).  MODE 1: y = f - E x.
__device__ __forceinline__ int ceildiv2(int a) { return (a >= 0) ? ((a + 1) >> 1) : -((-a) >> 1); }

__device__ __forceinline__ int floordiv2i(int a) { return (a >= 0) ? (a >> 1) : -((-a + 1) >> 1); }

// 1D interpolation of a coarse line at relative fine position r = fine - o (taps at coarse
// floor(r/2) - 1 .. floor(r/2) + 2 with the weights zw<R>; zero weights skipped at compile time
// of the unrolled loop).  `at(I)` returns the coarse value (0 outside the array).
template <int R, class At>
__device__ __forceinline__ double2 interp1(int r, At&& at) {
  const int Ib = floordiv2i(r);
  double2 s = make_double2(0.0, 0.0);
#pragma unroll
  for (int d = -1; d <= 2; ++d) {
    const double w = zw<R>(r - 2 * (Ib + d));
    if (w != 0.0) s = cadd(s, cscale(w, at(Ib + d)));
  }
  return s;
}

// 1D interpolation weights at relative fine position r (coarse taps floor(r/2) - 1, +0, +1):
// even r: (1/8, 3/4, 1/8) higher order, (0, 1, 0) bilinear; odd r: (0, 1/2, 1/2) both.
template <int R>
__device__ __forceinline__ void interp_w(int r, double& wm, double& w0, double& wp) {
  const bool odd = (r & 1) != 0;
  wm = odd ? 0.0 : (R == 2 ? 0.125 : 0.0);
  w0 = odd ? 0.5 : (R == 2 ? 0.75 : 1.0);
  wp = odd ? 0.5 : (R == 2 ? 0.125 : 0.0);
}

// Block = 32 x 8 threads.
// DOTS (MODE 0, inner FGMRES): the tile also runs pass 1 of the delayed CGS2 for its coarse
// points -- part[(2c) T + tile] = sum conj(V_c) (s v~_j), part[(2c+1) T + tile] = sum conj(V_c) w
// for c <= j, with V_j read as s v~_j (T tiles; w = E x is this tile's output) -- so the E output
// is dotted while it is still on chip and the separate dots kernel disappears from the iteration.
#ifndef HELM_GLKD_MINB   // DOTS variant: 3 CTAs/SM (80 registers, no spills) measured best
#define HELM_GLKD_MINB 3
#endif
template <int R, int MODE, int TCX, int TCY, bool DOTS = false>
__global__ void __launch_bounds__(256, DOTS ? HELM_GLKD_MINB : 6) k_galerkin_apply(Geo gf, Geo gc, int o, const double* __restrict__ kf, DVec xv,
                                                        DVec fv, DVec yv, const double2* __restrict__ V = nullptr,
                                                        long long ldv = 0, const int* __restrict__ jptr = nullptr,
                                                        DVec vt = DVec(), double2* __restrict__ part = nullptr) {
  HELM_PDL_ENTRY();
  constexpr int SX = 2 * TCX - 1 + 2 * R, SY = 2 * TCY - 1 + 2 * R;   // s = A t region (fine)
  constexpr int TXR = SX + 2, TYR = SY + 2;                          // t = Z x region (A halo)
  constexpr int CXW = TCX + 2 * R + 2, CYW = TCY + 2 * R + 2;         // coarse x region (+1 pad each side)
  constexpr int TXN = CYW * TXR, SSN = SY * SX;
  __shared__ double2 sx[CYW * CXW];
  __shared__ double2 txss[TXN > SSN ? TXN : SSN];   // tx (x-interpolated coarse rows), later s = A t
  __shared__ double2 stt[TYR * TXR];               // t = Z x
  __shared__ double2 ry[TCY * SX];                 // s restricted along y
  __shared__ double2 wt[DOTS ? TCX * TCY : 1];     // DOTS: this tile's E x
  double2* const tx = txss;
  double2* const ss = txss;
  const int tx_ = threadIdx.x, ty_ = threadIdx.y;
  const double2* __restrict__ x = xv.get();
  const int I0 = blockIdx.x * TCX, J0 = blockIdx.y * TCY;
  const int fx0s = 2 * I0 + o - R, fy0s = 2 * J0 + o - R;
  const int fx0t = fx0s - 1, fy0t = fy0s - 1;
  const int cx0 = I0 - R - 1, cy0 = J0 - R - 1;   // coarse index of sx column / row 0
  const double2 zero = make_double2(0.0, 0.0);
  // every phase walks its region as one flat index over the CTA's 256 threads (constant row
  // widths: the division is a multiply-shift), so no lanes idle on the ragged region widths
  const int tid = ty_ * 32 + tx_;
  for (int q = tid; q < CYW * CXW; q += 256) {
    const int r = q / CXW, c = q - r * CXW;
    const int J = cy0 + r, I = cx0 + c;
    sx[q] = (J >= 0 && J < gc.ny && I >= 0 && I < gc.nx) ? x[(size_t)J * gc.nx + I] : zero;
  }
  __syncthreads();
  // Z = tensor product of the 1D interpolations (Eq. 3.9 / 3.12): along x ...
  for (int q = tid; q < CYW * TXR; q += 256) {
    const int r = q / TXR, c = q - r * TXR;
    const int fx = fx0t + c;
    const int rr = fx - o;
    const int li = floordiv2i(rr) - cx0;
    double wm, w0, wp;
    interp_w<R>(rr, wm, w0, wp);
    if (fx < 0 || fx >= gf.nx) wm = w0 = wp = 0.0;
    const double2* line = sx + r * CXW + li;
    tx[q] = cadd(cadd(cscale(wm, line[-1]), cscale(w0, line[0])), cscale(wp, line[1]));
  }
  __syncthreads();
  // ... then along y
  for (int q = tid; q < TYR * TXR; q += 256) {
    const int r = q / TXR, c = q - r * TXR;
    const int fy = fy0t + r;
    const int rr = fy - o;
    const int lj = floordiv2i(rr) - cy0;
    double wm, w0, wp;
    interp_w<R>(rr, wm, w0, wp);
    if (fy < 0 || fy >= gf.ny) wm = w0 = wp = 0.0;
    stt[q] = cadd(cadd(cscale(wm, tx[(lj - 1) * TXR + c]), cscale(w0, tx[lj * TXR + c])),
                  cscale(wp, tx[(lj + 1) * TXR + c]));
  }
  __syncthreads();
  for (int q = tid; q < SY * SX; q += 256) {
    const int r = q / SX, c = q - r * SX;
    const int fy = fy0s + r, fx = fx0s + c;
    double2 v = zero;   // reading R4: restriction taps outside the array dropped
    if (fx >= 0 && fx < gf.nx && fy >= 0 && fy < gf.ny) {
      const Coef cf = coef_at(gf, fx, fy, kf[(size_t)fy * gf.nx + fx], 1.0, 0.0);
      const int t = (r + 1) * TXR + (c + 1);
      v = cmul(cf.ap, stt[t]);
      if (cf.aw != 0.0) v = cadd(v, cscale(cf.aw, stt[t - 1]));
      if (cf.ae != 0.0) v = cadd(v, cscale(cf.ae, stt[t + 1]));
      if (cf.as != 0.0) v = cadd(v, cscale(cf.as, stt[t - TXR]));
      if (cf.an != 0.0) v = cadd(v, cscale(cf.an, stt[t + TXR]));
    }
    ss[q] = v;
  }
  __syncthreads();
  // Z^T = tensor product of the transposed 1D interpolations: along y ...
  for (int q = tid; q < TCY * SX; q += 256) {
    const int jl = q / SX, c = q - jl * SX;
    const int iy = 2 * jl + R;
    double2 v = zero;
#pragma unroll
    for (int b = -R; b <= R; ++b) v = cadd(v, cscale(zw<R>(b), ss[(iy + b) * SX + c]));
    ry[q] = v;
  }
  __syncthreads();
  // ... then along x
  const double2* __restrict__ f = fv.get();
  double2* __restrict__ y = yv.get();
  for (int q = tid; q < TCY * TCX; q += 256) {
    const int jl = q / TCX, il = q - jl * TCX;
    const int J = J0 + jl, I = I0 + il;
    if (I >= gc.nx || J >= gc.ny) continue;
    const int ix = 2 * il + R;
    double2 s = zero;
#pragma unroll
    for (int a = -R; a <= R; ++a) s = cadd(s, cscale(zw<R>(a), ry[jl * SX + ix + a]));
    const size_t p = (size_t)J * gc.nx + I;
    y[p] = (MODE == 1) ? csub(cscale(fv.scale(), f[p]), s) : s;
    if (DOTS) wt[q] = s;
  }
  if (DOTS) {
    static_assert(TCX * TCY == 128, "pass-1 dots map 4 coarse points to each lane");
    __syncthreads();
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = (blockDim.x * blockDim.y) >> 5;
    const int ntiles = gridDim.x * gridDim.y, tile = blockIdx.y * gridDim.x + blockIdx.x;
    const int j = *jptr;
    const double2* __restrict__ xt = vt.get();
    const double xsc = vt.scale();
    double2 xr[4], wr[4];
    long long pp[4];
    bool ok[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int q = lane + 32 * r;
      const int I = I0 + q % TCX, J = J0 + q / TCX;
      ok[r] = I < gc.nx && J < gc.ny;
      pp[r] = ok[r] ? (long long)J * gc.nx + I : 0;
      xr[r] = ok[r] ? cscale(xsc, xt[pp[r]]) : zero;
      wr[r] = ok[r] ? wt[q] : zero;
    }
#pragma unroll 2
    for (int c = warp; c <= j; c += nwarps) {
      const double2* __restrict__ vc = V + (long long)c * ldv;
      double2 v[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) v[r] = ok[r] ? vc[pp[r]] : zero;
      double2 ax = zero, aw = zero;
#pragma unroll
      for (int r = 0; r < 4; ++r) {   // conj(v) x, conj(v) w
        ax.x = fma(v[r].x, xr[r].x, fma(v[r].y, xr[r].y, ax.x));
        ax.y = fma(v[r].x, xr[r].y, fma(-v[r].y, xr[r].x, ax.y));
        aw.x = fma(v[r].x, wr[r].x, fma(v[r].y, wr[r].y, aw.x));
        aw.y = fma(v[r].x, wr[r].y, fma(-v[r].y, wr[r].x, aw.y));
      }
#pragma unroll
      for (int sh = 16; sh > 0; sh >>= 1) {
        ax.x += __shfl_xor_sync(0xffffffffu, ax.x, sh);
        ax.y += __shfl_xor_sync(0xffffffffu, ax.y, sh);
        aw.x += __shfl_xor_sync(0xffffffffu, aw.x, sh);
        aw.y += __shfl_xor_sync(0xffffffffu, aw.y, sh);
      }
      if (c == j) {   // V_j is v~_j itself: read through the same scale as x (as k_dcgs_dots)
        ax = cscale(xsc, ax);
        aw = cscale(xsc, aw);
      }
      if (lane == 0) {
        part[(long long)(2 * c) * ntiles + tile] = ax;
        part[(long long)(2 * c + 1) * ntiles + tile] = aw;
      }
    }
  }
}

// ------------------------------------------------------------------ str-Glk E by column streaming
// The same y = Z^T A Z x (or f - E x) as k_galerkin_apply, with the same arithmetic (x-then-y
// interpolation, A with its zero multipliers skipped, Z^T along y then x, every sum in the same
// order from zero; results differ only where the compiler contracts a different mul/add pair
// into an FMA, ~1e-16), but the intermediate fine fields live in registers instead of
// shared memory: the tile kernel measured shared-memory bound (L1/TEX pipe 78 % busy, DRAM 7 %,
// ~98 16-byte shared accesses per coarse unknown; ncu, 1023^2 coarse grid).
// A warp owns 32 consecutive coarse columns I = I0 - 2 + lane (lane L: fine columns
// fe = 2I + o and fd = fe + 1) and writes the 28 outputs of lanes 2..29; x-neighbours come
// by warp shuffles, y-neighbours from the last rows kept in registers.  The warp walks a
// segment of S coarse output rows [J0, J1) from row J0 - 2 (4 rows of warm-up: step J loads
// x row J + 1, forms t on fine rows fe(J) = 2J + o and fd(J), s = A t on rows fd(J - 1) and
// fe(J), adds them into the Z^T-along-y sums of output rows J - 1, J, J + 1 and completes row
// J - 1).  Loads of the next step are issued before the current step's arithmetic.
#ifndef HELM_GLKS_MINB   // resident 128-thread blocks per SM the register cap aims at
#define HELM_GLKS_MINB 4
#endif
// residual mode (the s-step powers): 3 blocks per SM -- no spills (at 4 it spilled ~100 B per
// thread), 34.2 -> 32.0 us per apply on the 1023^2 level; plain mode keeps 4 (28.5 vs 29.7 us)
#ifndef HELM_GLKS_MINB_RES
#define HELM_GLKS_MINB_RES 3
#endif
#ifndef HELM_GLKS_FAST_UNROLL   // unroll of the interior-step loop (probe knob)
#define HELM_GLKS_FAST_UNROLL 2   // 22.3 vs 22.9 us (1), 22.5 (3), 23.0 (6) in residual mode
#endif
#define HELM_STR2(x) #x
#define HELM_PRAGMA_UNROLL(n) _Pragma(HELM_STR2(unroll n))
template <int R, int MODE>
__global__ void __launch_bounds__(128, MODE == 1 ? HELM_GLKS_MINB_RES : HELM_GLKS_MINB) k_glk_stream(Geo gf, Geo gc, int o, const double* __restrict__ kf, DVec xv,
                                                    DVec fv, DVec yv, int S, int nbands) {
  HELM_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int band = gw % nbands, seg = gw / nbands;
  const int J0 = seg * S;
  if (J0 >= gc.ny) return;   // whole warp
  const int J1 = min(gc.ny, J0 + S);
  const int I = band * 28 - 2 + lane;
  const bool xin = I >= 0 && I < gc.nx;
  const int fe = 2 * I + o, fd = fe + 1;
  const bool ein = fe >= 0 && fe < gf.nx, din = fd >= 0 && fd < gf.nx;
  const double2* __restrict__ x = xv.get();
  const double2 zero = make_double2(0.0, 0.0);
  const double wm_e = R == 2 ? 0.125 : 0.0, w0_e = R == 2 ? 0.75 : 1.0, wp_e = R == 2 ? 0.125 : 0.0;
  auto shup = [&](double2 v) {
    return make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
  };
  auto shdn = [&](double2 v) {
    return make_double2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
  };
  auto load_x = [&](int J) { return (xin && J >= 0 && J < gc.ny) ? x[(size_t)J * gc.nx + I] : zero; };
  auto row_in = [&](int fy) { return fy >= 0 && fy < gf.ny; };
  auto load_k = [&](int fy, int fx, bool in) { return (in && row_in(fy)) ? kf[(size_t)fy * gf.nx + fx] : 0.0; };
  // x-interpolated coarse row (t before the y interpolation) at this lane's two fine columns
  struct TX { double2 e, d; };
  auto xinterp = [&](double2 xs, auto allinc) {
    constexpr bool AI = decltype(allinc)::value;
    const double2 xm = shup(xs), xp = shdn(xs);
    TX t;
    // even relative column: taps I-1, I, I+1 (1/8, 3/4, 1/8 | 0, 1, 0); odd: I, I+1 (1/2, 1/2)
    // (zero weights dropped: the odd column is 0.5 (x_I + x_{I+1}); bilinear even = x_I)
    t.e = (AI || ein) ? (R == 2 ? cadd(cadd(cscale(wm_e, xm), cscale(w0_e, xs)), cscale(wp_e, xp)) : xs) : zero;
    t.d = (AI || din) ? cscale(0.5, cadd(xs, xp)) : zero;
    return t;
  };
  // s = A t at fine row fy for both columns; c = centre row, sth / nth = the rows below / above.
  // Interior rows of an interior band take constant off-diagonal multipliers (coef_at's values,
  // same operation order, no boundary branches).
  const double ih2 = 1.0 / (gf.h * gf.h);
  const bool band_int = __all_sync(0xffffffffu, fe >= 1 && fd <= gf.nx - 2);
  auto apply_A_row = [&](int fy, const TX& sth, const TX& c, const TX& nth, double ke, double kd, TX& s) {
    const double2 west_e = shup(c.d), east_d = shdn(c.e);
    if (band_int && fy >= 1 && fy <= gf.ny - 2) {
      // A = -Delta_h - k^2 (real centre 4/h^2 - k^2, neighbours -1/h^2): 2 + 2 multiplies
      const double ape = 4.0 * ih2 - ke * ke, apd = 4.0 * ih2 - kd * kd;
      const double2 ne = cadd(cadd(west_e, c.d), cadd(sth.e, nth.e));
      const double2 nd = cadd(cadd(c.e, east_d), cadd(sth.d, nth.d));
      s.e = make_double2(fma(ape, c.e.x, -ih2 * ne.x), fma(ape, c.e.y, -ih2 * ne.y));
      s.d = make_double2(fma(apd, c.d.x, -ih2 * nd.x), fma(apd, c.d.y, -ih2 * nd.y));
      return;
    }
    s.e = zero;
    s.d = zero;
    if (!row_in(fy)) return;
    if (ein) {
      const Coef cf = coef_at(gf, fe, fy, ke, 1.0, 0.0);
      double2 v = cmul(cf.ap, c.e);
      if (cf.aw != 0.0) v = cadd(v, cscale(cf.aw, west_e));
      if (cf.ae != 0.0) v = cadd(v, cscale(cf.ae, c.d));
      if (cf.as != 0.0) v = cadd(v, cscale(cf.as, sth.e));
      if (cf.an != 0.0) v = cadd(v, cscale(cf.an, nth.e));
      s.e = v;
    }
    if (din) {
      const Coef cf = coef_at(gf, fd, fy, kd, 1.0, 0.0);
      double2 v = cmul(cf.ap, c.d);
      if (cf.aw != 0.0) v = cadd(v, cscale(cf.aw, c.e));
      if (cf.ae != 0.0) v = cadd(v, cscale(cf.ae, east_d));
      if (cf.as != 0.0) v = cadd(v, cscale(cf.as, sth.d));
      if (cf.an != 0.0) v = cadd(v, cscale(cf.an, nth.d));
      s.d = v;
    }
  };
  auto add = [&](TX& acc, double w, const TX& s) {
    acc.e = cadd(acc.e, cscale(w, s.e));
    acc.d = cadd(acc.d, cscale(w, s.d));
  };
  const double2* __restrict__ f = fv.get();
  const double fsc = MODE == 1 ? fv.scale() : 1.0;
  double2* __restrict__ y = yv.get();

  int J = J0 - 2;
  // state: tx(J-1), tx(J); t rows fe(J-1), fd(J-1); Z^T_y sums of output rows J-1, J, J+1
  TX txm = xinterp(load_x(J - 1), std::false_type()), tx0 = xinterp(load_x(J), std::false_type());
  const TX tz = {zero, zero};
  TX tfe_m = tz, tfd_m = tz;   // rows fe(J-1), fd(J-1): only feed rows before J0 - 1
  TX acc0 = tz, acc1 = tz, acc2 = tz;
  // loads of step J: x row J+1, k on rows fd(J-1) and fe(J)
  double2 xn = load_x(J + 1);
  double kfd_e = load_k(2 * J + o - 1, fe, ein), kfd_d = load_k(2 * J + o - 1, fd, din);
  double kfe_e = load_k(2 * J + o, fe, ein), kfe_d = load_k(2 * J + o, fd, din);
  // residual mode: f of the output row (J - 1) loaded one step ahead
  auto load_f = [&](int Jr) {
    return (MODE == 1 && xin && Jr >= J0 && Jr < J1) ? f[(size_t)Jr * gc.nx + I] : zero;
  };
  double2 fpre = load_f(J - 1);
  // Steps in [Ja, Jb) touch only rows inside both grids (x rows J-1 .. J+2, fine rows
  // 2J+o-1 .. 2J+o+2, output row J-1 < J1 -- stored if >= J0 --, f row J < J1): they run without
  // the row-range tests, with int offsets and A's interior form -- on interior bands (FAST 2) with
  // no lane tests either; on the edge bands of a Dirichlet grid (FAST 1), where every
  // multiplier of an in-grid fine node is the interior one and out-of-grid t values are zero,
  // with the lanes outside the fine grid masked to zero.  Each warp runs at most ~4 general
  // steps, so the one-wave grid stays balanced (Sommerfeld edge bands: general steps only).
  const bool simpleA = gf.bc == BC_DIRICHLET || band_int;
  const int Ja = max(J, 1);   // the warm-up steps (output rows < J0: not stored) run fast too
  const int Jb = simpleA ? max(Ja, min(J1, min(gc.ny - 2, (gf.ny - 3 - o) / 2 + 1))) : Ja;
  auto step = [&](const int J, auto fastc) {
    constexpr int FAST = decltype(fastc)::value;
    constexpr bool ALLIN = FAST == 2;   // every lane's I, fe, fd inside the grids
    const double2 xc = xn;
    const double2 fo = fpre;
    const double a_fd_e = kfd_e, a_fd_d = kfd_d, a_fe_e = kfe_e, a_fe_d = kfe_d;
    if (FAST) {
      if (MODE == 1) fpre = (ALLIN || xin) ? f[J * gc.nx + I] : zero;
      xn = (ALLIN || xin) ? x[(J + 2) * gc.nx + I] : zero;
      const int r1 = (2 * J + o + 1) * gf.nx;
      kfd_e = (ALLIN || ein) ? kf[r1 + fe] : 0.0;
      kfd_d = (ALLIN || din) ? kf[r1 + fd] : 0.0;
      kfe_e = (ALLIN || ein) ? kf[r1 + gf.nx + fe] : 0.0;
      kfe_d = (ALLIN || din) ? kf[r1 + gf.nx + fd] : 0.0;
    } else {
      if (MODE == 1) fpre = load_f(J);
      if (J < J1) {   // next step's loads, in flight during this step's arithmetic
        xn = load_x(J + 2);
        kfd_e = load_k(2 * J + o + 1, fe, ein);
        kfd_d = load_k(2 * J + o + 1, fd, din);
        kfe_e = load_k(2 * J + o + 2, fe, ein);
        kfe_d = load_k(2 * J + o + 2, fd, din);
      }
    }
    const TX txp = xinterp(xc, std::integral_constant<bool, ALLIN>());   // tx(J+1)
    // y interpolation: fine rows fe(J) (taps J-1, J, J+1) and fd(J) (taps J, J+1)
    TX tfe, tfd;
    const bool fe_row = FAST || row_in(2 * J + o), fd_row = FAST || row_in(2 * J + o + 1);
    tfe.e = fe_row ? (R == 2 ? cadd(cadd(cscale(wm_e, txm.e), cscale(w0_e, tx0.e)), cscale(wp_e, txp.e)) : tx0.e) : zero;
    tfe.d = fe_row ? (R == 2 ? cadd(cadd(cscale(wm_e, txm.d), cscale(w0_e, tx0.d)), cscale(wp_e, txp.d)) : tx0.d) : zero;
    tfd.e = fd_row ? cscale(0.5, cadd(tx0.e, txp.e)) : zero;
    tfd.d = fd_row ? cscale(0.5, cadd(tx0.d, txp.d)) : zero;
    // s = A t on rows fd(J-1) (south fe(J-1), north fe(J)) and fe(J) (south fd(J-1), north fd(J))
    TX s_fdm, s_fe;
    if (FAST) {
      auto fastA = [&](const TX& sth, const TX& c, const TX& nth, double ke, double kd, TX& s) {
        const double2 west_e = shup(c.d), east_d = shdn(c.e);
        const double ape = 4.0 * ih2 - ke * ke, apd = 4.0 * ih2 - kd * kd;
        const double2 ne = cadd(cadd(west_e, c.d), cadd(sth.e, nth.e));
        const double2 nd = cadd(cadd(c.e, east_d), cadd(sth.d, nth.d));
        s.e = make_double2(fma(ape, c.e.x, -ih2 * ne.x), fma(ape, c.e.y, -ih2 * ne.y));
        s.d = make_double2(fma(apd, c.d.x, -ih2 * nd.x), fma(apd, c.d.y, -ih2 * nd.y));
        if (!ALLIN) {   // Dirichlet edge band: no fine node outside the grid
          if (!ein) s.e = zero;
          if (!din) s.d = zero;
        }
      };
      fastA(tfe_m, tfd_m, tfe, a_fd_e, a_fd_d, s_fdm);
      fastA(tfd_m, tfe, tfd, a_fe_e, a_fe_d, s_fe);
    } else {
      apply_A_row(2 * J + o - 1, tfe_m, tfd_m, tfe, a_fd_e, a_fd_d, s_fdm);
      apply_A_row(2 * J + o, tfd_m, tfe, tfd, a_fe_e, a_fe_d, s_fe);
    }
    // Z^T along y, in increasing fine-row order per output row (b = -R .. R)
    add(acc0, zw<R>(1), s_fdm);   // output J-1: b = +1, +2
    if (R == 2) add(acc0, zw<R>(2), s_fe);
    add(acc1, zw<R>(-1), s_fdm);  // output J: b = -1, 0
    add(acc1, zw<R>(0), s_fe);
    if (R == 2) add(acc2, zw<R>(-2), s_fe);   // output J+1: b = -2
    // output row J-1 is complete: Z^T along x (a = -R .. R), lanes 2..29
    {
      const double2 em = shup(acc0.e), dm = shup(acc0.d), ep = shdn(acc0.e);
      const int Jo = J - 1;
      if ((FAST ? Jo >= J0 : (Jo >= J0 && Jo < J1)) && lane >= 2 && lane < 30 && (ALLIN || I < gc.nx)) {
        double2 sacc = zero;
        if (R == 2) sacc = cadd(sacc, cscale(zw<R>(-2), em));
        sacc = cadd(sacc, cscale(zw<R>(-1), dm));
        sacc = cadd(sacc, cscale(zw<R>(0), acc0.e));
        sacc = cadd(sacc, cscale(zw<R>(1), acc0.d));
        if (R == 2) sacc = cadd(sacc, cscale(zw<R>(2), ep));
        const size_t p = FAST ? (size_t)(Jo * gc.nx + I) : (size_t)Jo * gc.nx + I;
        y[p] = (MODE == 1) ? csub(cscale(fsc, fo), sacc) : sacc;
      }
    }
    acc0 = acc1;
    acc1 = acc2;
    acc2 = tz;
    txm = tx0;
    tx0 = txp;
    tfe_m = tfe;
    tfd_m = tfd;
  };
  using General = std::integral_constant<int, 0>;
  for (; J < Ja; ++J) step(J, General());
  if (band_int) {
    HELM_PRAGMA_UNROLL(HELM_GLKS_FAST_UNROLL)
    for (; J < Jb; ++J) step(J, std::integral_constant<int, 2>());
  }
  else
    for (; J < Jb; ++J) step(J, std::integral_constant<int, 1>());
  for (; J <= J1; ++J) step(J, General());
}

// ------------------------------------------------------------------ ReD-Glk (§5.2.4)
// Printed stencils: Laplacian part Eq. 5.12 (x 1/(256 H^2)) and wavenumber part Eq. 5.14
// (x 1/64^2), each tap weighted by the wavenumber at its own coarse node.
__constant__ double c_glk_lap[25] = {-3, -44, -98, -44, -3, -44, -112, 56, -112, -44, -98, 56, 980,
                                     56, -98, -44, -112, 56, -112, -44, -3, -44, -98, -44, -3};
__constant__ double c_glk_mass[25] = {1, 28, 70, 28, 1, 28, 784, 1960, 784, 28, 70, 1960, 4900,
                                      1960, 70, 28, 784, 1960, 784, 28, 1, 28, 70, 28, 1};

// Value of the coarse field at (ii, jj) possibly outside the unknown array (ReD-Glk2 ghosts):
// Dirichlet: boundary node (index -1 / n) holds 0, ghost beyond it mirrors with a sign
// (Eq. 5.18: u_b = (u_ghost + u_in)/2, u_b = 0); Sommerfeld: ghost one layer out from the
// boundary node by Eq. 2.8 (u_g = u_in + 2 i H k_b u_b), per direction.
__device__ double2 glk2_val(const Geo& g, const double2* __restrict__ x, const double* __restrict__ k, int ii, int jj) {
  if (g.bc == BC_DIRICHLET) {
    double sgn = 1.0;
    for (int it = 0; it < 2; ++it) {
      if (ii == -1 || ii == g.nx || jj == -1 || jj == g.ny) return make_double2(0.0, 0.0);
      if (ii == -2) { ii = 0; sgn = -sgn; }
      else if (ii == g.nx + 1) { ii = g.nx - 1; sgn = -sgn; }
      else if (jj == -2) { jj = 0; sgn = -sgn; }
      else if (jj == g.ny + 1) { jj = g.ny - 1; sgn = -sgn; }
    }
    if (ii < 0 || ii >= g.nx || jj < 0 || jj >= g.ny) return make_double2(0.0, 0.0);
    return cscale(sgn, x[(size_t)jj * g.nx + ii]);
  }
  // Sommerfeld
  auto colv = [&](int ci, int row) -> double2 {   // value at column ci in [-1, nx], row in range
    if (ci == -1) {
      const size_t q = (size_t)row * g.nx;
      return cfma(make_double2(0.0, 2.0 * g.h * k[q]), x[q], x[q + 1]);
    }
    if (ci == g.nx) {
      const size_t q = (size_t)row * g.nx + g.nx - 1;
      return cfma(make_double2(0.0, 2.0 * g.h * k[q]), x[q], x[q - 1]);
    }
    return x[(size_t)row * g.nx + ci];
  };
  if (ii < -1 || ii > g.nx || jj < -1 || jj > g.ny) return make_double2(0.0, 0.0);
  if (jj == -1 || jj == g.ny) {
    const int r0 = (jj == -1) ? 0 : g.ny - 1, r1 = (jj == -1) ? 1 : g.ny - 2;
    const int ic = ii < 0 ? 0 : (ii >= g.nx ? g.nx - 1 : ii);
    const double kb = k[(size_t)r0 * g.nx + ic];
    return cfma(make_double2(0.0, 2.0 * g.h * kb), colv(ii, r0), colv(ii, r1));
  }
  return colv(ii, jj);
}

// VARIANT 1: ReD-Glk1, VARIANT 2: ReD-Glk2 (reading R14: the boundary layers use the plain
// second-order stencil A_2h, as PAPER.md:748 states, while the interior 5x5 rows carry the
// factor 4 of Z^T A Z).
template <int VARIANT, int MODE>
__global__ void k_apply_red_glk(Geo g, DVec xv, DVec fv, DVec yv, const double* __restrict__ k) {
  HELM_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.nx || j >= g.ny) return;
  const double2* __restrict__ x = xv.get();
  const double2* __restrict__ f = fv.get();
  double2* __restrict__ y = yv.get();
  const size_t p = (size_t)j * g.nx + i;
  bool use5;
  if (VARIANT == 1) use5 = (i >= 2 && i <= g.nx - 3 && j >= 2 && j <= g.ny - 3);
  else if (g.bc == BC_DIRICHLET) use5 = true;
  else use5 = (i >= 1 && i <= g.nx - 2 && j >= 1 && j <= g.ny - 2);
  double2 v;
  if (use5) {
    const double iH2 = 1.0 / (256.0 * g.h * g.h), im = 1.0 / 4096.0;
    v = make_double2(0.0, 0.0);
#pragma unroll
    for (int b = -2; b <= 2; ++b)
#pragma unroll
      for (int a = -2; a <= 2; ++a) {
        const int ii = i + a, jj = j + b;
        const bool in = (ii >= 0 && ii < g.nx && jj >= 0 && jj < g.ny);
        const double kk = in ? k[(size_t)jj * g.nx + ii] : 0.0;     // ghost wavenumber 0 (§5.2.4)
        const double2 xv = in ? x[(size_t)jj * g.nx + ii] : glk2_val(g, x, k, ii, jj);
        const int d = (b + 2) * 5 + (a + 2);
        const double c = c_glk_lap[d] * iH2 - c_glk_mass[d] * im * kk * kk;
        v = cadd(v, cscale(c, xv));
      }
  } else {
    Coef c = coef_at(g, i, j, k[p], 1.0, 0.0);
    v = stencil_apply(g, x, i, j, c);
  }
  if (MODE == 1) v = csub(cscale(fv.scale(), f[p]), v);
  y[p] = v;
}

// ReD-O4 (Eq. 5.11, reading R5: centre 5/H^2 - k^2) where the 5-wide cross fits,
// second-order Helmholtz stencil elsewhere (reading R6).
template <int MODE>
__global__ void k_apply_red_o4(Geo g, DVec xv, DVec fv, DVec yv, const double* __restrict__ k) {
  HELM_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.nx || j >= g.ny) return;
  const double2* __restrict__ x = xv.get();
  const double2* __restrict__ f = fv.get();
  double2* __restrict__ y = yv.get();
  const size_t p = (size_t)j * g.nx + i;
  bool fits;
  if (g.bc == BC_DIRICHLET) fits = (i >= 1 && i <= g.nx - 2 && j >= 1 && j <= g.ny - 2);
  else fits = (i >= 2 && i <= g.nx - 3 && j >= 2 && j <= g.ny - 3);
  double2 v;
  if (fits) {
    auto at = [&](int ii, int jj) -> double2 {
      if (ii < 0 || ii >= g.nx || jj < 0 || jj >= g.ny) return make_double2(0.0, 0.0);
      return x[(size_t)jj * g.nx + ii];
    };
    const double2 c = x[p];
    double2 d1 = cadd(cadd(at(i - 1, j), at(i + 1, j)), cadd(at(i, j - 1), at(i, j + 1)));
    double2 d2 = cadd(cadd(at(i - 2, j), at(i + 2, j)), cadd(at(i, j - 2), at(i, j + 2)));
    const double s = 1.0 / (12.0 * g.h * g.h);
    const double kk = k[p];
    v = make_double2(s * (60.0 * c.x - 16.0 * d1.x + d2.x) - kk * kk * c.x,
                     s * (60.0 * c.y - 16.0 * d1.y + d2.y) - kk * kk * c.y);
  } else {
    Coef c = coef_at(g, i, j, k[p], 1.0, 0.0);
    v = stencil_apply(g, x, i, j, c);
  }
  if (MODE == 1) v = csub(cscale(fv.scale(), f[p]), v);
  y[p] = v;
}

// ReD-O6 (Eq. 5.10: 7-point sixth-order second derivative per direction, centre k^2)
// where the 7-wide cross fits in the closed domain, second-order stencil elsewhere (reading R6).
template <int MODE>
__global__ void k_apply_red_o6(Geo g, DVec xv, DVec fv, DVec yv, const double* __restrict__ k) {
  HELM_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.nx || j >= g.ny) return;
  const double2* __restrict__ x = xv.get();
  const double2* __restrict__ f = fv.get();
  double2* __restrict__ y = yv.get();
  const size_t p = (size_t)j * g.nx + i;
  bool fits;
  if (g.bc == BC_DIRICHLET) fits = (i >= 2 && i <= g.nx - 3 && j >= 2 && j <= g.ny - 3);
  else fits = (i >= 3 && i <= g.nx - 4 && j >= 3 && j <= g.ny - 4);
  double2 v;
  if (fits) {
    auto at = [&](int ii, int jj) -> double2 {
      if (ii < 0 || ii >= g.nx || jj < 0 || jj >= g.ny) return make_double2(0.0, 0.0);
      return x[(size_t)jj * g.nx + ii];
    };
    auto ring = [&](int d) -> double2 {
      return cadd(cadd(at(i - d, j), at(i + d, j)), cadd(at(i, j - d), at(i, j + d)));
    };
    const double2 c = x[p];
    const double2 r1 = ring(1), r2 = ring(2), r3 = ring(3);
    const double s = 1.0 / (180.0 * g.h * g.h);
    const double kk = k[p];
    v = make_double2(s * (980.0 * c.x - 270.0 * r1.x + 27.0 * r2.x - 2.0 * r3.x) - kk * kk * c.x,
                     s * (980.0 * c.y - 270.0 * r1.y + 27.0 * r2.y - 2.0 * r3.y) - kk * kk * c.y);
  } else {
    Coef c = coef_at(g, i, j, k[p], 1.0, 0.0);
    v = stencil_apply(g, x, i, j, c);
  }
  if (MODE == 1) v = csub(cscale(fv.scale(), f[p]), v);
  y[p] = v;
}

// General 3x3 re-discretisation (Eq. 5.19):
//   y = (1/H^2) sum a_tap u_tap - k_c^2 sum b_tap u_tap over the 3x3 compact stencil, k_c the
// centre wavenumber (reading R19).  VAR 0: ReD-cmpO4, Singer-Turkel coefficients with gamma = 1,
// Sommerfeld ghosts u_ghost = u_inner + 2 i k H (1 - k^2 H^2/6) u_boundary;
// VAR 1: ReD-9ptO2 (Appendix B: a = (4.632, -1.316, 0.158), b = (1, 0, 0)),
// second-order ghosts u_ghost = u_inner + 2 i k H u_boundary (reading R22).  Dirichlet: boundary
// taps hold 0.  Corner ghost = mean of its two edge ghosts.
template <int VAR>
__device__ __forceinline__ double2 cmp_ghost_fac(double kk, double H) {
  if (VAR == 1) return make_double2(0.0, 2.0 * kk * H);
  return make_double2(0.0, 2.0 * kk * H * (1.0 - kk * kk * H * H / 6.0));
}

// value at (ii, jj) in [-1, nx] x [-1, ny] for the Sommerfeld compact stencil
template <int VAR>
__device__ __forceinline__ double2 cmp_val(const Geo& g, const double2* __restrict__ x, const double* __restrict__ k,
                                           int ii, int jj) {
  auto inside = [&](int a, int b) { return a >= 0 && a < g.nx && b >= 0 && b < g.ny; };
  auto X = [&](int a, int b) { return x[(size_t)b * g.nx + a]; };
  auto edge = [&](int a, int b) -> double2 {   // exactly one of a, b is outside by one layer
    if (a == -1) return cfma(cmp_ghost_fac<VAR>(k[(size_t)b * g.nx + 0], g.h), X(0, b), X(1, b));
    if (a == g.nx) return cfma(cmp_ghost_fac<VAR>(k[(size_t)b * g.nx + g.nx - 1], g.h), X(g.nx - 1, b), X(g.nx - 2, b));
    if (b == -1) return cfma(cmp_ghost_fac<VAR>(k[a], g.h), X(a, 0), X(a, 1));
    return cfma(cmp_ghost_fac<VAR>(k[(size_t)(g.ny - 1) * g.nx + a], g.h), X(a, g.ny - 1), X(a, g.ny - 2));
  };
  if (inside(ii, jj)) return X(ii, jj);
  const bool ox = (ii < 0 || ii >= g.nx), oy = (jj < 0 || jj >= g.ny);
  if (ox && oy) {   // corner ghost: mean of the two adjacent edge ghosts
    const int ai = ii < 0 ? 0 : g.nx - 1, bj = jj < 0 ? 0 : g.ny - 1;
    return cscale(0.5, cadd(edge(ai, jj), edge(ii, bj)));
  }
  return edge(ii, jj);
}

template <int MODE, int VAR>
__global__ void k_apply_red_cmpo4(Geo g, DVec xv, DVec fv, DVec yv, const double* __restrict__ k) {
  HELM_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.nx || j >= g.ny) return;
  const double2* __restrict__ x = xv.get();
  const double2* __restrict__ f = fv.get();
  double2* __restrict__ y = yv.get();
  const size_t p = (size_t)j * g.nx + i;
  constexpr double A0 = VAR == 1 ? 4.632 : 10.0 / 3.0, AS = VAR == 1 ? -1.316 : -2.0 / 3.0,
                   AC = VAR == 1 ? 0.158 : -1.0 / 6.0;
  constexpr double B0 = VAR == 1 ? 1.0 : 2.0 / 3.0 + 1.0 / 36.0, BS = VAR == 1 ? 0.0 : 1.0 / 12.0 - 1.0 / 72.0,
                   BC = VAR == 1 ? 0.0 : 1.0 / 144.0;
  double2 c, side, corner;
  if (g.bc == BC_DIRICHLET) {
    auto at = [&](int ii, int jj) -> double2 {
      if (ii < 0 || ii >= g.nx || jj < 0 || jj >= g.ny) return make_double2(0.0, 0.0);
      return x[(size_t)jj * g.nx + ii];
    };
    c = x[p];
    side = cadd(cadd(at(i - 1, j), at(i + 1, j)), cadd(at(i, j - 1), at(i, j + 1)));
    corner = cadd(cadd(at(i - 1, j - 1), at(i + 1, j - 1)), cadd(at(i - 1, j + 1), at(i + 1, j + 1)));
  } else {
    c = x[p];
    side = cadd(cadd(cmp_val<VAR>(g, x, k, i - 1, j), cmp_val<VAR>(g, x, k, i + 1, j)),
                cadd(cmp_val<VAR>(g, x, k, i, j - 1), cmp_val<VAR>(g, x, k, i, j + 1)));
    corner = cadd(cadd(cmp_val<VAR>(g, x, k, i - 1, j - 1), cmp_val<VAR>(g, x, k, i + 1, j - 1)),
                  cadd(cmp_val<VAR>(g, x, k, i - 1, j + 1), cmp_val<VAR>(g, x, k, i + 1, j + 1)));
  }
  const double iH2 = 1.0 / (g.h * g.h);
  const double k2 = k[p] * k[p];
  const double2 lap = cscale(iH2, cadd(cadd(cscale(A0, c), cscale(AS, side)), cscale(AC, corner)));
  const double2 mass = cadd(cadd(cscale(B0, c), cscale(BS, side)), cscale(BC, corner));
  double2 v = csub(lap, cscale(k2, mass));
  if (MODE == 1) v = csub(cscale(fv.scale(), f[p]), v);
  y[p] = v;
}

// ------------------------------------------------------------------ coarsest dense solve
// Dense M of the coarsest level, row-major n x n (row = unknown p).
__global__ void k_dense_op(Geo g, const double* __restrict__ k, double sr, double si, double2* __restrict__ Md) {
  HELM_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.nx || j >= g.ny) return;
  const size_t n = (size_t)g.nx * g.ny;
  const size_t p = (size_t)j * g.nx + i;
  Coef c = coef_at(g, i, j, k[p], sr, si);
  double2* row = Md + p * n;
  row[p] = c.ap;
  if (c.aw != 0.0) row[p - 1] = make_double2(c.aw, 0.0);
  if (c.ae != 0.0) row[p + 1] = make_double2(c.ae, 0.0);
  if (c.as != 0.0) row[p - g.nx] = make_double2(c.as, 0.0);
  if (c.an != 0.0) row[p + g.nx] = make_double2(c.an, 0.0);
}

// Gauss-Jordan with partial pivoting on the augmented [M | I] (n x 2n, row-major).
__global__ void k_gj_pivot(const double2* __restrict__ Aug, int n, int col, int* __restrict__ piv) {
  HELM_PDL_ENTRY();
  // one block: argmax_{r >= col} |Aug[r][col]|
  __shared__ double sv[1024];
  __shared__ int si[1024];
  double best = -1.0;
  int bi = col;
  for (int r = col + threadIdx.x; r < n; r += blockDim.x) {
    double2 a = Aug[(size_t)r * 2 * n + col];
    double m = a.x * a.x + a.y * a.y;
    if (m > best) { best = m; bi = r; }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      if (sv[threadIdx.x + s] > sv[threadIdx.x] ||
          (sv[threadIdx.x + s] == sv[threadIdx.x] && si[threadIdx.x + s] < si[threadIdx.x])) {
        sv[threadIdx.x] = sv[threadIdx.x + s];
        si[threadIdx.x] = si[threadIdx.x + s];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *piv = si[0];
}

__global__ void k_gj_swap_scale(double2* __restrict__ Aug, int n, int col, const int* __restrict__ piv,
                                double2* __restrict__ colbuf) {
  HELM_PDL_ENTRY();
  const int p = *piv;
  const int w = 2 * n;
  // swap rows col and p, then scale row col by 1/pivot; one block
  for (int c = threadIdx.x; c < w; c += blockDim.x) {
    double2 a = Aug[(size_t)col * w + c];
    double2 b = Aug[(size_t)p * w + c];
    Aug[(size_t)col * w + c] = b;
    Aug[(size_t)p * w + c] = a;
  }
  __syncthreads();
  __shared__ double2 pv;
  if (threadIdx.x == 0) pv = Aug[(size_t)col * w + col];
  __syncthreads();
  const double2 inv = cdiv(make_double2(1.0, 0.0), pv);
  for (int c = threadIdx.x; c < w; c += blockDim.x) Aug[(size_t)col * w + c] = cmul(Aug[(size_t)col * w + c], inv);
  __syncthreads();
  // save column col (multipliers) for the elimination step
  for (int r = threadIdx.x; r < n; r += blockDim.x) colbuf[r] = Aug[(size_t)r * w + col];
}

__global__ void k_gj_eliminate(double2* __restrict__ Aug, int n, int col, const double2* __restrict__ colbuf) {
  HELM_PDL_ENTRY();
  const int w = 2 * n;
  const size_t total = (size_t)n * w;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(t / w), c = (int)(t % w);
    if (r == col) continue;
    const double2 m = colbuf[r];
    if (m.x == 0.0 && m.y == 0.0) continue;
    Aug[t] = csub(Aug[t], cmul(m, Aug[(size_t)col * w + c]));
  }
}

__global__ void k_gj_extract(const double2* __restrict__ Aug, int n, double2* __restrict__ Minv) {
  HELM_PDL_ENTRY();
  const size_t total = (size_t)n * n;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(t / n), c = (int)(t % n);
    Minv[t] = Aug[(size_t)r * 2 * n + n + c];
  }
}

// y = Minv f, one warp per row.
// One CTA of HELM_GEMV_T threads per row: the coarsest M^-1 (n <= a few hundred) is re-read from
// L2 every V-cycle, so the row is split over the CTA (n CTAs instead of n/8) to have enough loads
// in flight; warp shuffles + one shared-memory step reduce it.
#define HELM_GEMV_T 128
__global__ void __launch_bounds__(HELM_GEMV_T) k_gemv(const double2* __restrict__ Minv, int n, DVec fv, DVec yv,
                                                      const double2* __restrict__ addq) {
  __shared__ double2 part[HELM_GEMV_T / 32];
  const int row = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double2* __restrict__ r = Minv + (size_t)row * n;
  // the inverse is set-up data: its first entries are loaded before the PDL wait (their latency
  // overlaps the predecessor, the down leg that writes f); same summation order as the loop
  constexpr int NP = 2;
  double2 rp[NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const int c = threadIdx.x + i * HELM_GEMV_T;
    rp[i] = c < n ? r[c] : make_double2(0.0, 0.0);
  }
  HELM_PDL_ENTRY();
  const double2* __restrict__ f = fv.get();
  double2 s = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    const int c = threadIdx.x + i * HELM_GEMV_T;
    if (c < n) s = cfma(rp[i], f[c], s);
  }
#pragma unroll 4
  for (int c = threadIdx.x + NP * HELM_GEMV_T; c < n; c += HELM_GEMV_T) s = cfma(r[c], f[c], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
    s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
  }
  if (lane == 0) part[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = part[0];
#pragma unroll
    for (int q = 1; q < HELM_GEMV_T / 32; ++q) t = cadd(t, part[q]);
    t = cscale(fv.scale(), t);
    double2* __restrict__ y = yv.get();
    y[row] = addq ? cadd(t, addq[row]) : t;
  }
}

// y = a + b
__global__ void k_add(const double2* __restrict__ a, const double2* __restrict__ b, double2* __restrict__ y, size_t n) {
  HELM_PDL_ENTRY();
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    y[e] = cadd(a[e], b[e]);
}

}  // namespace helm
