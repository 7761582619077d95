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
#include "kernels.cuh"

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

// ------------------------------------------------------------------ down leg
// CTA = TCX x TCY coarse points.  Fine footprint of the restriction: fine nodes
// 2I+o-1 .. 2I+o+1; the residual there needs u one node further out.
template <int TCX, int TCY>
__global__ void __launch_bounds__(256) k_vc_down(Geo F, Geo G, int o, DVec fv, const double* __restrict__ k,
                                                 double sr, double si, double omega, double2* __restrict__ u,
                                                 double2* __restrict__ fc) {
  HELM_PDL_ENTRY();
  constexpr int RX = 2 * TCX + 3, RY = 2 * TCY + 3;  // u region
  constexpr int QX = 2 * TCX + 1, QY = 2 * TCY + 1;  // r region
  __shared__ double2 su[RY * RX];
  __shared__ double2 sq[QY * QX];
  const double2* __restrict__ f = fv.get();
  const double fs = fv.scale();
  const int I0 = blockIdx.x * TCX, J0 = blockIdx.y * TCY;
  const int gx0 = 2 * I0 + o - 2, gy0 = 2 * J0 + o - 2;
  // fine points whose pre-smoothed u this CTA owns (a partition of the fine grid)
  const int xs = (I0 == 0) ? 0 : 2 * I0 + o - 1;
  const int xe = (I0 + TCX >= G.nx) ? F.nx : 2 * (I0 + TCX) + o - 1;
  const int ys = (J0 == 0) ? 0 : 2 * J0 + o - 1;
  const int ye = (J0 + TCY >= G.ny) ? F.ny : 2 * (J0 + TCY) + o - 1;
  for (int t = threadIdx.x; t < RX * RY; t += blockDim.x) {
    const int ix = t % RX, iy = t / RX;
    const int x = gx0 + ix, y = gy0 + iy;
    double2 uv = czero();
    if (x >= 0 && x < F.nx && y >= 0 && y < F.ny) {
      const size_t p = (size_t)y * F.nx + x;
      const Coef c = coef_at(F, x, y, k[p], sr, si);
      uv = cscale(omega, cdiv(cscale(fs, f[p]), c.ap));   // reading R9: first sweep from u = 0
      if (x >= xs && x < xe && y >= ys && y < ye) u[p] = uv;
    }
    su[t] = uv;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < QX * QY; t += blockDim.x) {
    const int ix = t % QX, iy = t / QX;
    const int x = gx0 + 1 + ix, y = gy0 + 1 + iy;
    double2 rv = czero();                      // reading R4: out-of-array taps dropped
    if (x >= 0 && x < F.nx && y >= 0 && y < F.ny) {
      const size_t p = (size_t)y * F.nx + x;
      const Coef c = coef_at(F, x, y, k[p], sr, si);
      const int q = (iy + 1) * RX + (ix + 1);
      rv = csub(cscale(fs, f[p]), stencil5(c, su[q], su[q - 1], su[q + 1], su[q - RX], su[q + RX]));
    }
    sq[t] = rv;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < TCX * TCY; t += blockDim.x) {
    const int I = I0 + t % TCX, J = J0 + t / TCX;
    if (I >= G.nx || J >= G.ny) continue;
    const int ix = 2 * (I - I0) + 1, iy = 2 * (J - J0) + 1;
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

// ------------------------------------------------------------------ up leg
// CTA = TX x TY fine points; u1 is formed on the tile plus a 1-node halo.
template <int TX, int TY>
__global__ void __launch_bounds__(256) k_vc_up(Geo F, Geo G, int o, const double2* __restrict__ u,
                                               const double2* __restrict__ e, DVec fv,
                                               const double* __restrict__ k, double sr, double si, double omega,
                                               const double2* __restrict__ addq, DVec yv) {
  HELM_PDL_ENTRY();
  constexpr int RX = TX + 2, RY = TY + 2;
  constexpr int CX = TX / 2 + 3, CY = TY / 2 + 3;
  __shared__ double2 se[CY * CX];
  __shared__ double2 s1[RY * RX];
  const double2* __restrict__ f = fv.get();
  const double fs = fv.scale();
  double2* __restrict__ y = yv.get();
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int cx0 = floordiv2(x0 - 1 - o), cy0 = floordiv2(y0 - 1 - o);
  for (int t = threadIdx.x; t < CX * CY; t += blockDim.x) {
    const int I = cx0 + t % CX, J = cy0 + t / CX;
    se[t] = (I >= 0 && I < G.nx && J >= 0 && J < G.ny) ? e[(size_t)J * G.nx + I] : czero();
  }
  __syncthreads();
  for (int t = threadIdx.x; t < RX * RY; t += blockDim.x) {
    const int x = x0 - 1 + t % RX, yy = y0 - 1 + t / RX;
    double2 v = czero();
    if (x >= 0 && x < F.nx && yy >= 0 && yy < F.ny) {
      const int ri = x - o, rj = yy - o;
      const int Ia = floordiv2(ri), Ja = floordiv2(rj);
      const bool ox = (ri & 1) != 0, oy = (rj & 1) != 0;
      const int lx = Ia - cx0, ly = Ja - cy0;
      double2 s;
      if (!ox && !oy) {
        s = se[ly * CX + lx];
      } else if (ox && !oy) {
        s = cadd(cscale(0.5, se[ly * CX + lx]), cscale(0.5, se[ly * CX + lx + 1]));
      } else if (!ox && oy) {
        s = cadd(cscale(0.5, se[ly * CX + lx]), cscale(0.5, se[(ly + 1) * CX + lx]));
      } else {
        s = cadd(cadd(cscale(0.25, se[ly * CX + lx]), cscale(0.25, se[ly * CX + lx + 1])),
                 cadd(cscale(0.25, se[(ly + 1) * CX + lx]), cscale(0.25, se[(ly + 1) * CX + lx + 1])));
      }
      v = cadd(s, u[(size_t)yy * F.nx + x]);
    }
    s1[t] = v;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < TX * TY; t += blockDim.x) {
    const int x = x0 + t % TX, yy = y0 + t / TX;
    if (x >= F.nx || yy >= F.ny) continue;
    const size_t p = (size_t)yy * F.nx + x;
    const Coef c = coef_at(F, x, yy, k[p], sr, si);
    const int q = (t / TX + 1) * RX + (t % TX + 1);
    const double2 r = csub(cscale(fs, f[p]), stencil5(c, s1[q], s1[q - 1], s1[q + 1], s1[q - RX], s1[q + RX]));
    double2 v = cadd(s1[q], cscale(omega, cdiv(r, c.ap)));
    if (addq) v = cadd(v, addq[p]);
    y[p] = v;
  }
}

// ------------------------------------------------------------------ single-CTA tail
// The remaining levels lt..last of a V-cycle (small grids) in one CTA with every array of
// those levels (k, f, u and two scratch fields) in shared memory: the stages of a level are
// separated by __syncthreads(); only the input f, the output u (+ q) and the coarsest dense
// inverse touch global memory.
struct LevelDesc {
  Geo g;
  int o;
  const double* k;
};

// Shared-memory bytes the tail needs for levels lt..last (host and device agree on layout).
__host__ __device__ inline size_t tail_smem_bytes(const LevelDesc* Ls, int lt, int last) {
  size_t b = 0;
  for (int l = lt; l <= last; ++l) {
    const size_t n = (size_t)Ls[l].g.nx * Ls[l].g.ny;
    b += n * 4 * sizeof(double2) + ((n * sizeof(double) + 15) / 16) * 16;   // keep 16-byte alignment
  }
  return b;
}

struct TailLevel {
  Geo g;
  int o;
  double* k;
  double2 *f, *u, *s, *t;
};

__device__ __forceinline__ void tail_jacobi(const TailLevel& L, const double2* u, const double2* f, double2* out,
                                            const double2* addq, double sr, double si, double omega) {
  const int n = L.g.nx * L.g.ny;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    const int i = p % L.g.nx, j = p / L.g.nx;
    const Coef c = coef_at(L.g, i, j, L.k[p], sr, si);
    const double2 r = csub(f[p], stencil_apply(L.g, u, i, j, c));
    double2 v = cadd(u[p], cscale(omega, cdiv(r, c.ap)));
    if (addq) v = cadd(v, addq[p]);
    out[p] = v;
  }
}

constexpr int TAIL_MAX_LEVELS = 24;

__global__ void __launch_bounds__(1024) k_vc_tail(const LevelDesc* __restrict__ Ls, int lt, int last, DVec fv,
                                                  DVec uv, const double2* __restrict__ addq, double sr, double si,
                                                  double omega, int nu_pre, int nu_post,
                                                  const double2* __restrict__ Minv) {
  HELM_PDL_ENTRY();
  extern __shared__ double2 tsm[];
  __shared__ TailLevel T[TAIL_MAX_LEVELS];
  __shared__ int curi[TAIL_MAX_LEVELS];   // 0: pre-smoothed iterate in s, 1: in t
  double2* const uout = uv.get();
  const double2* const fin = fv.get();
  const int nl = last - lt + 1;
  if (threadIdx.x == 0) {
    char* p = reinterpret_cast<char*>(tsm);
    for (int q = 0; q < nl; ++q) {
      const LevelDesc D = Ls[lt + q];
      const size_t n = (size_t)D.g.nx * D.g.ny;
      T[q].g = D.g;
      T[q].o = D.o;
      T[q].f = reinterpret_cast<double2*>(p); p += n * sizeof(double2);
      T[q].u = reinterpret_cast<double2*>(p); p += n * sizeof(double2);
      T[q].s = reinterpret_cast<double2*>(p); p += n * sizeof(double2);
      T[q].t = reinterpret_cast<double2*>(p); p += n * sizeof(double2);
      T[q].k = reinterpret_cast<double*>(p); p += ((n * sizeof(double) + 15) / 16) * 16;
    }
  }
  __syncthreads();
  for (int q = 0; q < nl; ++q) {
    const int n = T[q].g.nx * T[q].g.ny;
    const double* kg = Ls[lt + q].k;
    for (int p = threadIdx.x; p < n; p += blockDim.x) T[q].k[p] = kg[p];
  }
  {
    const int n = T[0].g.nx * T[0].g.ny;
    const double fs = fv.scale();
    for (int p = threadIdx.x; p < n; p += blockDim.x) T[0].f[p] = cscale(fs, fin[p]);
  }
  __syncthreads();
  // ---- down
  for (int q = 0; q < nl - 1; ++q) {
    const TailLevel L = T[q];
    const TailLevel G = T[q + 1];
    const int n = L.g.nx * L.g.ny;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
      const int i = p % L.g.nx, j = p / L.g.nx;
      const Coef c = coef_at(L.g, i, j, L.k[p], sr, si);
      L.s[p] = cscale(omega, cdiv(L.f[p], c.ap));
    }
    __syncthreads();
    double2* cur = L.s;
    for (int sw = 1; sw < nu_pre; ++sw) {
      double2* nxt = (cur == L.s) ? L.t : L.s;
      tail_jacobi(L, cur, L.f, nxt, nullptr, sr, si, omega);
      __syncthreads();
      cur = nxt;
    }
    double2* rb = (cur == L.s) ? L.t : L.s;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
      const int i = p % L.g.nx, j = p / L.g.nx;
      const Coef c = coef_at(L.g, i, j, L.k[p], sr, si);
      rb[p] = csub(L.f[p], stencil_apply(L.g, cur, i, j, c));
    }
    __syncthreads();
    const int nc = G.g.nx * G.g.ny;
    for (int P = threadIdx.x; P < nc; P += blockDim.x) {
      const int I = P % G.g.nx, J = P / G.g.nx;
      const int ci = 2 * I + L.o, cj = 2 * J + L.o;
      double2 s = czero();
      for (int b = -1; b <= 1; ++b) {
        const int jj = cj + b;
        if (jj < 0 || jj >= L.g.ny) continue;
        for (int a = -1; a <= 1; ++a) {
          const int ii = ci + a;
          if (ii < 0 || ii >= L.g.nx) continue;
          const double w = (a == 0 ? 2.0 : 1.0) * (b == 0 ? 2.0 : 1.0) * (1.0 / 16.0);
          s = cadd(s, cscale(w, rb[jj * L.g.nx + ii]));
        }
      }
      G.f[P] = s;
    }
    if (threadIdx.x == 0) curi[q] = (cur == L.s) ? 0 : 1;
    __syncthreads();
  }
  // ---- coarsest: dense inverse (reading R8), one warp per row
  {
    const TailLevel Cl = T[nl - 1];
    const int n = Cl.g.nx * Cl.g.ny;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int r = warp; r < n; r += nw) {
      double2 s = czero();
      for (int c = lane; c < n; c += 32) s = cfma(Minv[(size_t)r * n + c], Cl.f[c], s);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, off);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
      }
      if (lane == 0) {
        if (nl == 1) uout[r] = addq ? cadd(s, addq[r]) : s;
        else Cl.u[r] = s;
      }
    }
    __syncthreads();
  }
  // ---- up
  for (int q = nl - 2; q >= 0; --q) {
    const TailLevel L = T[q];
    const TailLevel G = T[q + 1];
    const bool top = (q == 0);
    double2* cur = curi[q] ? L.t : L.s;
    double2* ob = curi[q] ? L.s : L.t;
    const int n = L.g.nx * L.g.ny;
    double2* u1 = (nu_post == 0) ? L.u : ob;
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
      const int i = p % L.g.nx, j = p / L.g.nx;
      const int ri = i - L.o, rj = j - L.o;
      const int Ia = floordiv2(ri), Ja = floordiv2(rj);
      const bool ox = (ri & 1) != 0, oy = (rj & 1) != 0;
      double2 s = czero();
      for (int bj = 0; bj <= (oy ? 1 : 0); ++bj) {
        const int J = Ja + bj;
        if (J < 0 || J >= G.g.ny) continue;
        const double wy = oy ? 0.5 : 1.0;
        for (int ai = 0; ai <= (ox ? 1 : 0); ++ai) {
          const int I = Ia + ai;
          if (I < 0 || I >= G.g.nx) continue;
          const double wx = ox ? 0.5 : 1.0;
          s = cadd(s, cscale(wx * wy, G.u[J * G.g.nx + I]));
        }
      }
      u1[p] = cadd(s, cur[p]);
    }
    __syncthreads();
    double2* src = u1;
    for (int sw = 0; sw < nu_post; ++sw) {
      double2* dst = (sw == nu_post - 1) ? L.u : ((src == ob) ? cur : ob);
      tail_jacobi(L, src, L.f, dst, nullptr, sr, si, omega);
      __syncthreads();
      src = dst;
    }
    if (top) {
      for (int p = threadIdx.x; p < n; p += blockDim.x) uout[p] = addq ? cadd(L.u[p], addq[p]) : L.u[p];
    }
  }
}

}  // namespace helm
