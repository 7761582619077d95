// Host side of the C ABI declared in include/helm.h: hierarchy setup, kernel orchestration
// of the V-cycle, the A-DEF1 deflation operator, and flexible GMRES (outer and inner).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/helm.h"
#include "kernels.cuh"

using namespace helm;
using cplx = std::complex<double>;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return fail(HELM_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, \
                                       cudaGetErrorString(e_));                               \
  } while (0)

#define CKR(expr)              \
  do {                         \
    int r_ = (expr);           \
    if (r_ != HELM_OK) return r_; \
  } while (0)

struct Level {
  Geo g;
  int o;            // node offset of unknown 0 (1 Dirichlet, 0 Sommerfeld)
  size_t n;
  double* k = nullptr;
  double2* f = nullptr;  // rhs when this level is reached by recursion
  double2* u = nullptr;  // solution when reached by recursion
  double2* t = nullptr;  // scratch
};

struct Krylov {
  int m = 0;       // basis capacity
  size_t n = 0;
  double2* V = nullptr;   // (m+1) x n
  double2* Z = nullptr;   // m x n
  std::vector<cplx> H;    // (m+1) x m, column-major H[i + j*(m+1)]
  std::vector<double> cs;
  std::vector<cplx> sn, g;
};

}  // namespace

struct helm_ctx_s {
  cudaStream_t s = nullptr;
  helm_params p{};
  std::vector<Level> L;
  double2* Minv = nullptr;
  int ncoarsest = 0;
  double2* gal = nullptr;          // Galerkin 9-point coefficients on level 1
  double2 *dq = nullptr, *dt = nullptr;   // fine scratch for A-DEF1
  double2 *cc = nullptr, *ce = nullptr;   // coarse rhs / solution
  double2 *bx = nullptr, *xx = nullptr;   // device b/x for helm_solve_host
  Krylov outer, inner;
  double2* partial = nullptr;      // multidot partials
  size_t partial_cap = 0;
  double2* dres = nullptr;         // device scalar results
  cplx* hres = nullptr;            // pinned host mirror
  size_t dres_cap = 0;
  uint4* flush = nullptr;
  size_t flush_n = 0;
  long long launches = 0;
  int last_inner = 0;
  int sm_count = 148;
};

namespace {

dim3 blk2d() { return dim3(32, 8); }
dim3 grd2d(int nx, int ny) { return dim3((nx + 31) / 32, (ny + 7) / 8); }
int grid1d(const helm_ctx_s& C, size_t n) {
  size_t b = (n + 255) / 256;
  size_t cap = (size_t)C.sm_count * 8;
  return (int)std::max<size_t>(1, std::min(b, cap));
}

int post_launch(helm_ctx_s& C) {
  C.launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HELM_ECUDA, "kernel launch: %s", cudaGetErrorString(e));
  return HELM_OK;
}

int coarse_n(int n, int bc) {
  if (n < 3 || (n % 2) == 0) return -1;
  return bc == BC_DIRICHLET ? (n - 1) / 2 : (n + 1) / 2;
}

template <class T>
int dalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  CK(cudaMalloc((void**)p, count * sizeof(T)));
  return HELM_OK;
}

// ------------------------------------------------------------------ operator launches
int op_apply(helm_ctx_s& C, const Level& L, const double2* u, const double2* f, double2* y, double sr, double si) {
  if (f) k_apply_op<1><<<grd2d(L.g.nx, L.g.ny), blk2d(), 0, C.s>>>(L.g, u, f, y, L.k, sr, si);
  else k_apply_op<0><<<grd2d(L.g.nx, L.g.ny), blk2d(), 0, C.s>>>(L.g, u, nullptr, y, L.k, sr, si);
  return post_launch(C);
}

int restrict_(helm_ctx_s& C, int l, const double2* v, double2* vc) {
  const Level& F = C.L[l];
  const Level& G = C.L[l + 1];
  k_restrict<<<grd2d(G.g.nx, G.g.ny), blk2d(), 0, C.s>>>(F.g, G.g, F.o, v, vc);
  return post_launch(C);
}

int prolong_(helm_ctx_s& C, int l, const double2* e, const double2* base, double2* y) {
  const Level& F = C.L[l];
  const Level& G = C.L[l + 1];
  if (base) k_prolong<1><<<grd2d(F.g.nx, F.g.ny), blk2d(), 0, C.s>>>(F.g, G.g, F.o, e, base, y);
  else k_prolong<0><<<grd2d(F.g.nx, F.g.ny), blk2d(), 0, C.s>>>(F.g, G.g, F.o, e, nullptr, y);
  return post_launch(C);
}

// Deflation vectors level 0 <-> level 1 (bilinear: R=1, high order: R=2)
int defl_restrict(helm_ctx_s& C, const double2* v, double2* vc) {
  const Level& F = C.L[0];
  const Level& G = C.L[1];
  if (C.p.vectors == HELM_VECTORS_BILINEAR)
    k_restrict_z<1><<<grd2d(G.g.nx, G.g.ny), blk2d(), 0, C.s>>>(F.g, G.g, F.o, v, vc);
  else
    k_restrict_z<2><<<grd2d(G.g.nx, G.g.ny), blk2d(), 0, C.s>>>(F.g, G.g, F.o, v, vc);
  return post_launch(C);
}

int defl_prolong(helm_ctx_s& C, const double2* e, double2* y) {
  const Level& F = C.L[0];
  const Level& G = C.L[1];
  if (C.p.vectors == HELM_VECTORS_BILINEAR)
    k_prolong_z<1, 0><<<grd2d(F.g.nx, F.g.ny), blk2d(), 0, C.s>>>(F.g, G.g, F.o, e, nullptr, y);
  else
    k_prolong_z<2, 0><<<grd2d(F.g.nx, F.g.ny), blk2d(), 0, C.s>>>(F.g, G.g, F.o, e, nullptr, y);
  return post_launch(C);
}

// y = E x (f == null) or y = f - E x on level 1
int apply_E(helm_ctx_s& C, const double2* x, const double2* f, double2* y) {
  const Level& G = C.L[1];
  const dim3 gg = grd2d(G.g.nx, G.g.ny);
  switch (C.p.coarse_op) {
    case HELM_COARSE_GALERKIN:
      if (C.p.vectors == HELM_VECTORS_BILINEAR) {
        if (f) k_apply_stencil<1, 1><<<gg, blk2d(), 0, C.s>>>(G.g, C.gal, x, f, y);
        else k_apply_stencil<1, 0><<<gg, blk2d(), 0, C.s>>>(G.g, C.gal, x, nullptr, y);
      } else {
        if (f) k_apply_stencil<2, 1><<<gg, blk2d(), 0, C.s>>>(G.g, C.gal, x, f, y);
        else k_apply_stencil<2, 0><<<gg, blk2d(), 0, C.s>>>(G.g, C.gal, x, nullptr, y);
      }
      return post_launch(C);
    case HELM_COARSE_RED_GLK1:
      if (f) k_apply_red_glk<1, 1><<<gg, blk2d(), 0, C.s>>>(G.g, x, f, y, G.k);
      else k_apply_red_glk<1, 0><<<gg, blk2d(), 0, C.s>>>(G.g, x, nullptr, y, G.k);
      return post_launch(C);
    case HELM_COARSE_RED_GLK2:
      if (f) k_apply_red_glk<2, 1><<<gg, blk2d(), 0, C.s>>>(G.g, x, f, y, G.k);
      else k_apply_red_glk<2, 0><<<gg, blk2d(), 0, C.s>>>(G.g, x, nullptr, y, G.k);
      return post_launch(C);
    case HELM_COARSE_RED_O2:
      return op_apply(C, G, x, f, y, 1.0, 0.0);
    case HELM_COARSE_RED_O4:
      if (f) k_apply_red_o4<1><<<grd2d(G.g.nx, G.g.ny), blk2d(), 0, C.s>>>(G.g, x, f, y, G.k);
      else k_apply_red_o4<0><<<grd2d(G.g.nx, G.g.ny), blk2d(), 0, C.s>>>(G.g, x, nullptr, y, G.k);
      return post_launch(C);
  }
  return fail(HELM_EINVAL, "bad coarse_op");
}

// ------------------------------------------------------------------ V-cycle (§3.1)
int vcycle(helm_ctx_s& C, int l, const double2* f, double2* u, const double2* addq) {
  const int last = (int)C.L.size() - 1;
  Level& L = C.L[l];
  const double sr = C.p.beta1, si = C.p.beta2, w = C.p.omega;
  if (l == last) {
    const int n = (int)L.n;
    k_gemv<<<(n * 32 + 255) / 256, 256, 0, C.s>>>(C.Minv, n, f, u);
    CKR(post_launch(C));
    if (addq) {
      k_add<<<grid1d(C, L.n), 256, 0, C.s>>>(u, addq, u, L.n);
      CKR(post_launch(C));
    }
    return HELM_OK;
  }
  // pre-smoothing from u = 0 (reading R9)
  double2* cur = (C.p.nu_pre % 2 == 1) ? u : L.t;
  k_jacobi0<<<grd2d(L.g.nx, L.g.ny), blk2d(), 0, C.s>>>(L.g, f, cur, L.k, sr, si, w);
  CKR(post_launch(C));
  for (int s = 1; s < C.p.nu_pre; ++s) {
    double2* nxt = (cur == u) ? L.t : u;
    k_jacobi<<<grd2d(L.g.nx, L.g.ny), blk2d(), 0, C.s>>>(L.g, cur, f, nxt, L.k, sr, si, w, nullptr);
    CKR(post_launch(C));
    cur = nxt;
  }
  // residual -> restriction -> recursion
  CKR(op_apply(C, L, u, f, L.t, sr, si));
  Level& G = C.L[l + 1];
  CKR(restrict_(C, l, L.t, G.f));
  CKR(vcycle(C, l + 1, G.f, G.u, nullptr));
  // correction + post-smoothing; the last write lands in u
  const int np = C.p.nu_post;
  cur = (np % 2 == 1) ? L.t : u;
  CKR(prolong_(C, l, G.u, u, cur));
  for (int s = 0; s < np; ++s) {
    double2* nxt = (cur == u) ? L.t : u;
    const double2* q = (s == np - 1) ? addq : nullptr;
    k_jacobi<<<grd2d(L.g.nx, L.g.ny), blk2d(), 0, C.s>>>(L.g, cur, f, nxt, L.k, sr, si, w, q);
    CKR(post_launch(C));
    cur = nxt;
  }
  if (np == 0 && addq) {
    k_add<<<grid1d(C, L.n), 256, 0, C.s>>>(u, addq, u, L.n);
    CKR(post_launch(C));
  }
  return HELM_OK;
}

// ------------------------------------------------------------------ BLAS-1 helpers
int ensure_scratch(helm_ctx_s& C, size_t partial_elems, size_t dres_elems) {
  if (partial_elems > C.partial_cap) {
    if (C.partial) cudaFree(C.partial);
    CKR(dalloc(&C.partial, partial_elems));
    C.partial_cap = partial_elems;
  }
  if (dres_elems > C.dres_cap) {
    if (C.dres) cudaFree(C.dres);
    if (C.hres) cudaFreeHost(C.hres);
    CKR(dalloc(&C.dres, dres_elems));
    CK(cudaMallocHost((void**)&C.hres, dres_elems * sizeof(cplx)));
    C.dres_cap = dres_elems;
  }
  return HELM_OK;
}

constexpr int NV = 8;

// out[c] = V_c^H w, c < nvec   (out is a device pointer)
int multidot(helm_ctx_s& C, const double2* V, size_t ld, int nvec, const double2* w, size_t n, double2* out) {
  const int nb = std::min(grid1d(C, n), 2 * C.sm_count);
  dim3 g(nb, (nvec + NV - 1) / NV);
  k_multidot_partial<NV><<<g, 256, 0, C.s>>>(V, ld, nvec, w, n, C.partial);
  CKR(post_launch(C));
  k_multidot_final<<<(nvec * 32 + 255) / 256, 256, 0, C.s>>>(C.partial, nb, nvec, out, 0);
  return post_launch(C);
}

int multi_axpy(helm_ctx_s& C, const double2* V, size_t ld, int nvec, const double2* coeff, double sign, double2* w,
               size_t n) {
  k_multi_axpy<<<grid1d(C, n), 256, nvec * sizeof(double2), C.s>>>(V, ld, nvec, coeff, sign, w, n);
  return post_launch(C);
}

int fetch(helm_ctx_s& C, int count) {
  CK(cudaMemcpyAsync(C.hres, C.dres, count * sizeof(cplx), cudaMemcpyDeviceToHost, C.s));
  CK(cudaStreamSynchronize(C.s));
  return HELM_OK;
}

int krylov_alloc(Krylov& K, int m, size_t n) {
  K.m = m;
  K.n = n;
  CKR(dalloc(&K.V, (size_t)(m + 1) * n));
  CKR(dalloc(&K.Z, (size_t)m * n));
  K.H.assign((size_t)(m + 1) * m, cplx(0, 0));
  K.cs.assign(m, 0.0);
  K.sn.assign(m, cplx(0, 0));
  K.g.assign(m + 1, cplx(0, 0));
  return HELM_OK;
}

void krylov_free(Krylov& K) {
  if (K.V) cudaFree(K.V);
  if (K.Z) cudaFree(K.Z);
  K.V = K.Z = nullptr;
}

// Flexible GMRES (Algorithm 1 in flexible form, §6.3), x0 = 0, restarted when the
// basis capacity is exhausted.  Arnoldi orthogonalisation by classical Gram-Schmidt with one
// re-orthogonalisation pass (CGS2, batched dots; DESIGN.md §5 deviation from Alg. 1's MGS).
template <class OpA, class OpP>
int fgmres(helm_ctx_s& C, Krylov& K, OpA&& A, OpP&& P, const double2* b, double2* x, size_t n, double tol, int maxit,
           int* its_out, double* relres_out, int* conv_out, int* restarts_out) {
  const int m = K.m;
  CKR(ensure_scratch(C, (size_t)((m + NV) / NV * NV + NV) * 2 * C.sm_count, (size_t)(2 * m + 8)));
  CK(cudaMemsetAsync(x, 0, n * sizeof(double2), C.s));
  // ||b||
  CKR(multidot(C, b, n, 1, b, n, C.dres));
  CKR(fetch(C, 1));
  const double bnorm = std::sqrt(C.hres[0].real());
  int its = 0, restarts = 0, conv = 0;
  double relres = 0.0;
  if (bnorm == 0.0) {
    *its_out = 0; *relres_out = 0.0; *conv_out = 1; if (restarts_out) *restarts_out = 0;
    return HELM_OK;
  }
  double beta = bnorm;
  // V_0 = b / beta
  k_scale_copy<<<grid1d(C, n), 256, 0, C.s>>>(b, 1.0 / beta, K.V, n);
  CKR(post_launch(C));
  while (true) {
    std::fill(K.H.begin(), K.H.end(), cplx(0, 0));
    std::fill(K.g.begin(), K.g.end(), cplx(0, 0));
    K.g[0] = beta;
    int j = 0;
    bool done = false;
    for (; j < m && its < maxit; ++j) {
      double2* vj = K.V + (size_t)j * n;
      double2* zj = K.Z + (size_t)j * n;
      double2* w = K.V + (size_t)(j + 1) * n;
      CKR(P(vj, zj));
      CKR(A(zj, w));
      const int nv = j + 1;
      // CGS2
      CKR(multidot(C, K.V, n, nv, w, n, C.dres));
      CKR(multi_axpy(C, K.V, n, nv, C.dres, -1.0, w, n));
      CKR(multidot(C, K.V, n, nv, w, n, C.dres + nv));
      CKR(multi_axpy(C, K.V, n, nv, C.dres + nv, -1.0, w, n));
      CKR(multidot(C, w, n, 1, w, n, C.dres + 2 * nv));
      k_normalize<<<grid1d(C, n), 256, 0, C.s>>>(w, C.dres + 2 * nv, w, n);
      CKR(post_launch(C));
      CKR(fetch(C, 2 * nv + 1));
      const size_t ld = (size_t)m + 1;
      for (int i = 0; i < nv; ++i) K.H[i + j * ld] = C.hres[i] + C.hres[nv + i];
      const double hn = std::sqrt(std::max(0.0, C.hres[2 * nv].real()));
      K.H[(j + 1) + j * ld] = hn;
      for (int i = 0; i < j; ++i) {
        cplx t = K.cs[i] * K.H[i + j * ld] + K.sn[i] * K.H[i + 1 + j * ld];
        K.H[i + 1 + j * ld] = -std::conj(K.sn[i]) * K.H[i + j * ld] + K.cs[i] * K.H[i + 1 + j * ld];
        K.H[i + j * ld] = t;
      }
      cplx a = K.H[j + j * ld];
      double bb = hn;
      double den = std::sqrt(std::norm(a) + bb * bb);
      if (std::abs(a) == 0.0) { K.cs[j] = 0.0; K.sn[j] = 1.0; }
      else { K.cs[j] = std::abs(a) / den; K.sn[j] = (a / std::abs(a)) * bb / den; }
      K.H[j + j * ld] = K.cs[j] * a + K.sn[j] * bb;
      K.H[(j + 1) + j * ld] = 0.0;
      K.g[j + 1] = -std::conj(K.sn[j]) * K.g[j];
      K.g[j] = K.cs[j] * K.g[j];
      its++;
      relres = std::abs(K.g[j + 1]) / bnorm;
      if (relres <= tol || hn == 0.0) { done = true; conv = 1; ++j; break; }
    }
    // y = H^{-1} g ; x += Z y
    const int mm = j;
    const size_t ld = (size_t)m + 1;
    std::vector<cplx> y(mm);
    for (int i = mm - 1; i >= 0; --i) {
      cplx s = K.g[i];
      for (int q = i + 1; q < mm; ++q) s -= K.H[i + q * ld] * y[q];
      y[i] = s / K.H[i + i * ld];
    }
    if (mm > 0) {
      CK(cudaMemcpyAsync(C.dres, y.data(), mm * sizeof(cplx), cudaMemcpyHostToDevice, C.s));
      CKR(multi_axpy(C, K.Z, n, mm, C.dres, 1.0, x, n));
    }
    if (done || its >= maxit) break;
    // restart: r = b - A x ; V_0 = r / ||r||
    ++restarts;
    double2* r = K.V;
    CKR(A(x, r));
    k_scale_copy<<<grid1d(C, n), 256, 0, C.s>>>(r, -1.0, r, n);
    CKR(post_launch(C));
    k_add<<<grid1d(C, n), 256, 0, C.s>>>(r, b, r, n);
    CKR(post_launch(C));
    CKR(multidot(C, r, n, 1, r, n, C.dres));
    CKR(fetch(C, 1));
    beta = std::sqrt(C.hres[0].real());
    relres = beta / bnorm;
    if (relres <= tol) { conv = 1; break; }
    k_scale_copy<<<grid1d(C, n), 256, 0, C.s>>>(r, 1.0 / beta, K.V, n);
    CKR(post_launch(C));
  }
  *its_out = its;
  *relres_out = relres;
  *conv_out = conv;
  if (restarts_out) *restarts_out = restarts;
  return HELM_OK;
}

// e = E^{-1} c on level 1 by CSLP(V-cycle from level 1)-preconditioned FGMRES (reading R11).
int coarse_solve(helm_ctx_s& C, const double2* c, double2* e, int* its) {
  const Level& G = C.L[1];
  auto A = [&](const double2* x, double2* y) { return apply_E(C, x, nullptr, y); };
  auto P = [&](const double2* v, double2* z) { return vcycle(C, 1, v, z, nullptr); };
  double rr;
  int conv;
  return fgmres(C, C.inner, A, P, c, e, G.n, C.p.inner_tol, C.p.inner_maxit, its, &rr, &conv, nullptr);
}

// z = P_{A-DEF1} v (Eq. 3.21 / 5.2-5.5)
int adef1(helm_ctx_s& C, const double2* v, double2* z, int* inner_its) {
  Level& F = C.L[0];
  CKR(defl_restrict(C, v, C.cc));                         // v1 = I_h^{2h} v
  int its = 0;
  CKR(coarse_solve(C, C.cc, C.ce, &its));                 // v2 = A_{2h}^{-1} v1
  C.last_inner = its;
  if (inner_its) *inner_its = its;
  CKR(defl_prolong(C, C.ce, C.dq));                       // v' = I_{2h}^h v2  (= Q v)
  CKR(op_apply(C, F, C.dq, v, C.dt, 1.0, 0.0));           // t = v - A Q v  (= P_h v)
  return vcycle(C, 0, C.dt, z, C.dq);                     // z = M^{-1} t + Q v
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

void helm_default_params(helm_params* p) {
  if (!p) return;
  p->beta1 = 1.0;
  p->beta2 = 0.5;
  p->omega = 0.8;
  p->nu_pre = 1;
  p->nu_post = 1;
  p->coarse_op = HELM_COARSE_GALERKIN;
  p->inner_tol = 1e-1;
  p->inner_maxit = 200;
  p->max_levels = 64;
  p->restart = 0;
  p->max_coarsest = 4096;
  p->vectors = HELM_VECTORS_BILINEAR;
}

const char* helm_last_error(void) { return g_err.c_str(); }

const char* helm_build_info(void) { return "libhelm sm_100a complex128"; }

static void destroy_ctx(helm_ctx_s* C) {
  if (!C) return;
  for (auto& L : C->L) {
    cudaFree(L.k);
    cudaFree(L.f);
    cudaFree(L.u);
    cudaFree(L.t);
  }
  cudaFree(C->Minv);
  cudaFree(C->gal);
  cudaFree(C->dq);
  cudaFree(C->dt);
  cudaFree(C->cc);
  cudaFree(C->ce);
  cudaFree(C->bx);
  cudaFree(C->xx);
  cudaFree(C->partial);
  cudaFree(C->dres);
  cudaFree(C->flush);
  if (C->hres) cudaFreeHost(C->hres);
  krylov_free(C->outer);
  krylov_free(C->inner);
  delete C;
}

void helm_destroy(helm_ctx ctx) { destroy_ctx(ctx); }

static int setup_impl(helm_ctx_s& C, const helm_grid* grid, const double* k, int k_on_device) {
  const helm_params& p = C.p;
  if (grid->nx < 1 || grid->ny < 1 || !(grid->h > 0)) return fail(HELM_EINVAL, "bad grid");
  if (grid->bc != HELM_BC_DIRICHLET && grid->bc != HELM_BC_SOMMERFELD) return fail(HELM_EINVAL, "bad bc");
  if (grid->bc == HELM_BC_SOMMERFELD && (grid->nx < 2 || grid->ny < 2))
    return fail(HELM_EINVAL, "Sommerfeld grid needs >= 2 nodes per direction");
  if (p.max_levels < 2) return fail(HELM_EINVAL, "max_levels must be >= 2");
  if (p.nu_pre < 1 || p.nu_post < 0) return fail(HELM_EINVAL, "nu_pre >= 1, nu_post >= 0");
  if (p.inner_maxit < 1) return fail(HELM_EINVAL, "inner_maxit >= 1");
  if (p.vectors == HELM_VECTORS_BILINEAR) {
    if (p.coarse_op != HELM_COARSE_GALERKIN && p.coarse_op != HELM_COARSE_RED_O2 && p.coarse_op != HELM_COARSE_RED_O4)
      return fail(HELM_EINVAL, "coarse_op %d not defined for bilinear vectors", p.coarse_op);
  } else if (p.vectors == HELM_VECTORS_HIGH_ORDER) {
    if (p.coarse_op != HELM_COARSE_GALERKIN && p.coarse_op != HELM_COARSE_RED_GLK1 &&
        p.coarse_op != HELM_COARSE_RED_GLK2)
      return fail(HELM_EINVAL, "coarse_op %d not defined for high-order vectors", p.coarse_op);
  } else {
    return fail(HELM_EINVAL, "bad vectors %d", p.vectors);
  }
  int dev;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&C.sm_count, cudaDevAttrMultiProcessorCount, dev));
  // hierarchy (reading R7)
  Level L0;
  L0.g = Geo{grid->nx, grid->ny, grid->h, grid->bc};
  L0.o = grid->bc == HELM_BC_DIRICHLET ? 1 : 0;
  L0.n = (size_t)grid->nx * grid->ny;
  C.L.push_back(L0);
  while ((int)C.L.size() < p.max_levels) {
    const Level& F = C.L.back();
    int cx = coarse_n(F.g.nx, F.g.bc), cy = coarse_n(F.g.ny, F.g.bc);
    if (cx < 0 || cy < 0) break;
    Level G;
    G.g = Geo{cx, cy, 2.0 * F.g.h, F.g.bc};
    G.o = F.o;
    G.n = (size_t)cx * cy;
    C.L.push_back(G);
  }
  if (C.L.size() < 2) return fail(HELM_ESHAPE, "fine grid %dx%d is not coarsenable", grid->nx, grid->ny);
  const Level& Cst = C.L.back();
  if ((long long)Cst.n > p.max_coarsest)
    return fail(HELM_ESHAPE, "coarsest grid %dx%d exceeds max_coarsest=%d", Cst.g.nx, Cst.g.ny, p.max_coarsest);
  for (size_t l = 0; l < C.L.size(); ++l) {
    Level& Lv = C.L[l];
    CKR(dalloc(&Lv.k, Lv.n));
    CKR(dalloc(&Lv.t, Lv.n));
    if (l > 0) {
      CKR(dalloc(&Lv.f, Lv.n));
      CKR(dalloc(&Lv.u, Lv.n));
    }
  }
  CK(cudaMemcpyAsync(C.L[0].k, k, C.L[0].n * sizeof(double),
                     k_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, C.s));
  for (size_t l = 1; l < C.L.size(); ++l) {
    const Level& F = C.L[l - 1];
    Level& G = C.L[l];
    k_sample_k<<<grd2d(G.g.nx, G.g.ny), blk2d(), 0, C.s>>>(F.g, G.g, F.o, F.k, G.k);
    CKR(post_launch(C));
  }
  // coarsest dense inverse (reading R8): Gauss-Jordan with partial pivoting on device
  {
    const Level& Lc = C.L.back();
    const int n = (int)Lc.n;
    C.ncoarsest = n;
    double2* Md = nullptr;
    double2* Aug = nullptr;
    double2* colbuf = nullptr;
    int* piv = nullptr;
    CKR(dalloc(&Md, (size_t)n * n));
    CKR(dalloc(&Aug, (size_t)n * 2 * n));
    CKR(dalloc(&colbuf, n));
    CKR(dalloc(&piv, 1));
    CKR(dalloc(&C.Minv, (size_t)n * n));
    CK(cudaMemsetAsync(Md, 0, (size_t)n * n * sizeof(double2), C.s));
    k_dense_op<<<grd2d(Lc.g.nx, Lc.g.ny), blk2d(), 0, C.s>>>(Lc.g, Lc.k, p.beta1, p.beta2, Md);
    CKR(post_launch(C));
    // Aug = [Md | I]
    std::vector<cplx> eye((size_t)n * 2 * n, cplx(0, 0));
    for (int r = 0; r < n; ++r) eye[(size_t)r * 2 * n + n + r] = 1.0;
    CK(cudaMemcpyAsync(Aug, eye.data(), eye.size() * sizeof(cplx), cudaMemcpyHostToDevice, C.s));
    CK(cudaMemcpy2DAsync(Aug, 2 * n * sizeof(double2), Md, n * sizeof(double2), n * sizeof(double2), n,
                         cudaMemcpyDeviceToDevice, C.s));
    for (int col = 0; col < n; ++col) {
      k_gj_pivot<<<1, 1024, 0, C.s>>>(Aug, n, col, piv);
      CKR(post_launch(C));
      k_gj_swap_scale<<<1, 1024, 0, C.s>>>(Aug, n, col, piv, colbuf);
      CKR(post_launch(C));
      k_gj_eliminate<<<grid1d(C, (size_t)n * 2 * n), 256, 0, C.s>>>(Aug, n, col, colbuf);
      CKR(post_launch(C));
    }
    k_gj_extract<<<grid1d(C, (size_t)n * n), 256, 0, C.s>>>(Aug, n, C.Minv);
    CKR(post_launch(C));
    CK(cudaStreamSynchronize(C.s));
    cudaFree(Md);
    cudaFree(Aug);
    cudaFree(colbuf);
    cudaFree(piv);
  }
  // deflation coarse operator
  if (p.coarse_op == HELM_COARSE_GALERKIN) {
    const Level& F = C.L[0];
    const Level& G = C.L[1];
    if (p.vectors == HELM_VECTORS_BILINEAR) {
      CKR(dalloc(&C.gal, 9 * G.n));
      k_galerkin_coef<1><<<grd2d(G.g.nx, G.g.ny), blk2d(), 0, C.s>>>(F.g, G.g, F.o, F.k, C.gal);
    } else {
      CKR(dalloc(&C.gal, 25 * G.n));
      k_galerkin_coef<2><<<grd2d(G.g.nx, G.g.ny), blk2d(), 0, C.s>>>(F.g, G.g, F.o, F.k, C.gal);
    }
    CKR(post_launch(C));
  }
  CKR(dalloc(&C.dq, C.L[0].n));
  CKR(dalloc(&C.dt, C.L[0].n));
  CKR(dalloc(&C.cc, C.L[1].n));
  CKR(dalloc(&C.ce, C.L[1].n));
  {
    // inner basis capacity: inner_maxit, limited to a quarter of free HBM (restarted beyond)
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    const size_t per = 2 * C.L[1].n * sizeof(double2);
    const int cap = (int)std::max<size_t>(8, std::min<size_t>((size_t)p.inner_maxit, fr / 4 / per));
    CKR(krylov_alloc(C.inner, cap, C.L[1].n));
  }
  CK(cudaStreamSynchronize(C.s));
  return HELM_OK;
}

int helm_setup(helm_ctx* out, const helm_grid* grid, const double* k, int k_on_device, const helm_params* params,
               void* stream) {
  if (!out || !grid || !k) return fail(HELM_EINVAL, "null argument");
  *out = nullptr;
  helm_ctx_s* C = new helm_ctx_s();
  if (params) C->p = *params;
  else helm_default_params(&C->p);
  C->s = (cudaStream_t)stream;
  int r = setup_impl(*C, grid, k, k_on_device);
  if (r != HELM_OK) {
    destroy_ctx(C);
    return r;
  }
  *out = C;
  return HELM_OK;
}

int helm_num_levels(helm_ctx C) { return C ? (int)C->L.size() : fail(HELM_EINVAL, "null ctx"); }

int helm_level_info(helm_ctx C, int level, int* nx, int* ny, double* h) {
  if (!C || level < 0 || level >= (int)C->L.size()) return fail(HELM_EINVAL, "bad level");
  if (nx) *nx = C->L[level].g.nx;
  if (ny) *ny = C->L[level].g.ny;
  if (h) *h = C->L[level].g.h;
  return HELM_OK;
}

int helm_apply_A(helm_ctx C, const double* x, double* y) {
  if (!C || !x || !y) return fail(HELM_EINVAL, "null argument");
  return op_apply(*C, C->L[0], (const double2*)x, nullptr, (double2*)y, 1.0, 0.0);
}

int helm_apply_M(helm_ctx C, int level, const double* x, double* y) {
  if (!C || !x || !y || level < 0 || level >= (int)C->L.size()) return fail(HELM_EINVAL, "bad argument");
  return op_apply(*C, C->L[level], (const double2*)x, nullptr, (double2*)y, C->p.beta1, C->p.beta2);
}

int helm_restrict(helm_ctx C, int level, const double* v, double* vc) {
  if (!C || !v || !vc || level < 0 || level + 1 >= (int)C->L.size()) return fail(HELM_EINVAL, "bad argument");
  return restrict_(*C, level, (const double2*)v, (double2*)vc);
}

int helm_prolong(helm_ctx C, int level, const double* e, double* v) {
  if (!C || !v || !e || level < 0 || level + 1 >= (int)C->L.size()) return fail(HELM_EINVAL, "bad argument");
  return prolong_(*C, level, (const double2*)e, nullptr, (double2*)v);
}

int helm_apply_Zt(helm_ctx C, const double* v, double* vc) {
  if (!C || !v || !vc) return fail(HELM_EINVAL, "null argument");
  return defl_restrict(*C, (const double2*)v, (double2*)vc);
}

int helm_apply_Z(helm_ctx C, const double* e, double* v) {
  if (!C || !v || !e) return fail(HELM_EINVAL, "null argument");
  return defl_prolong(*C, (const double2*)e, (double2*)v);
}

int helm_apply_E(helm_ctx C, const double* x, double* y) {
  if (!C || !x || !y) return fail(HELM_EINVAL, "null argument");
  return apply_E(*C, (const double2*)x, nullptr, (double2*)y);
}

int helm_vcycle(helm_ctx C, int level, const double* f, double* u) {
  if (!C || !f || !u || level < 0 || level >= (int)C->L.size()) return fail(HELM_EINVAL, "bad argument");
  if (level > 0 && (f == (const double*)C->L[level].f || u == (double*)C->L[level].u))
    return fail(HELM_EINVAL, "aliasing internal buffers");
  return vcycle(*C, level, (const double2*)f, (double2*)u, nullptr);
}

int helm_deflate(helm_ctx C, const double* v, double* z, int* inner_its) {
  if (!C || !v || !z) return fail(HELM_EINVAL, "null argument");
  return adef1(*C, (const double2*)v, (double2*)z, inner_its);
}

int helm_solve(helm_ctx C, const double* b, double* x, double tol, int maxit, helm_report* rep) {
  if (!C || !b || !x) return fail(HELM_EINVAL, "null argument");
  if (b == x) return fail(HELM_EINVAL, "x may not alias b");
  if (maxit < 1 || !(tol > 0)) return fail(HELM_EINVAL, "bad tol/maxit");
  int m = C->p.restart > 0 ? std::min(C->p.restart, maxit) : maxit;
  if (C->outer.m < m || (C->outer.m > m && C->p.restart > 0)) {
    size_t fr = 0, tot = 0;
    if (C->outer.V) krylov_free(C->outer);
    CK(cudaMemGetInfo(&fr, &tot));
    const size_t per = 2 * C->L[0].n * sizeof(double2);
    m = (int)std::max<size_t>(8, std::min<size_t>((size_t)m, fr / 2 / per));
    CKR(krylov_alloc(C->outer, m, C->L[0].n));
  }
  long long inner_total = 0;
  int inner_max = 0, inner_solves = 0;
  auto A = [&](const double2* u, double2* y) { return op_apply(*C, C->L[0], u, nullptr, y, 1.0, 0.0); };
  auto P = [&](const double2* v, double2* z) {
    int its = 0;
    int r = adef1(*C, v, z, &its);
    inner_total += its;
    inner_max = std::max(inner_max, its);
    inner_solves++;
    return r;
  };
  auto t0 = std::chrono::steady_clock::now();
  int its = 0, conv = 0, restarts = 0;
  double relres = 0;
  CKR(fgmres(*C, C->outer, A, P, (const double2*)b, (double2*)x, C->L[0].n, tol, maxit, &its, &relres, &conv,
             &restarts));
  CK(cudaStreamSynchronize(C->s));
  auto t1 = std::chrono::steady_clock::now();
  if (rep) {
    rep->outer_iterations = its;
    rep->converged = conv;
    rep->relres = relres;
    rep->inner_solves = inner_solves;
    rep->inner_iterations_total = inner_total;
    rep->inner_iterations_max = inner_max;
    rep->restarts = restarts;
    rep->seconds = std::chrono::duration<double>(t1 - t0).count();
  }
  return HELM_OK;
}

int helm_solve_host(helm_ctx C, const double* b_host, double* x_host, double tol, int maxit, helm_report* rep) {
  if (!C || !b_host || !x_host) return fail(HELM_EINVAL, "null argument");
  const size_t n = C->L[0].n;
  if (!C->bx) CKR(dalloc(&C->bx, n));
  if (!C->xx) CKR(dalloc(&C->xx, n));
  CK(cudaMemcpyAsync(C->bx, b_host, n * sizeof(double2), cudaMemcpyHostToDevice, C->s));
  CKR(helm_solve(C, (const double*)C->bx, (double*)C->xx, tol, maxit, rep));
  CK(cudaMemcpyAsync(x_host, C->xx, n * sizeof(double2), cudaMemcpyDeviceToHost, C->s));
  CK(cudaStreamSynchronize(C->s));
  return HELM_OK;
}

int helm_flush_l2(helm_ctx C, size_t bytes) {
  if (!C) return fail(HELM_EINVAL, "null ctx");
  const size_t n = (bytes + 15) / 16;
  if (n > C->flush_n) {
    if (C->flush) cudaFree(C->flush);
    CKR(dalloc(&C->flush, n));
    C->flush_n = n;
  }
  k_l2flush<<<C->sm_count * 8, 256, 0, C->s>>>(C->flush, n, (unsigned)C->launches);
  return post_launch(*C);
}

long long helm_launch_count(helm_ctx C) { return C ? C->launches : 0; }

}  // extern "C"
