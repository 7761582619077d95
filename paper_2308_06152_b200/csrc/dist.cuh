// Row-strip domain decomposition of the hierarchy (north_star: the grid is
// partitioned across the GPUs of one box, halo exchange + allreduce for the dots, coarse
// levels agglomerated).  PAPER.md §4 (:463-469) distributes the (i, j)-ordered grid over MPI
// ranks by blocks with ghost layers and stops coarsening at a predefined size; here:
//
//  * every level l <= D is split into P contiguous row strips (rows are contiguous in HBM, so
//    a halo is one contiguous copy).  Rank q owns rows [a, b) and stores the block [s, e) of
//    global rows, its own rows plus at least GHOST rows of neighbour data (s even, e - s odd).
//    Every kernel of the single-GPU path runs unchanged on a block: the block is a grid of its
//    own whose edge rows get boundary treatment, and the transfer kernels see the block and
//    its coarse window (the coarse rows coincident with block rows, a pointer offset into the
//    coarse block, which contains it) as a fine grid and its coarse grid.  What the artificial
//    edges spoil stays more than GHOST - 3 rows away from the owned rows (no fused kernel
//    reads further than 3 rows), and the GHOST rows next to the owned ones are refreshed from
//    the neighbours before every kernel that reads them.
//  * levels below D are replicated: the down leg of level D writes its coarse rows into the
//    rank's replica, the replicas are completed by an all-gather of the owned rows, and every
//    rank runs the rest of the V-cycle (down to the dense coarsest solve) on the whole level.
//  * Krylov vectors are blocks too; dots and norms run over the owned rows and are summed over
//    the ranks (allreduce) before the scalar steps, which every rank then performs identically.
//
// Two transports with identical host logic: HELM_COMM_NCCL (one process per GPU; grouped
// ncclSend/ncclRecv halos, ncclAllReduce, ncclBroadcast all-gather; libnccl.so.2 is loaded at
// run time) and HELM_COMM_THREADS (P host threads of one process on one GPU, each with its
// own context and stream; exchanges are device copies from the peer's buffers ordered by CUDA
// events and host barriers -- no kernel ever waits on another rank, so this is safe on one
// GPU; it is how the decomposition is tested against the oracle on a single B200).
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace helm {

constexpr int GHOST = 6;          // halo rows exchanged on each side (>= 3 + margin)
constexpr int DIST_MAX_RANKS = 16;

struct DistRows {
  int a, b;   // owned global rows [a, b)
  int s, e;   // stored global rows [s, e) (levels <= D: the block; level D+1: the transfer window)
};

inline int cdiv2(int x) { return x >= 0 ? (x + 1) / 2 : -((-x) / 2); }

// Coarse window of a fine block [s, e) (s even): the coarse rows whose coincident fine rows
// lie in the block, so that the transfer kernels see (block, window) as a fine grid and its
// coarse grid with the usual node offset o.
inline void coarse_window(int s, int e, int dirichlet, int& ws, int& we) {
  const int H = e - s;
  ws = s / 2;
  we = ws + (dirichlet ? (H - 1) / 2 : (H + 1) / 2);
}

// Row partition of a hierarchy with global row counts ny[0..nl-1].  Returns D (deepest
// decomposed level, >= 1) or -1 with a reason.  plan[l * P + q]: owned rows [a, b) and, for
// l <= D, the stored block [s, e) = owned rows +- >= GHOST rows, s even, e - s odd, each
// block containing the coarse window of the block above; for l = D + 1 [s, e) is the window
// of the level-D block in the replicated level; below, the whole level.
inline int dist_plan(const std::vector<int>& ny, int dirichlet, int P, int min_rows, int want_levels,
                     std::vector<DistRows>& plan, std::string& why) {
  const int nl = (int)ny.size();
  const int o = dirichlet ? 1 : 0;
  plan.assign((size_t)nl * P, DistRows{0, 0, 0, 0});
  if (P < 1 || P > DIST_MAX_RANKS) {
    why = "nranks must be in [1, 16]";
    return -1;
  }
  for (int q = 0; q < P; ++q) {
    plan[q].a = (int)((long long)ny[0] * q / P);
    plan[q].b = (int)((long long)ny[0] * (q + 1) / P);
  }
  // coarse row J is owned by the rank owning its coincident fine row 2J + o
  for (int l = 1; l < nl; ++l)
    for (int q = 0; q < P; ++q) {
      DistRows& r = plan[(size_t)l * P + q];
      const DistRows& f = plan[(size_t)(l - 1) * P + q];
      r.a = std::min(ny[l], std::max(0, cdiv2(f.a - o)));
      r.b = std::min(ny[l], std::max(0, cdiv2(f.b - o)));
    }
  const int need = std::max(GHOST, min_rows);
  int D = -1;
  for (int l = 0; l <= nl - 2; ++l) {
    bool ok = true;
    for (int q = 0; q < P; ++q) ok = ok && (plan[(size_t)l * P + q].b - plan[(size_t)l * P + q].a >= need);
    if (!ok) break;
    D = l;
  }
  if (want_levels > 0) {
    if (want_levels - 1 > D) {
      why = "dist_levels too large: a rank would own fewer than " + std::to_string(need) + " rows";
      return -1;
    }
    D = want_levels - 1;
  }
  if (D < 1) {
    why = "grid too small for " + std::to_string(P) + " ranks: levels 0 and 1 must give every rank >= " +
          std::to_string(need) + " rows";
    return -1;
  }
  auto fix_parity = [&](DistRows& r, int l) {   // e - s odd (ny[l] is odd on coarsenable levels)
    if (((r.e - r.s) & 1) == 0) {
      if (r.e < ny[l]) r.e += 1;
      else r.s -= 2;
    }
  };
  for (int q = 0; q < P; ++q) {
    for (int l = 0; l <= D; ++l) {
      DistRows& r = plan[(size_t)l * P + q];
      r.s = std::max(0, r.a - GHOST) & ~1;
      r.e = std::min(ny[l], r.b + GHOST);
      fix_parity(r, l);
    }
    for (int l = 0; l <= D; ++l) {
      const DistRows& r = plan[(size_t)l * P + q];
      int ws, we;
      coarse_window(r.s, r.e, dirichlet, ws, we);
      DistRows& c = plan[(size_t)(l + 1) * P + q];
      if (l + 1 <= D) {   // the coarse block must contain the window
        if (ws < c.s) c.s = ws & ~1;
        if (we > c.e) c.e = we;
        fix_parity(c, l + 1);
      } else {
        c.s = ws;
        c.e = we;
      }
    }
    for (int l = 0; l <= D + 1; ++l) {
      const DistRows& r = plan[(size_t)l * P + q];
      if (r.s < 0 || r.e > ny[l] || r.e - r.s < 3) {
        why = "internal: block outside the grid";
        return -1;
      }
      if (l <= D && ((r.a > 0 && r.s > r.a - GHOST) || (r.b < ny[l] && r.e < r.b + GHOST) || (r.s & 1) ||
                     !((r.e - r.s) & 1))) {
        why = "internal: block lacks ghost rows";
        return -1;
      }
    }
    for (int l = D + 2; l < nl; ++l) {
      plan[(size_t)l * P + q].s = 0;
      plan[(size_t)l * P + q].e = ny[l];
    }
  }
  return D;
}

// ------------------------------------------------------------------ halo kernels
// Copy the GHOST owned rows next to each neighbour into the send buffers (x read through its
// DVec: a Krylov basis vector is addressed by a device-side column index).
__global__ void k_halo_pack(DVec xv, int nx, int own0, int nown, int has_up, int has_dn, double2* __restrict__ sup,
                            double2* __restrict__ sdn) {
  HELM_PDL_ENTRY();
  const double2* x = xv.get();
  const int n = GHOST * nx;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    if (has_up) sup[t] = x[(size_t)own0 * nx + t];
    if (has_dn) sdn[t] = x[(size_t)(own0 + nown - GHOST) * nx + t];
  }
}

__global__ void k_halo_unpack(DVec xv, int nx, int own0, int nown, int has_up, int has_dn,
                              const double2* __restrict__ rup, const double2* __restrict__ rdn) {
  HELM_PDL_ENTRY();
  double2* x = xv.get();
  const int n = GHOST * nx;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    if (has_up) x[(size_t)(own0 - GHOST) * nx + t] = rup[t];
    if (has_dn) x[(size_t)(own0 + nown) * nx + t] = rdn[t];
  }
}

struct PeerPtrs {
  const double2* p[DIST_MAX_RANKS];
};

// out[i] = sum_q src_q[i] in rank order (the same bits on every rank)
__global__ void k_sum_ranks(PeerPtrs src, int P, int n, double2* __restrict__ out) {
  HELM_PDL_ENTRY();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double2 s = src.p[0][i];
    for (int q = 1; q < P; ++q) s = cadd(s, src.p[q][i]);
    out[i] = s;
  }
}

// ------------------------------------------------------------------ transports
struct HostBarrier {
  std::mutex m;
  std::condition_variable cv;
  int n = 1, count = 0;
  long long gen = 0;
  void wait() {
    std::unique_lock<std::mutex> lk(m);
    const long long g = gen;
    if (++count == n) {
      count = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

// Registered per-rank device pointers of a thread group (HELM_COMM_THREADS).
struct GroupRank {
  cudaEvent_t ev = nullptr;
  std::vector<double2*> send_up, send_dn;   // per level
  std::vector<double2*> gathered;           // per level: replicated f arrays (all-gathered levels)
  double2* red = nullptr;                   // allreduce slot
};

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// Load NCCL once: the copy already in the process (torch's), else HELM_NCCL_LIB, else the
// default search path.
inline const NcclApi* nccl_api(std::string& why) {
  static NcclApi api;
  static bool tried = false;
  static std::string err;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h && getenv("HELM_NCCL_LIB")) h = dlopen(getenv("HELM_NCCL_LIB"), RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
    } else {
      api.h = h;
      bool ok = true;
      auto sym = [&](auto& fp, const char* name) {
        fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
        if (!fp) ok = false;
      };
      sym(api.GetUniqueId, "ncclGetUniqueId");
      sym(api.CommInitRank, "ncclCommInitRank");
      sym(api.CommDestroy, "ncclCommDestroy");
      sym(api.Send, "ncclSend");
      sym(api.Recv, "ncclRecv");
      sym(api.AllReduce, "ncclAllReduce");
      sym(api.Broadcast, "ncclBroadcast");
      sym(api.GroupStart, "ncclGroupStart");
      sym(api.GroupEnd, "ncclGroupEnd");
      sym(api.GetErrorString, "ncclGetErrorString");
      if (!ok) {
        err = "libnccl.so.2 lacks a required symbol";
        api.h = nullptr;
      }
    }
  }
  if (!api.h) {
    why = err;
    return nullptr;
  }
  return &api;
}

}  // namespace helm

// A group of P ranks that live as threads of one process (HELM_COMM_THREADS).
struct helm_group_s {
  int n = 1;
  helm::HostBarrier bar;
  std::vector<helm::GroupRank> rank;
  std::vector<int> status;   // setup outcome per rank
};
