// Peer-memory transport for the row-strip decomposition (HELM_COMM_PEER): one
// process per GPU of one NVLink/NVSwitch node.  Every rank owns an "arena" (one cudaMalloc'd
// allocation, mapped into every peer through CUDA IPC) holding its outgoing halo rows, its
// rank-sum slot, its all-gather slot and its flags.  An exchange is two kernels with no host in
// the loop and no NCCL: the producer kernel writes its slot and then publishes an epoch flag
// (release, system scope); the consumer kernel waits for the peers' flags (acquire), reads
// their slots directly over NVLink and publishes an acknowledgement, which the next producer
// of the same slot waits for (no slot is overwritten before every reader is done).  Epochs
// are device counters in each rank's own arena, advanced by the producer kernels: every rank
// issues the same exchanges in the same order, so the counters stay in lockstep, and a solve
// captured in a CUDA graph replays correctly.
//
// Kernels of different ranks wait on each other here, so this transport needs one GPU per rank
// (never several ranks on one GPU).  Waits give up after ~10 s of GPU clock and raise an error
// flag the host checks after each solve, so a broken peer cannot hang the job forever.
#pragma once
#include <cuda/atomic>

#include "dist.cuh"
#include "kernels.cuh"

namespace helm {

enum PeerFlag {
  PF_HALO_READY = 0, PF_HALO_ACK, PF_RED_READY, PF_RED_ACK, PF_GAT_READY, PF_GAT_ACK, PF_ERROR,
  PF_EP_HALO, PF_EP_RED, PF_EP_GAT,   // this rank's epoch counters (device-side, so graph replays advance them)
  PF_COUNT
};
constexpr int PF_STRIDE = 16;                       // one 128-byte line per flag
constexpr size_t PEER_RED_CAP = 2 * 4096 + 8;      // rank-sum slot (complex values)
constexpr long long PEER_TIMEOUT_CYCLES = 20000000000LL;   // ~10 s at 2 GHz

// Byte offsets inside an arena (identical on every rank: computed from the global plan).
struct PeerLayout {
  size_t flags = 0;                 // PF_COUNT * PF_STRIDE uint64
  std::vector<size_t> up, dn;       // per level: outgoing GHOST rows (to rank - 1 / rank + 1)
  size_t red = 0;                   // PEER_RED_CAP complex
  size_t gat = 0, gat_n = 0;        // all-gather slot (complex values)
  size_t bytes = 0;
};

inline PeerLayout peer_layout(const std::vector<int>& nx, int D, const std::vector<DistRows>& plan, int P) {
  PeerLayout L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o += (bytes + 255) / 256 * 256;
    return at;
  };
  L.flags = take(PF_COUNT * PF_STRIDE * sizeof(unsigned long long));
  L.up.assign(nx.size(), 0);
  L.dn.assign(nx.size(), 0);
  for (int l = 0; l <= D; ++l) {
    L.up[l] = take((size_t)GHOST * nx[l] * sizeof(double2));
    L.dn[l] = take((size_t)GHOST * nx[l] * sizeof(double2));
  }
  L.red = take(PEER_RED_CAP * sizeof(double2));
  size_t rows = 0;
  for (int q = 0; q < P; ++q) {
    const DistRows& r = plan[(size_t)(D + 1) * P + q];
    rows = std::max<size_t>(rows, (size_t)(r.b - r.a));
  }
  L.gat_n = rows * nx[D + 1];
  L.gat = take(L.gat_n * sizeof(double2));
  L.bytes = o;
  return L;
}

__device__ __forceinline__ unsigned long long* pflag(char* arena, int f) {
  return reinterpret_cast<unsigned long long*>(arena) + (size_t)f * PF_STRIDE;
}

// (the block has synchronised after its slot writes; thread 0's system-scope fence here orders
// them -- cumulatively, through the barrier -- before the flag)
__device__ __forceinline__ void peer_publish(char* arena, int f, unsigned long long e) {
  __threadfence_system();
  cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> a(*pflag(arena, f));
  a.store(e, cuda::memory_order_release);
}

// thread 0 of the calling block waits until the peer's flag reaches e (acquire); on timeout
// the local error flag is raised and the wait abandoned
__device__ __forceinline__ void peer_wait(char* peer, int f, unsigned long long e, char* me) {
  if (e == 0) return;
  {   // after one timeout every later wait fails fast: the solve ends quickly and reports it
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> err(*pflag(me, PF_ERROR));
    if (err.load(cuda::memory_order_relaxed)) return;
  }
  cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> a(*pflag(peer, f));
  const long long t0 = clock64();
  while (a.load(cuda::memory_order_acquire) < e) {
    if (clock64() - t0 > PEER_TIMEOUT_CYCLES) {
      cuda::atomic_ref<unsigned long long, cuda::thread_scope_system> err(*pflag(me, PF_ERROR));
      err.store(1ull, cuda::memory_order_relaxed);
      return;
    }
    __nanosleep(64);
  }
  __threadfence_system();
}

// producer: epoch of this exchange = counter + 1 (read by every block before the last one
// advances it); consumer: the counter as the producer left it
__device__ __forceinline__ unsigned long long peer_epoch(char* me, int ch) {
  cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> a(*pflag(me, ch));
  return a.load(cuda::memory_order_relaxed);
}

struct PeerSet {
  char* a[DIST_MAX_RANKS];   // every rank's arena, mapped into this process (own arena included)
};

// last CTA to arrive (ticket in `counter`, reset by the last one); every thread's prior writes
// are made visible system-wide first (the peers read them over NVLink)
__device__ __forceinline__ bool peer_last_block(unsigned* counter) {
  __shared__ bool last;
  __syncthreads();   // the block's writes, then one system-scope fence by the signalling thread
  if (threadIdx.x == 0) {
    __threadfence_system();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) *counter = 0u;
  return last;
}

// ---- halo: (1) pack my boundary rows into my arena, publish HALO_READY = e
__global__ void k_peer_halo_put(DVec xv, int nx, int own0, int nown, int up, int dn, PeerSet ps, int me, size_t off_up,
                                size_t off_dn, unsigned* counter) {
  HELM_PDL_ENTRY();
  char* mine = ps.a[me];
  const unsigned long long e = peer_epoch(mine, PF_EP_HALO) + 1;
  if (threadIdx.x == 0) {   // the readers of my previous slots are done (acknowledged epoch e - 1)
    if (up) peer_wait(ps.a[me - 1], PF_HALO_ACK, e - 1, mine);
    if (dn) peer_wait(ps.a[me + 1], PF_HALO_ACK, e - 1, mine);
  }
  __syncthreads();
  const double2* x = xv.get();
  double2* sup = reinterpret_cast<double2*>(mine + off_up);
  double2* sdn = reinterpret_cast<double2*>(mine + off_dn);
  const int n = GHOST * nx;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    if (up) sup[t] = x[(size_t)own0 * nx + t];
    if (dn) sdn[t] = x[(size_t)(own0 + nown - GHOST) * nx + t];
  }
  if (peer_last_block(counter) && threadIdx.x == 0) {
    *pflag(mine, PF_EP_HALO) = e;
    peer_publish(mine, PF_HALO_READY, e);
  }
}

// ---- halo: (2) wait for the neighbours' rows of epoch e, copy them into my ghost rows, ack
__global__ void k_peer_halo_get(DVec xv, int nx, int own0, int nown, int up, int dn, PeerSet ps, int me, size_t off_up,
                                size_t off_dn, unsigned* counter) {
  HELM_PDL_ENTRY();
  char* mine = ps.a[me];
  const unsigned long long e = peer_epoch(mine, PF_EP_HALO);
  if (threadIdx.x == 0) {
    if (up) peer_wait(ps.a[me - 1], PF_HALO_READY, e, mine);
    if (dn) peer_wait(ps.a[me + 1], PF_HALO_READY, e, mine);
  }
  __syncthreads();
  double2* x = xv.get();
  // rank - 1 wrote its bottom rows into its "dn" slot, rank + 1 its top rows into its "up" slot
  const double2* rup = up ? reinterpret_cast<const double2*>(ps.a[me - 1] + off_dn) : nullptr;
  const double2* rdn = dn ? reinterpret_cast<const double2*>(ps.a[me + 1] + off_up) : nullptr;
  const int n = GHOST * nx;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    if (up) x[(size_t)(own0 - GHOST) * nx + t] = __ldcv(rup + t);   // fetched again every time (peer memory: no stale cached line)
    if (dn) x[(size_t)(own0 + nown) * nx + t] = __ldcv(rdn + t);
  }
  if (peer_last_block(counter) && threadIdx.x == 0) peer_publish(mine, PF_HALO_ACK, e);
}

// ---- rank sum of n values (one block each): put my values, then sum every rank's in rank order
__global__ void k_peer_red_put(const double2* __restrict__ buf, int n, PeerSet ps, int me, int P, size_t off_red) {
  HELM_PDL_ENTRY();
  char* mine = ps.a[me];
  const unsigned long long e = peer_epoch(mine, PF_EP_RED) + 1;
  if (threadIdx.x == 0)
    for (int q = 0; q < P; ++q)
      if (q != me) peer_wait(ps.a[q], PF_RED_ACK, e - 1, mine);
  __syncthreads();
  double2* slot = reinterpret_cast<double2*>(mine + off_red);
  for (int i = threadIdx.x; i < n; i += blockDim.x) slot[i] = buf[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    *pflag(mine, PF_EP_RED) = e;
    peer_publish(mine, PF_RED_READY, e);
  }
}

__global__ void k_peer_red_sum(double2* __restrict__ buf, int n, PeerSet ps, int me, int P, size_t off_red) {
  HELM_PDL_ENTRY();
  char* mine = ps.a[me];
  const unsigned long long e = peer_epoch(mine, PF_EP_RED);
  if (threadIdx.x == 0)
    for (int q = 0; q < P; ++q)
      if (q != me) peer_wait(ps.a[q], PF_RED_READY, e, mine);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double2 s = __ldcv(reinterpret_cast<const double2*>(ps.a[0] + off_red) + i);
    for (int q = 1; q < P; ++q) s = cadd(s, __ldcv(reinterpret_cast<const double2*>(ps.a[q] + off_red) + i));
    buf[i] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) peer_publish(mine, PF_RED_ACK, e);
}

struct PeerRows {
  int a[DIST_MAX_RANKS], b[DIST_MAX_RANKS];   // owned rows of the all-gathered level, per rank
};

// ---- all-gather of a replicated level's f: put my owned rows, then fetch every peer's
__global__ void k_peer_gat_put(const double2* __restrict__ f, int nx, PeerRows rows, PeerSet ps, int me, int P,
                               size_t off_gat, unsigned* counter) {
  HELM_PDL_ENTRY();
  char* mine = ps.a[me];
  const unsigned long long e = peer_epoch(mine, PF_EP_GAT) + 1;
  if (threadIdx.x == 0)
    for (int q = 0; q < P; ++q)
      if (q != me) peer_wait(ps.a[q], PF_GAT_ACK, e - 1, mine);
  __syncthreads();
  double2* slot = reinterpret_cast<double2*>(mine + off_gat);
  const long long n = (long long)(rows.b[me] - rows.a[me]) * nx;
  const double2* src = f + (size_t)rows.a[me] * nx;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    slot[t] = src[t];
  if (peer_last_block(counter) && threadIdx.x == 0) {
    *pflag(mine, PF_EP_GAT) = e;
    peer_publish(mine, PF_GAT_READY, e);
  }
}

__global__ void k_peer_gat_get(double2* __restrict__ f, int nx, PeerRows rows, PeerSet ps, int me, int P,
                               size_t off_gat, unsigned* counter) {
  HELM_PDL_ENTRY();
  char* mine = ps.a[me];
  const unsigned long long e = peer_epoch(mine, PF_EP_GAT);
  if (threadIdx.x == 0)
    for (int q = 0; q < P; ++q)
      if (q != me) peer_wait(ps.a[q], PF_GAT_READY, e, mine);
  __syncthreads();
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    const double2* slot = reinterpret_cast<const double2*>(ps.a[q] + off_gat);
    double2* dst = f + (size_t)rows.a[q] * nx;
    const long long n = (long long)(rows.b[q] - rows.a[q]) * nx;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
      dst[t] = __ldcv(slot + t);
  }
  if (peer_last_block(counter) && threadIdx.x == 0) peer_publish(mine, PF_GAT_ACK, e);
}

}  // namespace helm

// ------------------------------------------------------------------ fused Krylov rank sums
// The delayed-CGS2 step of a decomposed inner / outer FGMRES with the two rank sums fused into
// its kernels over peer memory (no separate exchange kernels): the pass-1 reduction publishes
// this rank's dots in its arena; every pass-2 block waits for the peers' dots and sums them (rank
// order) before deriving the coefficients; pass 2's last block publishes the local |w'|^2; the
// step-B kernel sums the norms.  4 kernels per step instead of 8.
namespace helm {

// dynamic shared memory of k_dcgs_update (as helm.cu's dcgs_update_smem), 16-byte aligned
__host__ __device__ inline size_t dcgs_update_smem_dev(int m) {
  const size_t a = (size_t)(2 * m + 2) * sizeof(double2), b = dcgs_smem(m);
  return ((a > b ? a : b) + 15) / 16 * 16;
}

__device__ __forceinline__ void peer_wait_all(const PeerSet& ps, int me, int P, int f, unsigned long long e) {
  for (int q = 0; q < P; ++q)
    if (q != me) peer_wait(ps.a[q], f, e, ps.a[me]);
}

// pass-1 reduction (one warp per output) + publish of this rank's sums (last block)
__global__ void __launch_bounds__(256) k_dcgs_reduce_peer(const double2* __restrict__ part, long long np,
                                                          const FgmState* st, double2* __restrict__ dots,
                                                          unsigned* counter, PeerSet ps, int me, int P,
                                                          size_t off_red) {
  HELM_PDL_ENTRY();
  const int ntot = 2 * (st->j + 1);
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c < ntot) {
    double2 s = make_double2(0.0, 0.0);
    for (long long b = lane; b < np; b += 32) s = cadd(s, part[(long long)c * np + b]);
    s = warp_sum2(s);
    if (lane == 0) dots[c] = s;
  }
  if (!last_block(counter)) return;
  char* mine = ps.a[me];
  __shared__ unsigned long long se;
  if (threadIdx.x == 0) {
    se = peer_epoch(mine, PF_EP_RED) + 1;
    peer_wait_all(ps, me, P, PF_RED_ACK, se - 1);   // every reader of my previous slot is done
  }
  __syncthreads();
  double2* slot = reinterpret_cast<double2*>(mine + off_red);
  for (int i = threadIdx.x; i < ntot; i += blockDim.x) slot[i] = dots[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    *pflag(mine, PF_EP_RED) = se;
    peer_publish(mine, PF_RED_READY, se);
  }
}

// pass 2 with the rank sum of the dots in every block's prologue; extra block 0 runs the
// rotation part of step A (and leaves the summed dots in `dots` for step B); the last block
// acknowledges the dots and publishes this rank's |w'|^2.  Dynamic shared memory:
// dcgs_update_smem(m) + (2m + 4) complex.
__global__ void __launch_bounds__(DU_THREADS, HELM_DU_MINB) k_dcgs_update_peer(
    const double2* __restrict__ V, long long ld, const int* __restrict__ jptr, double2* __restrict__ dots, DVec xv,
    DVec wv, long long n, double2* __restrict__ part, FgmState* st, double2* H, double* cs, double2* sn, double2* g,
    double2* __restrict__ rawc, unsigned* counter, int m, PeerSet ps, int me, int P, size_t off_red) {
  HELM_PDL_ENTRY();
  extern __shared__ double2 sab[];
  double2* sd = sab + (dcgs_update_smem_dev(m) / sizeof(double2));   // summed dots
  __shared__ DuRed<DU_WARPS, DU_ELEMS / 32> red;
  __shared__ double s_beta;
  __shared__ double2 s_hjj;
  __shared__ unsigned long long se;
  char* mine = ps.a[me];
  const int j = *jptr;
  const int ntot = 2 * (j + 1);
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      se = peer_epoch(mine, PF_EP_RED);
      peer_wait_all(ps, me, P, PF_RED_READY, se);
    }
    __syncwarp();
    for (int c = threadIdx.x; c < ntot; c += 32) {
      double2 s = __ldcv(reinterpret_cast<const double2*>(ps.a[0] + off_red) + c);
      for (int q = 1; q < P; ++q) s = cadd(s, __ldcv(reinterpret_cast<const double2*>(ps.a[q] + off_red) + c));
      sd[c] = s;
    }
    __syncwarp();
    dcgs_coefs_warp(j, sd, sab, &s_beta, &s_hjj);
  }
  __syncthreads();
  const bool extra = blockIdx.x == 0;
  const int nb = (int)gridDim.x - 1, tb = (int)blockIdx.x - 1;
  double nrm = 0.0;
  if (extra) {
    for (int c = threadIdx.x; c < ntot; c += blockDim.x) dots[c] = sd[c];   // for step B
    if (threadIdx.x < 32) dcgs_stepA_rot_warp(st, H, cs, sn, g, sd, rawc, s_beta, sab);
  } else {
    const double ib = (1.0 / s_beta) * xv.scale();
    const double2 hjj = s_hjj;
    double2* x = xv.get();
    double2* w = wv.get();
    const long long tiles = (n + DU_ELEMS - 1) / DU_ELEMS;
    for (long long tile = tb; tile < tiles; tile += nb)
      nrm += dcgs_update_tile<DU_WARPS, DU_ELEMS / 32>(V, ld, j, sab, ib, hjj, x, w, n, tile, red);
  }
  const double t = block_sum(nrm);
  if (threadIdx.x == 0) part[blockIdx.x] = make_double2(t, 0.0);
  if (!last_block(counter)) return;
  if (threadIdx.x < 32) {
    double s = 0.0;   // this rank's |w'|^2 (fixed order)
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += part[b].x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) {
      peer_publish(mine, PF_RED_ACK, se);                 // every block of this rank read the dots
      const unsigned long long e2 = se + 1;
      peer_wait_all(ps, me, P, PF_RED_ACK, se);           // and every peer: my slot is free again
      reinterpret_cast<double2*>(mine + off_red)[0] = make_double2(s, 0.0);
      *pflag(mine, PF_EP_RED) = e2;
      peer_publish(mine, PF_RED_READY, e2);
    }
  }
}

// step B after the rank sum of |w'|^2 (one warp); h_jj from the summed dots
__global__ void k_dcgs_stepB_peer(FgmState* st, double2* H, double* cs, double2* sn, double2* g,
                                  const double2* __restrict__ dots, double2* __restrict__ rawc,
                                  cudaGraphConditionalHandle hcond, int use_h, PeerSet ps, int me, int P,
                                  size_t off_red) {
  HELM_PDL_ENTRY();
  extern __shared__ double2 srb[];
  __shared__ double s_beta;
  __shared__ double2 s_hjj;
  __shared__ double2 snorm[1];
  if (threadIdx.x >= 32) return;
  char* mine = ps.a[me];
  if (threadIdx.x == 0) {
    const unsigned long long e2 = peer_epoch(mine, PF_EP_RED);
    peer_wait_all(ps, me, P, PF_RED_READY, e2);
    double2 s = __ldcv(reinterpret_cast<const double2*>(ps.a[0] + off_red));
    for (int q = 1; q < P; ++q) s = cadd(s, __ldcv(reinterpret_cast<const double2*>(ps.a[q] + off_red)));
    snorm[0] = s;
    peer_publish(mine, PF_RED_ACK, e2);
  }
  __syncwarp();
  dcgs_coefs_warp(st->j, dots, srb, &s_beta, &s_hjj);
  __syncwarp();
  dcgs_stepB_warp(st, H, cs, sn, g, dots, s_hjj, snorm, 1, rawc, hcond, use_h, srb);
}

}  // namespace helm
