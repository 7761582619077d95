#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_grid(int nsync, double* buf, int n) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int s = 0; s < nsync; ++s) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) buf[i] = acc + s;
    g.sync();
    acc += buf[(i + 777) % n];
  }
  if (acc == -1.0) buf[0] = 1;
}
__global__ void k_plain(double* buf) { if (threadIdx.x == 9999) buf[0] = 1; }
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  double* buf; cudaMalloc(&buf, 1 << 24);
  for (int bpsm : {1, 2, 4}) for (int threads : {256, 1024}) for (int nsync : {0, 20}) {
    if (threads == 1024 && bpsm > 2) continue;
    int grid = 148 * bpsm; int n = grid * threads;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < 50; ++i) {
      k_plain<<<148, 256, 0, s>>>(buf);
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = grid; cfg.blockDim = threads; cfg.stream = s;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_grid, nsync, buf, n);
    }
    cudaStreamEndCapture(s, &g);
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("inst fail\n"); continue; }
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s); for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid %d x %d nsync %d: %.3f us per (plain + coop) pair; %s\n", grid, threads, nsync, ms * 1e3 / 250, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
