#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_cl(int nsync, int* out) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  double acc = 0;
  for (int s = 0; s < nsync; ++s) {
    sm[threadIdx.x] = acc + s;
    cl.sync();
    const double* rem = cl.map_shared_rank(sm, (cl.block_rank() + 1) % cl.num_blocks());
    acc += rem[threadIdx.x];
    cl.sync();
  }
  if (acc == -1.0) out[0] = 1;
}
__global__ void k_plain(int* out) { if (threadIdx.x == 9999) out[0] = 1; }
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaFuncSetAttribute(k_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int cs : {8, 16}) for (size_t smem : {(size_t)16384, (size_t)200 * 1024}) for (int nsync : {0, 10, 40}) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < 50; ++i) {
      k_plain<<<148, 256, 0, s>>>(nullptr);
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = cs; cfg.blockDim = 1024; cfg.dynamicSmemBytes = smem; cfg.stream = s;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_cl, nsync, (int*)nullptr);
    }
    cudaStreamEndCapture(s, &g);
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("inst fail %s\n", cudaGetErrorString(cudaGetLastError())); continue; }
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s); for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cluster %d smem %zu nsync %d: %.3f us per (plain + cluster) pair; err %s\n", cs, smem, nsync, ms * 1e3 / 250, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
