#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int* p) { if (p && threadIdx.x == 1234567) p[0] = 1; }
__global__ void k_pdl(int* p) { asm volatile("griddepcontrol.wait;" ::: "memory"); asm volatile("griddepcontrol.launch_dependents;"); if (p && threadIdx.x == 1234567) p[0] = 1; }
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int blocks : {1, 148, 800}) for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < 200; ++i) {
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = blocks; cfg.blockDim = 256; cfg.stream = s;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = pdl;
      cfg.attrs = at; cfg.numAttrs = 1;
      if (pdl) cudaLaunchKernelEx(&cfg, k_pdl, (int*)nullptr); else cudaLaunchKernelEx(&cfg, k_empty, (int*)nullptr);
    }
    cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s); for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("blocks %d pdl %d: %.3f us per kernel\n", blocks, pdl, ms * 1e3 / 1000);
  }
  return 0;
}
