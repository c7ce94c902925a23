// mb_pdl.cu — per-kernel overhead of a chain of small dependent kernels captured in a CUDA
// graph, with and without programmatic dependent launch (griddepcontrol.wait at entry,
// launch_dependents right after).  Each kernel: 1 CTA or 148 CTAs, reads a value the
// previous one wrote (correctness check), ~1 us of work.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kstep(int* buf, int i, int pdl, int spin) {
  if (pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
  }
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (buf[0] != i) buf[1] = 1;   // ordering violated
    buf[0] = i + 1;
  }
}
int main() {
  int* buf;
  cudaMalloc(&buf, 8);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int grid : {1, 148})
    for (int spin : {0, 2000})
      for (int pdl = 0; pdl < 2; ++pdl) {
        const int N = 40;
        cudaMemset(buf, 0, 8);
        cudaGraph_t g;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < N; ++i) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(grid);
          cfg.blockDim = dim3(256);
          cfg.stream = s;
          cudaLaunchAttribute la[1];
          la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          la[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = la;
          cfg.numAttrs = pdl ? 1 : 0;
          cudaLaunchKernelEx(&cfg, kstep, buf, i, pdl, spin);
        }
        cudaStreamEndCapture(s, &g);
        cudaGraphExec_t ge;
        cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
        if (e != cudaSuccess) { printf("instantiate: %s\n", cudaGetErrorString(e)); return 1; }
        for (int w = 0; w < 3; ++w) { cudaMemset(buf, 0, 8); cudaGraphLaunch(ge, s); }
        cudaStreamSynchronize(s);
        cudaMemset(buf, 0, 8);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        int h[2];
        cudaMemcpy(h, buf, 8, cudaMemcpyDeviceToHost);
        printf("grid %3d spin %5d pdl %d: %.2f us per kernel (final %d, violations %d) %s\n", grid, spin, pdl,
               ms * 1e3 / N, h[0], h[1], cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
