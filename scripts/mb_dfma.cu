// mb_dfma.cu — FP64 CUDA-core (DFMA) throughput on this GPU: many warps x 8 independent
// chains.  The FP64 tensor path (DMMA) is measured by mb_lat.cu / peak_fp64.cu.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int n, double a, double b) {
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x + i;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o;
  cudaMalloc(&o, (size_t)sms * 4 * 1024 * 8);
  const int n = 4096;
  for (int tpb : {256, 512, 1024}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<sms * 2, tpb>>>(o, n, 0.9999, 1e-3);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double fma = (double)sms * 2 * tpb * n * 8;
      if (rep) printf("tpb %d: %.3f ms, %.2f TFLOP/s FP64 FMA (%.1f DFMA/clk/SM at 1.965 GHz)\n", tpb, ms,
                      2 * fma / ms / 1e9, fma / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  return 0;
}
