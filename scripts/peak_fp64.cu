// peak_fp64.cu — measure the B200 FP64 peaks that MEASURED_PEAKS.json lacks:
//   DFMA (CUDA cores) and DMMA (mma.sync.m8n8k4.f64, legacy tensor path).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peak_fp64 scripts/peak_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8, iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * (double)threads * blocks;
    if (rep) printf("{\"dfma_tflops\": %.2f, ", fl / ms / 1e9);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per warp per mma: 8*8*4 FMA = 256 FMA = 512 flop
    double fl = 512.0 * 8 * (iters / 4) * (threads / 32.0) * blocks;
    if (rep) printf("\"dmma_tflops\": %.2f, \"sms\": %d}\n", fl / ms / 1e9, sms);
  }
  cudaError_t e = cudaGetLastError();
  if (e) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
