// mb_dmma_occ.cu — DMMA throughput vs warps per SM and independent accumulator chains
// per warp (how much occupancy / ILP the projection tiles need on B200).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_dmma_occ scripts/mb_dmma_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// same with a shared-memory fragment load (LDS.128) per 2 MMAs, like the projection tiles
template <int CH>
__global__ void dmma_lds_kernel(double* out, int iters) {
  __shared__ double2 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(i * 1e-3, 1.0);
  __syncthreads();
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    double2 a = sm[(lane + it) & 1023];
    double2 b[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) b[i] = sm[(lane * 3 + i * 32 + it) & 1023];
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a.x), "d"(b[i].x));
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a.y), "d"(b[i].y));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CH, bool LDS>
void run(int sms, int warps, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    if (LDS) dmma_lds_kernel<CH><<<sms, 32 * warps>>>(out, iters);
    else dmma_kernel<CH><<<sms, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const double mmas = (LDS ? 2.0 : 1.0) * CH * iters * (double)warps * sms;
  printf("{\"lds\": %d, \"warps_per_sm\": %d, \"chains\": %d, \"tflops\": %.2f}\n", LDS, warps, CH,
         512.0 * mmas / ms / 1e9);
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 12, 16, 32}) {
    run<2, false>(sms, w, out);
    run<4, false>(sms, w, out);
    run<8, false>(sms, w, out);
    run<16, false>(sms, w, out);
    run<2, true>(sms, w, out);
    run<4, true>(sms, w, out);
    run<8, true>(sms, w, out);
  }
  return 0;
}
