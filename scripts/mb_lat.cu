// mb_lat.cu — dependent-chain latency of DFMA, DMMA (m8n8k4.f64), FFMA, DADD, DSETP, shfl.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double x, long long* out, double* sink, int n) {
  double a = x + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, 0.999, 1e-3);
  long long t1 = clock64();
  double c0 = a, c1 = -a;
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(x), "d"(0.5));
  long long t2 = clock64();
  float f = (float)a;
  for (int i = 0; i < n; ++i) f = fmaf(f, 0.999f, 1e-3f);
  long long t3 = clock64();
  double s = a;
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, 1e-9);
  long long t4 = clock64();
  double v = a;
  for (int i = 0; i < n; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 0.0;
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / n; out[1] = (t2 - t1) / n; out[2] = (t3 - t2) / n; out[3] = (t4 - t3) / n; out[4] = (t5 - t4) / n;
  }
  sink[threadIdx.x] = a + c0 + c1 + f + s + v;
}
// throughput: many warps, many independent DMMA chains
__global__ void tp(double x, double* sink, int n) {
  double c[8][2];
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = x + j;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(x), "d"(0.5));
  double s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  long long* o; double* sk; cudaMalloc(&o, 64); cudaMalloc(&sk, 1 << 26);
  for (int r = 0; r < 2; ++r) {
    k<<<1, 32>>>(1.0, o, sk, 256);
    long long h[5]; cudaMemcpy(h, o, 40, cudaMemcpyDeviceToHost);
    printf("latency clk: dfma %lld dmma %lld ffma %lld dadd %lld shfl64+dadd %lld\n", h[0], h[1], h[2], h[3], h[4]);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int wpb : {2, 4, 8, 16}) {
    int n = 2000;
    tp<<<148, 32 * wpb>>>(1.0, sk, n);
    cudaEventRecord(e0);
    tp<<<148, 32 * wpb>>>(1.0, sk, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 512.0 * 8 * n * wpb * 148;
    printf("dmma tput warps/SM=%d chains/warp=8: %.1f TF\n", wpb, fl / ms / 1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
