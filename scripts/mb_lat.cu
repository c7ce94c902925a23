// mb_lat.cu — dependent-chain latencies (cycles per op) on one warp: DFMA, sqrt, 1/x, rsqrt,
// warp REDUX, double shuffle, 5-level double butterfly sum, shared load, __syncthreads (256).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double seed) {
  const int lane = threadIdx.x & 31;
  double x = seed + lane * 1e-3;
  __shared__ double sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  constexpr int N = 256;
  long long t0, t1;
#define TIME(slot, body) \
  t0 = clock64(); for (int i = 0; i < N; ++i) { body; } t1 = clock64(); if (threadIdx.x == 0) cyc[slot] = (t1 - t0) / N;
  TIME(0, x = fma(x, 0.999999, 1e-7));
  TIME(1, x = sqrt(x) + 0.5);
  TIME(2, x = 1.0 / x + 0.5);
  TIME(3, x = rsqrt(x) + 0.5);
  unsigned u = (unsigned)lane;
  TIME(4, u = __reduce_max_sync(0xffffffffu, u + 1));
  TIME(5, x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31) * 0.5 + 0.25);
  TIME(6, { double s = x; for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o); x = s * 1e-3; });
  int idx = lane;
  TIME(7, idx = (int)sm[idx & 63] & 63);
  TIME(8, { __syncthreads(); x += 1.0; });
  TIME(9, x = x * 0.999999 + 1e-7);
  out[threadIdx.x] = x + u + idx;
}
int main() {
  double* o; long long* c;
  cudaMallocManaged(&o, 256 * 8); cudaMallocManaged(&c, 16 * 8);
  for (int r = 0; r < 2; ++r) k<<<1, 256>>>(o, c, 1.5);
  cudaDeviceSynchronize();
  const char* nm[] = {"DFMA", "sqrt+add", "1/x+add", "rsqrt+add", "REDUX max", "shfl.f64+fma", "warp_sum f64 (5 lvl)", "LDS dep", "syncthreads(256)", "DMUL+DADD"};
  for (int i = 0; i < 10; ++i) printf("%-22s %lld cycles\n", nm[i], c[i]);
  return 0;
}
