// mb_trinv.cu — cycle breakdown of k_trinv_small's column-axpy substitution (csrc/k_formw.cu):
// load phase vs substitution loop, per warp, k = 128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_trinv scripts/mb_trinv.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
constexpr int KMAX = 160, W = 8, U = (KMAX + 31) / 32;
__global__ void __launch_bounds__(256) k(const double* __restrict__ L1, int kk, double* out, long long* cyc) {
  extern __shared__ double ts_[];
  const int ld = kk + 1;
  double* Lt = ts_;
  double* dinv = Lt + (size_t)kk * ld;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j0 = blockIdx.x * W;
  long long t0 = clock64();
#pragma unroll 2
  for (int i = j0 + w; i < kk; i += W) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int m = lane + 32 * u;
      v[u] = m <= i ? L1[(long)i * kk + m] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int m = lane + 32 * u;
      if (m <= i) Lt[(long)m * ld + i] = v[u];
    }
  }
  __syncthreads();
  for (int i = j0 + threadIdx.x; i < kk; i += blockDim.x) dinv[i] = 1.0 / Lt[(long)i * ld + i];
  __syncthreads();
  long long t1 = clock64();
  const int j = j0 + w;
  const int Ur = (kk + 31) >> 5;
  double r[U];
#pragma unroll
  for (int u = 0; u < U; ++u) r[u] = (lane + 32 * u == j) ? 1.0 : 0.0;
#ifdef PIPE
  // software-pipelined: column m + 1 and 1/L(m+1,m+1) are loaded during step m
  const uint32_t lt_s = (uint32_t)__cvta_generic_to_shared(Lt), dv_s = (uint32_t)__cvta_generic_to_shared(dinv);
  auto lds = [](uint32_t a) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
  };
  long long ph0 = 0, ph1 = 0;
  double cn[U], dn = lds(dv_s + 8 * j);
#pragma unroll
  for (int u = 0; u < U; ++u) cn[u] = u < Ur ? lds(lt_s + 8 * (j * ld + min(lane + 32 * u, kk - 1))) : 0.0;
  for (int m = j; m < kk; ++m) {
    double cv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cv[u] = cn[u];
    const double dm = dn;
    if (m + 1 < kk) {
      dn = lds(dv_s + 8 * (m + 1));
#pragma unroll
      for (int u = 0; u < U; ++u) cn[u] = u < Ur ? lds(lt_s + 8 * ((m + 1) * ld + min(lane + 32 * u, kk - 1))) : 0.0;
    }
    long long a0 = clock64();
    const int um = m >> 5;
    double v = r[0];
#pragma unroll
    for (int u = 1; u < U; ++u)
      if (u == um) v = r[u];
    const double sv = __shfl_sync(0xffffffffu, v, m & 31);
    long long a1 = clock64();
    const double xm = sv * dm;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = lane + 32 * u;
      const double t = fma(-cv[u], xm, r[u]);
      r[u] = i == m ? xm : ((i > m && i < kk) ? t : r[u]);
    }
    long long a2 = clock64();
    ph0 += a1 - a0;
    ph1 += a2 - a1;
  }
  if (lane == 0 && blockIdx.x == 0 && w == 0) { cyc[2 * kk + 0] = ph0; cyc[2 * kk + 1] = ph1; }
#else
  for (int m = j; m < kk; ++m) {
    const int um = m >> 5;
    double v = r[0];
#pragma unroll
    for (int u = 1; u < U; ++u)
      if (u == um) v = r[u];
    const double* col = Lt + (long)m * ld;
    double cv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cv[u] = u < Ur ? col[min(lane + 32 * u, kk - 1)] : 0.0;
    const double xm = __shfl_sync(0xffffffffu, v, m & 31) * dinv[m];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = lane + 32 * u;
      const double t = fma(-cv[u], xm, r[u]);
      r[u] = i == m ? xm : ((i > m && i < kk) ? t : r[u]);
    }
  }
#endif
  long long t2 = clock64();
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int i = lane + 32 * u;
    if (i < kk) out[(long)j * kk + i] = i < j ? 0.0 : r[u];
  }
  if (lane == 0) {
    cyc[(blockIdx.x * W + w) * 2] = t1 - t0;
    cyc[(blockIdx.x * W + w) * 2 + 1] = t2 - t1;
  }
}
int main() {
  const int kk = 128;
  double *L, *out;
  long long* cyc;
  cudaMallocManaged(&L, kk * kk * 8);
  cudaMallocManaged(&out, kk * kk * 8);
  cudaMallocManaged(&cyc, 2 * kk * 8 + 64);
  for (int i = 0; i < kk; ++i)
    for (int m = 0; m < kk; ++m) L[i * kk + m] = m > i ? 0.0 : (m == i ? 1.0 : 0.01 * ((i * 7 + m * 3) % 11 - 5));
  const int sb = (kk * (kk + 1) + kk) * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<kk / W, 256, sb>>>(L, kk, out, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("kernel %.1f us; warp 0: load %lld cyc, loop %lld cyc (%lld/step); warp 127: load %lld loop %lld\n", ms * 1e3,
           cyc[0], cyc[1], cyc[1] / kk, cyc[2 * 127], cyc[2 * 127 + 1]);
  }
  printf("phases (warp 0, per step): select+shfl %lld, mul+update %lld\n", cyc[2 * kk] / kk, cyc[2 * kk + 1] / kk);
  // check L * Linv^T ~ I on a few entries
  double err = 0;
  for (int i = 0; i < kk; ++i)
    for (int j = 0; j < kk; ++j) {
      double s = 0;
      for (int m = 0; m < kk; ++m) s += L[i * kk + m] * out[j * kk + m];
      err = fmax(err, fabs(s - (i == j)));
    }
  printf("max |L Linv - I| = %.3e\n", err);
  return 0;
}
