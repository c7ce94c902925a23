// mb_factor2.cu — per-phase cycle counts of one right-looking pivoted Cholesky step.
#include <cstdio>
#include <cfloat>
#include <cuda_runtime.h>
__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__global__ void mb(const double* G, int nb, long long* out, double* sink) {
  __shared__ double A[32 * 33], R[32 * 33], dg[32];
  __shared__ int chosen[32], s_p;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int lda = 33, ldr = 33;
  for (int e = tid; e < nb * nb; e += blockDim.x) A[(e / nb) * lda + e % nb] = G[e];
  for (int l = tid; l < nb; l += blockDim.x) { dg[l] = G[l * nb + l]; chosen[l] = 0; }
  __syncthreads();
  long long ta = 0, tb = 0, tc = 0, td = 0;
  for (int i = 0; i < nb; ++i) {
    long long t0 = clock64();
    if (w == 0) {
      double ms = 0.0, best = -DBL_MAX; int bl = 1 << 30;
      for (int l = lane; l < nb; l += 32) {
        if (chosen[l]) continue;
        const double x = dg[l];
        ms += fmax(x, 0.0);
        if (x > best) { best = x; bl = l; }
      }
      ms = wsum(ms);
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (ob > best || (ob == best && ol < bl)) { best = ob; bl = ol; }
      }
      if (lane == 0) { s_p = bl; sink[1] = ms; }
    }
    __syncthreads();
    long long t1 = clock64();
    const int p = s_p;
    const double rii = sqrt(dg[p]);
    long long t2 = clock64();
    for (int l = tid; l < nb; l += blockDim.x) {
      double v;
      if (l == p) v = rii; else if (chosen[l]) v = 0.0; else v = A[p * lda + l] / rii;
      R[i * ldr + l] = v;
    }
    __syncthreads();
    long long t3 = clock64();
    if (tid == 0) chosen[p] = 1;
    for (int e = tid; e < nb * nb; e += blockDim.x) {
      const int r = e / nb, c = e % nb;
      if (r == p || c == p) continue;
      const double rr = R[i * ldr + r], rc = R[i * ldr + c];
      const double a = fma(-rr, rc, A[r * lda + c]);
      A[r * lda + c] = a;
      if (r == c) dg[r] = a;
    }
    __syncthreads();
    long long t4 = clock64();
    ta += t1 - t0; tb += t2 - t1; tc += t3 - t2; td += t4 - t3;
  }
  if (tid == 0) { out[0] = ta; out[1] = tb; out[2] = tc; out[3] = td; }
}
// division / sqrt latency
__global__ void lat(double x, long long* out, double* sink) {
  double a = x; long long t0 = clock64();
  for (int i = 0; i < 64; ++i) a = 1.0 / (a + 1.0);
  long long t1 = clock64();
  double b = x;
  for (int i = 0; i < 64; ++i) b = sqrt(b + 1.0);
  long long t2 = clock64();
  double c = x;
  for (int i = 0; i < 64; ++i) c = fma(c, 0.999, 1e-3);
  long long t3 = clock64();
  out[0] = (t1 - t0) / 64; out[1] = (t2 - t1) / 64; out[2] = (t3 - t2) / 64;
  sink[0] = a + b + c;
}
int main() {
  const int nb = 32;
  double h[nb * nb], B[nb * nb];
  for (int i = 0; i < nb * nb; ++i) B[i] = ((i * 7919) % 1000) / 1000.0 - 0.5;
  for (int i = 0; i < nb; ++i) for (int j = 0; j < nb; ++j) {
    double s = (i == j) ? 1.0 : 0.0;
    for (int k = 0; k < nb; ++k) s += B[k * nb + i] * B[k * nb + j];
    h[i * nb + j] = s; }
  double *dG, *sink; long long* dout;
  cudaMalloc(&dG, sizeof(h)); cudaMalloc(&dout, 64); cudaMalloc(&sink, 64);
  cudaMemcpy(dG, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    mb<<<1, 256>>>(dG, nb, dout, sink);
    long long o[4]; cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost);
    printf("per 32 steps: argmax %lld, sqrt %lld, Rrow(div) %lld, schur %lld clk\n", o[0], o[1], o[2], o[3]);
    lat<<<1, 1>>>(0.5, dout, sink);
    cudaMemcpy(o, dout, 24, cudaMemcpyDeviceToHost);
    printf("latency: div %lld sqrt %lld dfma %lld clk\n", o[0], o[1], o[2]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
