// mb_factor.cu — microbenchmark of the a3 factorisation pieces on one CTA (clock64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -o /tmp/mb scripts/mb_factor.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2309_16002_b200/csrc/k_filter_coop.cu"

using namespace rbrp;

__global__ void mb(const double* G, int nb, long long* out, double* sink) {
  __shared__ double A[32 * 33], R[32 * 33], T[32 * 33];
  __shared__ int perm[128], ch[128];
  __shared__ double mass[128], dg[128];
  __shared__ int rd;
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += blockDim.x) A[(e / nb) * 33 + e % nb] = G[e];
  __syncthreads();
  long long t0 = clock64();
  int kept = cta_pivchol(A, 33, nb, 1, nullptr, 1.0 / nb, R, 33, perm, mass, dg, ch, &rd);
  long long t1 = clock64();
  cta_trinv(R, 33, perm, kept, T, 33);
  long long t2 = clock64();
  // barrier-only loop
  for (int i = 0; i < 3 * nb; ++i) __syncthreads();
  long long t3 = clock64();
  // warp argmax only
  double acc = 0;
  if (tid < 32) {
    for (int i = 0; i < nb; ++i) {
      double x = dg[(tid + i) % nb];
      double m = warp_sum(x);
      acc += m;
    }
  }
  __syncthreads();
  long long t4 = clock64();
  if (tid == 0) {
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = kept;
    sink[0] = acc + T[0];
  }
}

int main() {
  const int nb = 32;
  double h[nb * nb];
  // SPD: G = B^T B + I
  double B[nb * nb];
  for (int i = 0; i < nb * nb; ++i) B[i] = ((i * 7919) % 1000) / 1000.0 - 0.5;
  for (int i = 0; i < nb; ++i)
    for (int j = 0; j < nb; ++j) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int k = 0; k < nb; ++k) s += B[k * nb + i] * B[k * nb + j];
      h[i * nb + j] = s;
    }
  double *dG, *sink;
  long long* dout;
  cudaMalloc(&dG, sizeof(h));
  cudaMalloc(&dout, 64);
  cudaMalloc(&sink, 64);
  cudaMemcpy(dG, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    mb<<<1, 256>>>(dG, nb, dout, sink);
    long long o[5];
    cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost);
    printf("pivchol %lld clk, trinv %lld clk, 96 syncthreads %lld clk, 32 warp_sums %lld clk, kept %lld\n",
           o[0], o[1], o[2], o[3], o[4]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
