// mb_factor3.cu — cycles of cta_chol_inv (fast path) on one CTA.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2309_16002_b200/csrc/k_filter_coop.cu"
using namespace rbrp;
namespace rbrp {
template <int EPT>
__device__ int cta_chol_inv_t(const double* __restrict__ Gg, int nb, int mode, const int32_t* forced,
                            double tau_b, double* R, int ld, double* Tm, int ldt, int* perm,
                            double* mass, double* dg, int* chosen, int* rank_def, long long* tt) {
  long long t_a = 0, t_b = 0, t_c = 0;
  __shared__ int s_p, s_cut;
  __shared__ double s_rii, s_inv;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  double thr = 0.0;
  int er[EPT], ec[EPT];
  double a[EPT], ta[EPT];
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int e = tid + k * blockDim.x;
    if (e < nb * nb) {
      er[k] = e / nb;
      ec[k] = e - er[k] * nb;
      a[k] = Gg[er[k] * kMaxB + ec[k]];
      if (er[k] == ec[k]) dg[er[k]] = a[k];
    } else {
      er[k] = -1;
      ec[k] = -1;
      a[k] = 0.0;
    }
    ta[k] = 0.0;
  }
  for (int e = tid; e < nb * ldt; e += blockDim.x) Tm[e] = 0.0;
  for (int l = tid; l < nb; l += blockDim.x) chosen[l] = 0;
  if (tid == 0) *rank_def = 0;
  __syncthreads();
  int kept = nb;
  for (int i = 0; i < nb; ++i) {
    long long c0 = clock64();
    if (w == 0) {
      double ms = 0.0, best = -DBL_MAX;
      int bl = 1 << 30;
      for (int l = lane; l < nb; l += 32) {
        if (chosen[l]) continue;
        const double x = dg[l];
        ms += fmax(x, 0.0);
        if (x > best) { best = x; bl = l; }
      }
      ms = warp_sum(ms);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (ob > best || (ob == best && ol < bl)) { best = ob; bl = ol; }
      }
      // all fp64 arithmetic warp-uniform (single-lane fp64 is very slow); lane 0 stores
      if (i == 0) thr = tau_b * ms;
      int cut = 0;
      if (mode == 1 && (!(ms > 0.0) || ms < thr)) cut = 1;          // l.8 cut
      int p = bl;
      if (mode == 2) p = i;
      if (mode == 1 && forced) p = forced[i];
      const double dp = dg[p];
      if (!cut && !(dp > 0.0)) cut = 2;                             // non-positive pivot
      const double rii = sqrt(fmax(dp, 0.0));
      const double inv = 1.0 / rii;
      if (lane == 0) {
        if (mode == 1) mass[i] = ms;
        if (!cut) {
          s_rii = rii;
          s_inv = inv;
          perm[i] = p;
          Tm[i * ldt + i] = inv;
        }
        s_p = p;
        s_cut = cut;
      }
    }
    __syncthreads();
    long long c1 = clock64(); t_a += c1 - c0;
    if (s_cut) {
      if (tid == 0 && s_cut == 2) *rank_def = 1;
      kept = i;
      break;
    }
    const int p = s_p;
    const double inv = s_inv, rii = s_rii;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int c = ec[k];
      const double rv = a[k] * inv, tv = -ta[k] * inv;   // computed by every lane
      if (er[k] == p) R[i * ld + c] = (c == p) ? rii : (chosen[c] ? 0.0 : rv);   // row i of R
      if (c == p && er[k] < i) Tm[er[k] * ldt + i] = tv;                        // column i of T
    }
    __syncthreads();
    long long c2 = clock64(); t_b += c2 - c1;
    if (tid == 0) chosen[p] = 1;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int r = er[k], c = ec[k];
      if (r < 0) continue;
      const double ric = R[i * ld + c];
      a[k] = fma(-R[i * ld + r], ric, a[k]);
      if (r == c) dg[r] = a[k];
      if (r <= i) ta[k] = fma(Tm[r * ldt + i], ric, ta[k]);
    }
    __syncthreads();
    t_c += clock64() - c2;
  }
  if (threadIdx.x == 0) { tt[0] = t_a; tt[1] = t_b; tt[2] = t_c; }
  __syncthreads();
  return kept;
}

}

__global__ void __launch_bounds__(256, 1) mb(const double* G, int nb, int mode, long long* out) {
  __shared__ double R[32 * 33], T[32 * 33], mass[128], dg[128];
  __shared__ int perm[128], ch[128], rd;
  long long t0 = clock64();
  int kept = cta_chol_inv_t<4>(G, nb, mode, nullptr, 1.0 / nb, R, 33, T, 33, perm, mass, dg, ch, &rd, out + 2);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = kept; }
}
int main() {
  const int nb = 32;
  static double h[128 * 128];
  double B[nb * nb];
  for (int i = 0; i < nb * nb; ++i) B[i] = ((i * 7919) % 1000) / 1000.0 - 0.5;
  for (int i = 0; i < nb; ++i) for (int j = 0; j < nb; ++j) {
    double s = (i == j) ? 1.0 : 0.0;
    for (int k = 0; k < nb; ++k) s += B[k * nb + i] * B[k * nb + j];
    h[i * 128 + j] = s; }
  double* dG; long long* o; cudaMalloc(&dG, sizeof(h)); cudaMalloc(&o, 64);
  cudaMemcpy(dG, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int mode = 1; mode <= 2; ++mode) for (int r = 0; r < 2; ++r) {
    mb<<<1, 256>>>(dG, nb, mode, o);
    long long hh[5]; cudaMemcpy(hh, o, 40, cudaMemcpyDeviceToHost);
    printf("mode %d: %lld clk for %lld steps (%.0f per step) argmax %lld rrow %lld schur %lld\n", mode, hh[0], hh[1], (double)hh[0] / hh[1], hh[2], hh[3], hh[4]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
