// mb_trinv_blk.cu — phase timing of k_trinv_blk (csrc/k_formw.cu), copied with %globaltimer
// stamps (after 0a zeroing, 0b diagonal blocks, the grid barrier, every level step, the end).
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
constexpr int kTbThreads = 256;
template <typename T>
__global__ void __launch_bounds__(kTbThreads) k_trinv_blk(double* __restrict__ L1, int k, double* __restrict__ Tsc,
                                                          T* __restrict__ LinvT, int64_t ldo, long long* stamps) {
  int ns = 0;
  auto ST = [&]() { if (blockIdx.x == 0 && threadIdx.x == 0) { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); stamps[ns] = t; } ++ns; };
  ST();
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double Ps[32][33], Qs[32][33];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int64_t kk = k;
  // phase 0a: zero the strictly upper triangle (one warp per row)
  for (int64_t i = (int64_t)blockIdx.x * (kTbThreads / 32) + ty; i < kk; i += (int64_t)gridDim.x * (kTbThreads / 32))
    for (int64_t j = i + 1 + tx; j < kk; j += 32) L1[i * kk + j] = 0.0;
  __syncthreads();
  ST();
  // phase 0b: invert the 32 x 32 diagonal blocks in place (lower part only): warp w runs the
  // columns w, w + 8, w + 16, w + 24 together, column-oriented substitution with lane i
  // owning row i (step m: x_m = r_m / L(m,m) broadcast by a shuffle, r_i -= L(i,m) x_m for
  // i > m; for m below a column's start r_m = 0, so every column runs all 32 steps)
  const int nbk = (k + 31) / 32;
  for (int b = blockIdx.x; b < nbk; b += gridDim.x) {
    const int o = 32 * b, cb = min(32, k - o);
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += kTbThreads) {
      const int i = e >> 5, j = e & 31;
      Ps[i][j] = (i < cb && j <= i) ? L1[(int64_t)(o + i) * kk + o + j] : (i == j ? 1.0 : 0.0);
    }
    __syncthreads();
    const double dl = 1.0 / Ps[tx][tx];   // lane tx: 1 / L(tx, tx)
    double r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) r[u] = (tx == ty + 8 * u) ? 1.0 : 0.0;
    for (int m = 0; m < 32; ++m) {
      const double dm = __shfl_sync(0xffffffffu, dl, m);
      const double lim = Ps[tx][m];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double xm = __shfl_sync(0xffffffffu, r[u], m) * dm;
        r[u] = tx == m ? xm : (tx > m ? fma(-lim, xm, r[u]) : r[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) Qs[tx][ty + 8 * u] = r[u];   // x_i of column j = ty + 8u at row tx
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += kTbThreads) {
      const int i = e >> 5, j = e & 31;
      if (i < cb && j <= i) L1[(int64_t)(o + i) * kk + o + j] = Qs[i][j];
    }
  }
  __syncthreads();
  ST();
  grid.sync();
  ST();
  for (int sb = 32; sb < k; sb *= 2) {
    const int npair = (k + 2 * sb - 1) / (2 * sb);
    const int tps = sb / 32;   // 32-wide tiles per s
    // step 1: T(p) = B A^{-1}, B = L1(C rows, A cols): cs x s, A^{-1} lower (m >= c)
    // step 2: L1(C, A) = -C^{-1} T(p): C^{-1} lower (m <= r)
    for (int step = 0; step < 2; ++step) {
      for (int64_t w = blockIdx.x;; w += gridDim.x) {
        // work item w -> (pair p, row tile rt, column tile ct)
        int p = 0;
        int64_t ww = w;
        int cs = 0, rtiles = 0;
        for (; p < npair; ++p) {
          const int c0 = 2 * p * sb + sb;
          cs = c0 < k ? min(sb, k - c0) : 0;
          rtiles = (cs + 31) / 32;
          const int64_t items = (int64_t)rtiles * tps;
          if (ww < items) break;
          ww -= items;
        }
        if (p >= npair) break;
        const int rt = (int)(ww / tps), ct = (int)(ww - (int64_t)rt * tps);
        const int a0 = 2 * p * sb, c0 = a0 + sb;
        double* Tp = Tsc + (int64_t)p * sb * sb;   // [cs][sb]
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const int c = 32 * ct + tx;
        // K range: step 1: m in [32 ct, sb) (A^{-1}(m, c) = 0 for m < c);
        //          step 2: m in [0, 32 rt + 32) (C^{-1}(r, m) = 0 for m > r)
        const int mlo = step == 0 ? 32 * ct : 0;
        const int mhi = step == 0 ? sb : min(cs, 32 * rt + 32);
        for (int m0 = mlo; m0 < mhi; m0 += 32) {
          __syncthreads();
          for (int e = tid; e < 32 * 32; e += kTbThreads) {
            const int i = e >> 5, j = e & 31;
            const int r = 32 * rt + i, m = m0 + j, mr = m0 + i, cc = 32 * ct + j;
            double pv = 0.0, qv = 0.0;
            if (step == 0) {
              if (r < cs && m < mhi) pv = L1[(int64_t)(c0 + r) * kk + a0 + m];           // B(r, m)
              if (mr < mhi) qv = L1[(int64_t)(a0 + mr) * kk + a0 + cc];                  // A^{-1}(mr, cc)
            } else {
              if (r < cs && m < mhi) pv = L1[(int64_t)(c0 + r) * kk + c0 + m];           // C^{-1}(r, m)
              if (mr < mhi) qv = Tp[(int64_t)mr * sb + cc];                              // T(mr, cc)
            }
            Ps[i][j] = pv;
            Qs[i][j] = qv;
          }
          __syncthreads();
#pragma unroll 8
          for (int mm = 0; mm < 32; ++mm) {
            const double q = Qs[mm][tx];
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = fma(Ps[ty + 8 * u][mm], q, acc[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = 32 * rt + ty + 8 * u;
          if (r < cs) {
            if (step == 0) Tp[(int64_t)r * sb + c] = acc[u];
            else L1[(int64_t)(c0 + r) * kk + a0 + c] = -acc[u];
          }
        }
      }
      grid.sync();
      ST();
    }
  }
  // final: LinvT (k x ldo) = L_1^{-T}, zero above the diagonal and in the padding
  for (int64_t e = (int64_t)blockIdx.x * kTbThreads + tid; e < kk * ldo; e += (int64_t)gridDim.x * kTbThreads) {
    const int64_t j = e / ldo, i = e - j * ldo;
    LinvT[e] = (i >= j && i < kk) ? (T)L1[i * kk + j] : T(0);
  }
  __syncthreads();
  ST();
}


int main() {
  for (int k : {128, 240, 512}) {
    std::vector<double> h((size_t)k * k);
    for (int i = 0; i < k; ++i)
      for (int m = 0; m < k; ++m) h[(size_t)i * k + m] = m > i ? 0.0 : (m == i ? 1.0 : 0.01 * ((i * 7 + m * 3) % 11 - 5));
    double *L, *T, *LT;
    long long* st;
    cudaMalloc(&L, (size_t)k * k * 8);
    cudaMalloc(&T, (size_t)k * k * 8);
    cudaMalloc(&LT, (size_t)k * k * 8);
    cudaMalloc(&st, 64 * 8);
    for (int grid : {16, 64, 148}) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(L, h.data(), (size_t)k * k * 8, cudaMemcpyHostToDevice);
        cudaMemset(st, 0, 64 * 8);
        int ki = k;
        int64_t ldo = k;
        void* args[] = {&L, &ki, &T, &LT, &ldo, &st};
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_trinv_blk<double>, dim3(grid), dim3(kTbThreads), args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        long long hs[64];
        cudaMemcpy(hs, st, sizeof(hs), cudaMemcpyDeviceToHost);
        if (rep < 2) continue;
        printf("k=%d grid=%d err=%s kernel %.1f us; stamps (us):", k, grid, cudaGetErrorString(e), ms * 1e3);
        for (int i = 1; i < 16 && hs[i] > hs[0]; ++i) printf(" %.1f", (hs[i] - hs[0]) * 1e-3);
        printf("\n");
      }
    }
  }
  return 0;
}
