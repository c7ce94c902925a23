// k_formw.cu — a6 interpolation matrix, Alg. 3.
//
// L_1 = L(S,:) is exactly lower-triangular in selection order (reading R13), so
// L_2 L_1^{-1} is a triangular solve (north_star step 6).  We form
// L_1^{-1} once (k_trinv: one warp per column, forward substitution in fp64), then
// W = L L_1^{-1} for all local rows with the tile GEMM (k_gemm_nt, B = L_1^{-T}), and
// finally W(S,:) = I exactly (Alg. 3 l.2).  W_CLIPPED is reported when
// min |diag L_1| < 1e-12 max |diag L_1| (Remark 5.2, reading R17).
#include <float.h>

#include "launch.cuh"

namespace rbrp {

template <typename T>
__global__ void k_gather_L1(const T* __restrict__ L, int64_t ldl, const int64_t* __restrict__ S,
                            int64_t k, int64_t n_local, int64_t row_offset, double* __restrict__ L1) {
  const int64_t i = blockIdx.x;
  const int64_t r = S[i] - row_offset;
  if (r < 0 || r >= n_local) return;   // another rank's skeleton (zeroed / shared buffer)
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) L1[i * k + j] = (double)L[r * ldl + j];
}

template <typename T>
cudaError_t launch_gather_L1(const T* L, int64_t ldl, const int64_t* S, int64_t k, int64_t n_local,
                             int64_t row_offset, double* L1, cudaStream_t s) {
  if (k <= 0) return cudaSuccess;
  k_gather_L1<T><<<(unsigned)k, 256, 0, s>>>(L, ldl, S, k, n_local, row_offset, L1);
  return cudaGetLastError();
}

constexpr int kTrinvWarps = 4;

// Column j of L_1^{-1}: x_j = 1/L(j,j); x_i = -(sum_{j<=m<i} L(i,m) x_m) / L(i,i).
// Written transposed: LinvT(j, m) = x_m (zeros for m < j).
template <typename T>
__global__ void __launch_bounds__(32 * kTrinvWarps) k_trinv(const double* __restrict__ L1, int64_t k,
                                                            T* __restrict__ LinvT, int64_t ldo, DevState* st) {
  extern __shared__ double xs[];   // [kTrinvWarps][k]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * kTrinvWarps + w;
  if (blockIdx.x == 0 && w == 0) {
    double mx = 0.0, mn = DBL_MAX;
    for (int64_t i = lane; i < k; i += 32) {
      const double a = fabs(L1[i * k + i]);
      mx = fmax(mx, a);
      mn = fmin(mn, a);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (lane == 0 && mn < 1e-12 * mx) atomicOr(&st->flags, (uint32_t)RBRP_F_W_CLIPPED);
  }
  if (j >= k) return;
  double* x = xs + (int64_t)w * k;
  const double xj = 1.0 / L1[j * k + j];   // fp64 math warp-uniform (single-lane fp64 is slow)
  if (lane == 0) x[j] = xj;
  __syncwarp();
  // row i's segment L(i, j..i-1) (the first 32 NB of it) is loaded one step ahead, so
  // the L2 latency overlaps the previous step's dot product and butterfly
  constexpr int NB = 16;
  double cur[NB], nxt[NB];
  auto load_row = [&](int64_t i, double* buf) {
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int64_t m = j + lane + 32 * u;
      buf[u] = m < i ? L1[i * k + m] : 0.0;
    }
  };
  double dnext = 1.0;
  if (j + 1 < k) {
    load_row(j + 1, cur);
    dnext = L1[(j + 1) * k + j + 1];
  }
  for (int64_t i = j + 1; i < k; ++i) {
    const double dii = dnext;
    if (i + 1 < k) {
      load_row(i + 1, nxt);
      dnext = L1[(i + 1) * k + i + 1];
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int64_t m = j + lane + 32 * u;
      if (m < i) s += cur[u] * x[m];
    }
    for (int64_t m = j + 32 * NB + lane; m < i; m += 32) s += L1[i * k + m] * x[m];
    s = warp_sum(s);
    const double xi = -s / dii;
    if (lane == 0) x[i] = xi;
    __syncwarp();
#pragma unroll
    for (int u = 0; u < NB; ++u) cur[u] = nxt[u];
  }
  for (int64_t m = lane; m < ldo; m += 32) LinvT[j * ldo + m] = (m < j || m >= k) ? T(0) : (T)x[m];
}

// Small k (L_1 fits in shared memory): L_1 staged once per CTA (rows only from the CTA's
// first column on), one warp per column j of L_1^{-1} as in k_trinv, but every operand of
// the substitution step now comes from shared memory and 1/L(i,i) is precomputed, so a
// step costs one shared-memory dot product + butterfly instead of an L2 round trip.
constexpr int kTrinvSmallK = 160;   // k^2 + (k + 8 k) doubles of shared memory
constexpr int kTrinvSmallWarps = 8;
template <typename T>
__global__ void __launch_bounds__(32 * kTrinvSmallWarps) k_trinv_small(const double* __restrict__ L1, int64_t k,
                                                                       T* __restrict__ LinvT, int64_t ldo,
                                                                       DevState* st) {
  extern __shared__ double ts_[];
  const int kk = (int)k;
  double* Ls = ts_;                    // [k][k]
  double* dinv = Ls + (size_t)kk * kk; // [k]
  double* xw = dinv + kk;              // [warps][k]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j0 = blockIdx.x * kTrinvSmallWarps;
  {   // rows [j0, k) of L_1 in one bulk copy (16-byte aligned: j0 * k * 8 and the size)
    __shared__ __align__(8) uint64_t bar;
    const int64_t first = (int64_t)j0 * kk, cnt = (int64_t)kk * kk - first;
    const bool bulk = ((first * 8) % 16 == 0) && ((cnt * 8) % 16 == 0) && ((uintptr_t)L1 % 16 == 0);
    if (bulk) {
      const uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar);
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb), "r"((uint32_t)(cnt * 8))
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                (uint32_t)__cvta_generic_to_shared(Ls + first)),
            "l"(L1 + first), "r"((uint32_t)(cnt * 8)), "r"(sb)
            : "memory");
      }
      __syncthreads();
      asm volatile(
          "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}\n" ::"r"(sb)
          : "memory");
    } else {
      for (int64_t e = first + threadIdx.x; e < (int64_t)kk * kk; e += blockDim.x) Ls[e] = L1[e];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kk; i += blockDim.x) dinv[i] = 1.0 / Ls[(int64_t)i * kk + i];
  if (blockIdx.x == 0 && w == 0) {   // W_CLIPPED check (Remark 5.2, reading R17)
    double mx = 0.0, mn = DBL_MAX;
    for (int i = lane; i < kk; i += 32) {
      const double a = fabs(L1[(int64_t)i * kk + i]);
      mx = fmax(mx, a);
      mn = fmin(mn, a);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (lane == 0 && mn < 1e-12 * mx) atomicOr(&st->flags, (uint32_t)RBRP_F_W_CLIPPED);
  }
  __syncthreads();
  const int j = j0 + w;
  if (j >= kk) return;
  double* x = xw + (size_t)w * kk;
  if (lane == 0) x[j] = dinv[j];
  __syncwarp();
  for (int i = j + 1; i < kk; ++i) {
    const double* li = Ls + (int64_t)i * kk;
    double s = 0.0;
    for (int m = j + lane; m < i; m += 32) s = fma(li[m], x[m], s);
    s = warp_sum(s);
    if (lane == 0) x[i] = -s * dinv[i];
    __syncwarp();
  }
  for (int64_t m = lane; m < ldo; m += 32) LinvT[(int64_t)j * ldo + m] = (m < j || m >= kk) ? T(0) : (T)x[m];
}

template <typename T>
cudaError_t launch_trinv(const double* L1, int64_t k, T* LinvT, int64_t ldo, DevState* st, cudaStream_t s) {
  if (k <= 0) return cudaSuccess;
  if (k <= kTrinvSmallK) {
    const size_t smem = (size_t)(k * k + k + kTrinvSmallWarps * k) * sizeof(double);
    static bool attr = false;   // once, for the largest k of this path
    if (!attr) {
      const size_t mx = (size_t)(kTrinvSmallK * kTrinvSmallK + kTrinvSmallK + kTrinvSmallWarps * kTrinvSmallK) * 8;
      cudaFuncSetAttribute(k_trinv_small<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
      attr = true;
    }
    k_trinv_small<T><<<ceil_div(k, kTrinvSmallWarps), 32 * kTrinvSmallWarps, smem, s>>>(L1, k, LinvT, ldo, st);
    return cudaGetLastError();
  }
  size_t smem = (size_t)kTrinvWarps * k * sizeof(double);
  cudaFuncSetAttribute(k_trinv<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_trinv<T><<<ceil_div(k, kTrinvWarps), 32 * kTrinvWarps, smem, s>>>(L1, k, LinvT, ldo, st);
  return cudaGetLastError();
}

template <typename T>
__global__ void k_w_identity(T* __restrict__ W, int64_t ldw, const int64_t* __restrict__ S,
                             int64_t k, int64_t n_local, int64_t row_offset) {
  const int64_t i = blockIdx.x;
  const int64_t r = S[i] - row_offset;
  if (r < 0 || r >= n_local) return;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) W[r * ldw + j] = (j == i) ? T(1) : T(0);
}

template <typename T>
cudaError_t launch_w_identity(T* W, int64_t ldw, const int64_t* S, int64_t k, int64_t n_local,
                              int64_t row_offset, cudaStream_t s) {
  if (k <= 0) return cudaSuccess;
  k_w_identity<T><<<(unsigned)k, 256, 0, s>>>(W, ldw, S, k, n_local, row_offset);
  return cudaGetLastError();
}

#define INSTW(T)                                                                                  \
  template cudaError_t launch_gather_L1<T>(const T*, int64_t, const int64_t*, int64_t, int64_t,  \
                                           int64_t, double*, cudaStream_t);                      \
  template cudaError_t launch_trinv<T>(const double*, int64_t, T*, int64_t, DevState*, cudaStream_t); \
  template cudaError_t launch_w_identity<T>(T*, int64_t, const int64_t*, int64_t, int64_t,       \
                                            int64_t, cudaStream_t);
INSTW(double)
INSTW(float)

}  // namespace rbrp
