// k_paper.cu — the paper-literal left-looking form of Alg. 2 (RBRP_FORM_PAPER, SURVEY
// §8(f) NEXT-1): X is never modified, so each block makes one read-only pass over X.
//
//   l.6  V = X(S_t,:)^T - Q Q^T X(S_t,:)^T        k_cgs_dots + k_cgs_update, twice
//                                                          (CGS2, reading R11)
//   l.13  L-hat = X Q_b                            k_lhat_paper (read-only pass) or k_lhat
//   l.16  d <- max(0, d - ||L-hat(i,:)||^2)        fused, or k_downdate (reading R14)
//   l.10  Q <- [Q, Q_b]                            k_append_q
//   reading R13   L-hat(earlier skeletons,:) = 0 exactly   k_zero_prev (X(s,:) Q_b is only
//                                                          zero up to rounding)
#include "launch.cuh"

namespace rbrp {

// l.6 (CGS, one pass): C = V Q^T (b_t x k), then V <- V - C Q.  Two launches per pass
// (the update needs every dot product), two passes (CGS2).  Each Q element read from L2
// serves kRB candidate rows.  Every sum runs in a fixed order: bitwise reproducible and
// identical on every rank.
constexpr int kRB = 8;         // candidate rows per CTA
constexpr int kDotM = 8;       // Q rows per CTA (dots): one per warp
constexpr int kUpdC = 64;      // columns per CTA (update)
constexpr int kUpdG = 4;       // m-groups per column (partial sums combined in fixed order)

// C(i, m) = V(i,:) . Q(m,:): CTA (m-block, row-block); V rows staged in shared memory;
// warp w takes m = m0 + w, lanes stride the columns, one butterfly per (i, m)
template <typename T>
__global__ void __launch_bounds__(256) k_cgs_dots(const double* __restrict__ Vg, int64_t d,
                                                  const T* __restrict__ Qall, double* __restrict__ C,
                                                  int64_t ldc, const DevState* st) {
  if (st->stop) return;
  const int64_t k = st->k;
  const int bt = st->b_t;
  const int64_t m0 = (int64_t)blockIdx.x * kDotM;
  const int i0 = blockIdx.y * kRB;
  if (m0 >= k || i0 >= bt) return;
  const int ni = bt - i0 < kRB ? bt - i0 : kRB;
  extern __shared__ __align__(16) double vs[];   // [kRB][d], then one mbarrier
  __shared__ __align__(8) uint64_t bar;
  const uint32_t bytes = (uint32_t)((int64_t)ni * d * 8);
  if ((d & 1) == 0) {   // one bulk copy of the ni contiguous rows (latency paid once)
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb), "r"(bytes) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              (uint32_t)__cvta_generic_to_shared(vs)),
          "l"(Vg + (int64_t)i0 * d), "r"(bytes), "r"(sb)
          : "memory");
    }
    for (int64_t e = (int64_t)ni * d + threadIdx.x; e < (int64_t)kRB * d; e += blockDim.x) vs[e] = 0.0;
    __syncthreads();
    asm volatile(
        "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}\n" ::"r"(sb)
        : "memory");
  } else {
    for (int64_t e = threadIdx.x; e < (int64_t)kRB * d; e += blockDim.x)
      vs[e] = e < (int64_t)ni * d ? Vg[(int64_t)i0 * d + e] : 0.0;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t m = m0 + w;
  if (m >= k) return;
  const T* q = Qall + m * d;
  double s[kRB];
#pragma unroll
  for (int r = 0; r < kRB; ++r) s[r] = 0.0;
#pragma unroll 8
  for (int64_t j = lane; j < d; j += 32) {
    const double qj = (double)q[j];
#pragma unroll
    for (int r = 0; r < kRB; ++r) s[r] += qj * vs[r * d + j];
  }
#pragma unroll
  for (int r = 0; r < kRB; ++r) {
    const double t = warp_sum(s[r]);
    if (lane == 0 && r < ni) C[(int64_t)(i0 + r) * ldc + m] = t;
  }
}

// V(i, j) -= sum_m C(i, m) Q(m, j): CTA (column block, row block); thread (column, g)
// sums m in the g-th quarter of [0, k) (ascending), quarters combined in order g = 0..3;
// each Q(m, j) load serves kRB rows
template <typename T>
__global__ void __launch_bounds__(kUpdC * kUpdG) k_cgs_update(double* __restrict__ Vg, int64_t d,
                                                              const T* __restrict__ Qall,
                                                              const double* __restrict__ C, int64_t ldc,
                                                              const DevState* st) {
  if (st->stop) return;
  const int64_t k = st->k;
  const int bt = st->b_t;
  const int i0 = blockIdx.y * kRB;
  if (i0 >= bt || k <= 0) return;
  const int ni = bt - i0 < kRB ? bt - i0 : kRB;
  const int cl = threadIdx.x % kUpdC, gq = threadIdx.x / kUpdC;
  const int64_t j = (int64_t)blockIdx.x * kUpdC + cl;
  extern __shared__ double cs[];   // [kRB][k]
  for (int64_t e = threadIdx.x; e < (int64_t)kRB * k; e += blockDim.x) {
    const int64_t r = e / k, m = e % k;
    cs[e] = r < ni ? C[(int64_t)(i0 + r) * ldc + m] : 0.0;
  }
  __syncthreads();
  const int64_t per = (k + kUpdG - 1) / kUpdG;
  const int64_t ma = gq * per, mbnd = ma + per < k ? ma + per : k;
  double acc[kRB];
#pragma unroll
  for (int r = 0; r < kRB; ++r) acc[r] = 0.0;
  if (j < d) {
#pragma unroll 8
    for (int64_t m = ma; m < mbnd; ++m) {
      const double qm = (double)Qall[m * d + j];
#pragma unroll
      for (int r = 0; r < kRB; ++r) acc[r] += cs[r * k + m] * qm;
    }
  }
  __shared__ double part[kUpdG][kRB][kUpdC];
#pragma unroll
  for (int r = 0; r < kRB; ++r) part[gq][r][cl] = acc[r];
  __syncthreads();
  if (gq == 0 && j < d) {
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
      if (r >= ni) break;
      double t = part[0][r][cl];
#pragma unroll
      for (int g2 = 1; g2 < kUpdG; ++g2) t += part[g2][r][cl];
      Vg[(int64_t)(i0 + r) * d + j] -= t;
    }
  }
}

template <typename T>
cudaError_t launch_cgs2_rows(double* Vg, int64_t d, const T* Qall, int64_t k_cap, double* C,
                             const DevState* st, cudaStream_t s) {
  const dim3 gd((unsigned)ceil_div(k_cap, kDotM), kMaxB / kRB), gu((unsigned)ceil_div(d, kUpdC), kMaxB / kRB);
  const size_t smem = (size_t)kRB * d * sizeof(double);
  cudaFuncSetAttribute(k_cgs_dots<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_cgs_update<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kRB * k_cap * 8));
  for (int pass = 0; pass < 2; ++pass) {
    k_cgs_dots<T><<<gd, 256, smem, s>>>(Vg, d, Qall, C, k_cap, st);
    k_cgs_update<T><<<gu, kUpdC * kUpdG, (size_t)kRB * k_cap * 8, s>>>(Vg, d, Qall, C, k_cap, st);
  }
  return cudaGetLastError();
}

// Q <- [Q, Q_b]: rows [k, k + b') of Qall from the block's Q_b rows (l.10)
template <typename T>
__global__ void k_append_q(const T* __restrict__ Qt, int64_t d, T* __restrict__ Qall, const DevState* st) {
  if (st->stop) return;
  const int j = blockIdx.x;
  if (j >= st->b_prime) return;
  const int64_t k0 = st->k;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) Qall[(k0 + j) * d + c] = Qt[(int64_t)j * d + c];
}

template <typename T>
cudaError_t launch_append_q(const T* Qt, int64_t d, T* Qall, const DevState* st, cudaStream_t s) {
  k_append_q<T><<<kMaxB, 256, 0, s>>>(Qt, d, Qall, st);
  return cudaGetLastError();
}

// L-hat(s, k0 : k0+b') = 0 for the earlier skeletons s (their rows of X lie in span(Q),
// which Q_b is orthogonal to; reading R13 makes L_1 exactly lower-triangular)
template <typename T>
__global__ void k_zero_prev(T* __restrict__ L, int64_t ldl, const int64_t* __restrict__ S,
                            int64_t n_local, int64_t row_offset, const DevState* st) {
  if (st->stop) return;
  const int64_t k0 = st->k;
  const int bp = st->b_prime;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; i < k0; i += (int64_t)gridDim.x * blockDim.y) {
    const int64_t r = S[i] - row_offset;
    if (r < 0 || r >= n_local) continue;
    for (int j = threadIdx.x; j < bp; j += blockDim.x) L[r * ldl + k0 + j] = T(0);
  }
}

template <typename T>
cudaError_t launch_zero_prev(T* L, int64_t ldl, const int64_t* S, int64_t n_local, int64_t row_offset,
                             const DevState* st, cudaStream_t s) {
  k_zero_prev<T><<<64, dim3(32, 8), 0, s>>>(L, ldl, S, n_local, row_offset, st);
  return cudaGetLastError();
}

// l.16 downdate for the two-kernel path: d(i) <- max(0, d(i) - ||L-hat(i,:)||^2) (fp64,
// j ascending)
template <typename T>
__global__ void k_downdate(const T* __restrict__ L, int64_t ldl, int64_t n, double* __restrict__ dvec,
                           DevState* st, int fused_max) {
  if (st->stop) return;
  const int bp = st->b_prime;
  if (bp <= 0 || bucket_of(bp) <= fused_max) return;   // the fused kernel downdated already
  const int64_t k0 = st->k;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const T* l = L + i * ldl + k0;
    double s = 0.0;
    for (int j = 0; j < bp; ++j) {
      const double v = (double)l[j];
      s += v * v;
    }
    dvec[i] = fmax(dvec[i] - s, 0.0);
  }
  proj_end_stamp(st);   // end of the projection pass on this path (L-hat + downdate)
}

template <typename T>
cudaError_t launch_downdate(const T* L, int64_t ldl, int64_t n, double* dvec, DevState* st,
                            int fused_max, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_downdate<T><<<ceil_div(n, 256), 256, 0, s>>>(L, ldl, n, dvec, st, fused_max);
  return cudaGetLastError();
}

#define INSTP(T)                                                                                      \
  template cudaError_t launch_cgs2_rows<T>(double*, int64_t, const T*, int64_t, double*,             \
                                           const DevState*, cudaStream_t);                            \
  template cudaError_t launch_append_q<T>(const T*, int64_t, T*, const DevState*, cudaStream_t);      \
  template cudaError_t launch_zero_prev<T>(T*, int64_t, const int64_t*, int64_t, int64_t,             \
                                           const DevState*, cudaStream_t);                            \
  template cudaError_t launch_downdate<T>(const T*, int64_t, int64_t, double*, DevState*, int,        \
                                          cudaStream_t);
INSTP(double)
INSTP(float)

}  // namespace rbrp
