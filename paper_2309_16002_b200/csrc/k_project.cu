// k_project.cu — a4 projection (Alg. 2 l.13 and l.16) in the residual
// form of north_star step (4) / P:523 footnote, plus the C = A B^T tile GEMM reused
// for W (Alg. 3).
//
//   k_lhat    L-hat = X_res Q_b  (n x b'), written into columns [k, k+b') of L.
//   k_update  X_res <- X_res - L-hat Q_b^T and d(i) = ||x_res,i||^2 (fp64), fused:
//             every residual row is read once and written once per block.
//   k_fixup   rows of S'_t: residual and d set to 0, L-hat(S'_t,:) = R_total^T
//             (reading R13), which makes L_1 exactly lower-triangular.
//
// FP64 / FP32 on the CUDA cores (DFMA / FFMA): tcgen05 has no f64 kind (probed), and at
// b' <= 128 the projection is FP64-pipe-bound at fp64 (intensity 2b'/8 flop/B vs a
// ridge of ~5.6).  Register tiles 4 x (BN/8) per thread, operands staged in shared
// memory, global loads for the next K-chunk issued before the FMAs of the current one.
#include "launch.cuh"

namespace rbrp {

constexpr int kGemmThreads = 256;
constexpr int kKC = 16;

template <typename T, int BN>
struct GemmCfg {
  static constexpr int TN = BN / 8;                 // columns per thread
  static constexpr int TM = (BN == 128) ? 2 : 4;    // rows per thread
  static constexpr int BM = 32 * TM;                // rows per CTA
  static constexpr int PAD = 4;
  static constexpr int A_PER = BM * kKC / kGemmThreads;   // A elements per thread per chunk
  static constexpr int B_PER = (BN * kKC + kGemmThreads - 1) / kGemmThreads;
};

// C[m0:m0+BM, n0:n0+BN] = A[m0:, :K] * B[n0:, :K]^T  (row-major A, B; K-contiguous)
template <typename T, int BN>
__device__ __forceinline__ void gemm_nt_tile(const T* __restrict__ A, int64_t lda,
                                             const T* __restrict__ B, int64_t ldb, int64_t M,
                                             int64_t N, int64_t K, int64_t m0, int64_t n0,
                                             T (&acc)[GemmCfg<T, BN>::TM][GemmCfg<T, BN>::TN]) {
  using C = GemmCfg<T, BN>;
  __shared__ __align__(16) T As[kKC][C::BM + C::PAD];
  __shared__ __align__(16) T Bs[kKC][BN + C::PAD];
  const int tid = threadIdx.x;
  const int ty = tid / 8, tx = tid % 8;
#pragma unroll
  for (int r = 0; r < C::TM; ++r)
#pragma unroll
    for (int c = 0; c < C::TN; ++c) acc[r][c] = T(0);

  // A-load mapping: thread -> row ar, columns [ac0, ac0 + A_PER)
  constexpr int TPR = kKC / C::A_PER;   // threads per row
  const int ar = tid / TPR, ac0 = (tid % TPR) * C::A_PER;
  T ra[C::A_PER], rb[C::B_PER];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int e = 0; e < C::A_PER; ++e) {
      const int64_t gr = m0 + ar, gc = k0 + ac0 + e;
      ra[e] = (gr < M && gc < K) ? A[gr * lda + gc] : T(0);
    }
#pragma unroll
    for (int e = 0; e < C::B_PER; ++e) {
      const int idx = tid + e * kGemmThreads;
      const int j = idx / kKC, c = idx % kKC;
      const int64_t gj = n0 + j, gc = k0 + c;
      rb[e] = (idx < BN * kKC && gj < N && gc < K) ? B[gj * ldb + gc] : T(0);
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int e = 0; e < C::A_PER; ++e) As[ac0 + e][ar] = ra[e];
#pragma unroll
    for (int e = 0; e < C::B_PER; ++e) {
      const int idx = tid + e * kGemmThreads;
      if (idx < BN * kKC) Bs[idx % kKC][idx / kKC] = rb[e];
    }
  };
  load(0);
  for (int64_t k0 = 0; k0 < K; k0 += kKC) {
    __syncthreads();
    store();
    __syncthreads();
    if (k0 + kKC < K) load(k0 + kKC);
#pragma unroll
    for (int kk = 0; kk < kKC; ++kk) {
      T a[C::TM], b[C::TN];
#pragma unroll
      for (int r = 0; r < C::TM; ++r) a[r] = As[kk][ty * C::TM + r];
#pragma unroll
      for (int c = 0; c < C::TN; ++c) b[c] = Bs[kk][tx * C::TN + c];
#pragma unroll
      for (int r = 0; r < C::TM; ++r)
#pragma unroll
        for (int c = 0; c < C::TN; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
    }
  }
}

template <typename T, int BN>
__global__ void __launch_bounds__(kGemmThreads) k_lhat(const T* __restrict__ Xres, int64_t ldx,
                                                       const T* __restrict__ Qt, int64_t n,
                                                       int64_t d, T* __restrict__ L, int64_t ldl,
                                                       DevState* st) {
  using C = GemmCfg<T, BN>;
  if (st->stop) return;
  const int bp = st->b_prime;
  if (bp <= 0 || bucket_of(bp) != BN) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->ts0 = gtimer();
  const int64_t k0 = st->k;
  const int64_t m0 = (int64_t)blockIdx.x * C::BM;
  T acc[C::TM][C::TN];
  gemm_nt_tile<T, BN>(Xres, ldx, Qt, d, n, bp, d, m0, 0, acc);
  const int ty = threadIdx.x / 8, tx = threadIdx.x % 8;
#pragma unroll
  for (int r = 0; r < C::TM; ++r) {
    const int64_t row = m0 + ty * C::TM + r;
    if (row >= n) continue;
#pragma unroll
    for (int c = 0; c < C::TN; ++c) {
      const int col = tx * C::TN + c;
      if (col < bp) L[row * ldl + k0 + col] = acc[r][c];
    }
  }
}

template <typename T>
cudaError_t launch_lhat(const T* Xres, int64_t ldx, const T* Qt, int64_t n, int64_t d, T* L,
                        int64_t ldl, DevState* st, int bucket, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  switch (bucket) {
    case 16: k_lhat<T, 16><<<ceil_div(n, GemmCfg<T, 16>::BM), kGemmThreads, 0, s>>>(Xres, ldx, Qt, n, d, L, ldl, st); break;
    case 32: k_lhat<T, 32><<<ceil_div(n, GemmCfg<T, 32>::BM), kGemmThreads, 0, s>>>(Xres, ldx, Qt, n, d, L, ldl, st); break;
    case 64: k_lhat<T, 64><<<ceil_div(n, GemmCfg<T, 64>::BM), kGemmThreads, 0, s>>>(Xres, ldx, Qt, n, d, L, ldl, st); break;
    default: k_lhat<T, 128><<<ceil_div(n, GemmCfg<T, 128>::BM), kGemmThreads, 0, s>>>(Xres, ldx, Qt, n, d, L, ldl, st); break;
  }
  return cudaGetLastError();
}

// generic C = A B^T (used for W = L L_1^{-1} with B = L_1^{-T})
template <typename T, int BN>
__global__ void __launch_bounds__(kGemmThreads) k_gemm_nt(const T* __restrict__ A, int64_t lda,
                                                          const T* __restrict__ B, int64_t ldb,
                                                          T* __restrict__ Cm, int64_t ldc, int64_t M,
                                                          int64_t N, int64_t K) {
  using C = GemmCfg<T, BN>;
  const int64_t m0 = (int64_t)blockIdx.x * C::BM, n0 = (int64_t)blockIdx.y * BN;
  T acc[C::TM][C::TN];
  gemm_nt_tile<T, BN>(A, lda, B, ldb, M, N, K, m0, n0, acc);
  const int ty = threadIdx.x / 8, tx = threadIdx.x % 8;
#pragma unroll
  for (int r = 0; r < C::TM; ++r) {
    const int64_t row = m0 + ty * C::TM + r;
    if (row >= M) continue;
#pragma unroll
    for (int c = 0; c < C::TN; ++c) {
      const int64_t col = n0 + tx * C::TN + c;
      if (col < N) Cm[row * ldc + col] = acc[r][c];
    }
  }
}

template <typename T>
cudaError_t launch_gemm_nt(const T* A, int64_t lda, const T* B, int64_t ldb, T* Cm, int64_t ldc,
                           int64_t M, int64_t N, int64_t K, cudaStream_t s) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  dim3 grid(ceil_div(M, GemmCfg<T, 64>::BM), ceil_div(N, 64));
  k_gemm_nt<T, 64><<<grid, kGemmThreads, 0, s>>>(A, lda, B, ldb, Cm, ldc, M, N, K);
  return cudaGetLastError();
}

// X_res(rows, :) -= P(rows, :b') Q_b^T ; d(rows) = ||x_res||^2
constexpr int kUpdRows = 64, kUpdCols = 64;

template <typename T, int BP>
__global__ void __launch_bounds__(256) k_update(T* __restrict__ X, int64_t ldx,
                                                const T* __restrict__ Qt, const T* __restrict__ L,
                                                int64_t ldl, int64_t n, int64_t d,
                                                double* __restrict__ dvec, DevState* st) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T (*Ps)[kUpdRows + 4] = reinterpret_cast<T (*)[kUpdRows + 4]>(smem_raw);
  T (*Qs)[kUpdCols + 4] = reinterpret_cast<T (*)[kUpdCols + 4]>(smem_raw + sizeof(T) * BP * (kUpdRows + 4));
  if (st->stop) return;
  const int bp = st->b_prime;
  if (bp <= 0 || bucket_of(bp) != BP) return;
  const int64_t k0 = st->k;
  const int tid = threadIdx.x, tr = tid / 16, tc = tid % 16;
  const int64_t r0 = (int64_t)blockIdx.x * kUpdRows;
  for (int e = tid; e < kUpdRows * BP; e += 256) {
    const int r = e / BP, j = e % BP;
    Ps[j][r] = (j < bp && r0 + r < n) ? L[(r0 + r) * ldl + k0 + j] : T(0);
  }
  double nrm[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t c0 = 0; c0 < d; c0 += kUpdCols) {
    __syncthreads();
    for (int e = tid; e < BP * kUpdCols; e += 256) {
      const int j = e / kUpdCols, c = e % kUpdCols;
      Qs[j][c] = (c0 + c < d) ? Qt[(int64_t)j * d + c0 + c] : T(0);
    }
    T acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int64_t gr = r0 + tr * 4 + r, gc = c0 + tc * 4 + c;
        acc[r][c] = (gr < n && gc < d) ? X[gr * ldx + gc] : T(0);
      }
    __syncthreads();
#pragma unroll 8
    for (int j = 0; j < BP; ++j) {
      T a[4], q[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = Ps[j][tr * 4 + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) q[c] = Qs[j][tc * 4 + c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fma(-a[r], q[c], acc[r][c]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int64_t gr = r0 + tr * 4 + r, gc = c0 + tc * 4 + c;
        if (gr < n && gc < d) {
          X[gr * ldx + gc] = acc[r][c];
          const double v = (double)acc[r][c];
          nrm[r] += v * v;
        }
      }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    double v = nrm[r];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t gr = r0 + tr * 4 + r;
    if (tc == 0 && gr < n) dvec[gr] = v;
  }
  proj_end_stamp(st);
}

template <typename T>
cudaError_t launch_update(T* Xres, int64_t ldx, const T* Qt, const T* L, int64_t ldl, int64_t n,
                          int64_t d, double* dvec, DevState* st, int bucket, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int g = ceil_div(n, kUpdRows);
  auto go = [&](auto kern, int BP) {
    const size_t smem = sizeof(T) * BP * ((kUpdRows + 4) + (kUpdCols + 4));
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<g, 256, smem, s>>>(Xres, ldx, Qt, L, ldl, n, d, dvec, st);
  };
  switch (bucket) {
    case 16: go(k_update<T, 16>, 16); break;
    case 32: go(k_update<T, 32>, 32); break;
    case 64: go(k_update<T, 64>, 64); break;
    default: go(k_update<T, 128>, 128); break;
  }
  return cudaGetLastError();
}

// rows of S'_t: residual 0, d 0, L-hat(S'_t,:) = R_total^T
template <typename T>
__global__ void __launch_bounds__(256) k_fixup(T* __restrict__ X, int64_t ldx,
                                               double* __restrict__ dvec, T* __restrict__ L,
                                               int64_t ldl, const double* __restrict__ Rtot,
                                               const int64_t* __restrict__ S, int64_t n_local,
                                               int64_t row_offset, int64_t d, DevState* st) {
  if (st->stop) return;
  const int bp = st->b_prime;
  const int i = blockIdx.x;
  if (i >= bp) return;
  const int64_t k0 = st->k;
  if (i == 0 && threadIdx.x < 32) {
    // diag(L_1) of this block = diag(R_V(1:b',1:b')) as stored in L (Remark 5.2 trigger):
    // min / max over the warp (lanes j, j + 32, ...), all loads in flight together
    const int lane = threadIdx.x;
    double mn = INFINITY, mx = 0.0;
#pragma unroll
    for (int u = 0; u < kMaxB / 32; ++u) {
      const int j = lane + 32 * u;
      if (j < bp) {
        const double a = fabs((double)(T)Rtot[j * kMaxB + j]);
        mn = fmin(mn, a);
        mx = fmax(mx, a);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
      st->ldiag_min = fmin(st->ldiag_min, mn);
      st->ldiag_max = fmax(st->ldiag_max, mx);
    }
  }
  const int64_t r = S[k0 + i] - row_offset;
  if (r < 0 || r >= n_local) return;
  if (X)   // residual form: the skeleton's residual row is 0 (paper form: X is read only)
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) X[r * ldx + c] = T(0);
  for (int j = threadIdx.x; j < bp; j += blockDim.x)
    L[r * ldl + k0 + j] = (j <= i) ? (T)Rtot[j * kMaxB + i] : T(0);
  if (threadIdx.x == 0) dvec[r] = 0.0;
}

template <typename T>
cudaError_t launch_fixup(T* Xres, int64_t ldx, double* dvec, T* L, int64_t ldl, const double* Rtot,
                         const int64_t* S, int64_t n_local, int64_t row_offset, int64_t d,
                         DevState* st, cudaStream_t s) {
  k_fixup<T><<<kMaxB, 256, 0, s>>>(Xres, ldx, dvec, L, ldl, Rtot, S, n_local, row_offset, d, st);
  return cudaGetLastError();
}

#define INST(T)                                                                                  \
  template cudaError_t launch_lhat<T>(const T*, int64_t, const T*, int64_t, int64_t, T*, int64_t, \
                                      DevState*, int, cudaStream_t);                              \
  template cudaError_t launch_update<T>(T*, int64_t, const T*, const T*, int64_t, int64_t,        \
                                        int64_t, double*, DevState*, int, cudaStream_t);          \
  template cudaError_t launch_fixup<T>(T*, int64_t, double*, T*, int64_t, const double*,          \
                                       const int64_t*, int64_t, int64_t, int64_t, DevState*,      \
                                       cudaStream_t);                                             \
  template cudaError_t launch_gemm_nt<T>(const T*, int64_t, const T*, int64_t, T*, int64_t,       \
                                         int64_t, int64_t, int64_t, cudaStream_t);
INST(double)
INST(float)

}  // namespace rbrp
