// k_project_mma.cu — a4 projection on the FP64 tensor path (DMMA, mma.sync.m8n8k4.f64).
//
// B200 has no FP64 kind for tcgen05 (ptxas rejects kind::f64); the legacy DMMA path
// reaches the full FP64 rate (measured 37.2 TFLOP/s vs 33.8 for DFMA, profiles/).
//
//   k_nt_mma<BN>     C[m, n0+j] = sum_k A[m,k] B[n0+j,k]   (row-major A, B; K contiguous)
//                    = L-hat = X_res Q_b^T (Alg. 2 l.13) and W = L L_1^{-1} (Alg. 3).
//   k_update_mma<BP> X_res -= L-hat Q_b and d(i) = ||x_res,i||^2 (l.16), fused:
//                    each residual row is read once and written once per block.
//
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64): lane = 4 g + q;  A(8x4): A[g][q];
// B(4x8): B[q][g];  C/D(8x8): C[g][2q + i], i = 0, 1.
// In k_nt_mma an A-row segment x[2q, 2q+1] (one 16-byte load) feeds two MMAs whose K
// index is permuted as k = 2q + h; the B fragments are read with the same permutation
// (one 16-byte shared load gives both), so no shuffles are needed.
#include <stdlib.h>

#include <algorithm>

#include "launch.cuh"

namespace rbrp {

__device__ __forceinline__ void dmma(double2& d, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d.x), "+d"(d.y)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

constexpr int kMmaWarps = 8;

// Tile configuration: RG row groups of 8 rows per warp (each B fragment read from shared
// memory feeds RG MMAs), KC-column K chunks through an NS-stage cp.async pipeline
// (NS = as many stages as fit in ~200 KB, at most 4).  Strides: X / B tiles = KC + 8
// doubles (= 8 mod 16: conflict-free 16-byte fragment loads), Q tiles for 8-byte loads =
// KC + 4 (= 4 mod 16: conflict-free per half-warp).
template <int BN, int RG_, int KC_, bool UPD>
struct PCfg {
  static constexpr int RG = RG_;
  // fall back to 32-column chunks when two stages of the requested tile do not fit
  static constexpr int KC = (8 * RG_ * kMmaWarps * (KC_ + 8) + BN * (KC_ + 8)) * 8 * 2 > 200 * 1024 ? 32 : KC_;
  static constexpr int XLD = KC + 8;
  static constexpr int BLD = UPD ? KC + 4 : KC + 8;
  static constexpr int ROWS = 8 * RG * kMmaWarps;
  static constexpr int STAGE = ROWS * XLD + BN * BLD;
  static constexpr int NSF = (200 * 1024) / (STAGE * 8);
  static constexpr int NS = NSF < 4 ? NSF : 4;
  static constexpr size_t SMEM = sizeof(double) * NS * STAGE;
  static_assert(NS >= 2, "tile too large");
};

template <int ROWS, int KC, int XLD>
__device__ __forceinline__ void stage_x(double* xs, const double* __restrict__ A, int64_t lda,
                                        int64_t r0, int64_t M, int64_t c0, int64_t K, int tid) {
#pragma unroll
  for (int i = 0; i < (ROWS * KC / 2) / (32 * kMmaWarps); ++i) {
    const int e = tid + i * 32 * kMmaWarps;
    const int r = e / (KC / 2), c = (e % (KC / 2)) * 2;
    const bool ok = (r0 + r < M) && (c0 + c < K);
    cp_async16(xs + r * XLD + c, ok ? A + (r0 + r) * lda + c0 + c : A, ok);
  }
}
template <int BN, int KC, int LD>
__device__ __forceinline__ void stage_b(double* bs, const double* __restrict__ B, int64_t ldb,
                                        int64_t n0, int64_t nrows, int64_t c0, int64_t K, int tid) {
  for (int e = tid; e < BN * (KC / 2); e += 32 * kMmaWarps) {
    const int j = e / (KC / 2), c = (e % (KC / 2)) * 2;
    const bool ok = (n0 + j < nrows) && (c0 + c < K);
    cp_async16(bs + j * LD + c, ok ? B + (n0 + j) * ldb + c0 + c : B, ok);
  }
}

// ---------------------------------------------------------------------------------
// C = A B^T: ROWS-row tiles x BN columns; persistent CTAs (one per SM) walk their tiles
// and the 32-column K chunks of each tile as ONE flattened sequence, so the cp.async
// pipeline never drains between tiles.  Warp w owns rows [w*8*RG, (w+1)*8*RG) of a tile.
// Requirements (checked by the launcher): K % 8 == 0, lda % 2 == 0, ldb % 2 == 0,
// 16-byte aligned A and B.
// ---------------------------------------------------------------------------------
template <int BN, int RG_, int KC_>
__global__ void __launch_bounds__(32 * kMmaWarps, 1) k_nt_mma(const double* __restrict__ A, int64_t lda,
                                                              const double* __restrict__ B, int64_t ldb,
                                                              double* __restrict__ C, int64_t ldc,
                                                              int64_t M, int64_t N, int64_t K,
                                                              DevState* st, int mode) {
  using Cf = PCfg<BN, RG_, KC_, false>;
  constexpr int RG = Cf::RG, kKC = Cf::KC, kXld = Cf::XLD, kBld = Cf::BLD;
  extern __shared__ __align__(16) double sm[];
  int64_t col0 = 0, Nn = N;
  if (mode == 1) {   // L-hat: N = b', columns written at L[:, k + j]
    if (st->stop) return;
    const int bp = st->b_prime;
    if (bp <= 0 || bucket_of(bp) != BN) return;
    Nn = bp;
    col0 = st->k;
    if (blockIdx.x == 0 && threadIdx.x == 0) st->ts0 = gtimer();
  }
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int64_t ntm = (M + Cf::ROWS - 1) / Cf::ROWS;
  const int64_t ntn = (Nn + BN - 1) / BN;
  const int64_t ntiles = ntm * ntn;
  const int nchunk = (int)((K + kKC - 1) / kKC);
  const int64_t nmine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = nmine * nchunk;
  auto tile_of = [&](int64_t j, int64_t& r0, int64_t& n0) {
    const int64_t t = blockIdx.x + j * gridDim.x;
    r0 = (t % ntm) * Cf::ROWS;
    n0 = (t / ntm) * BN;
  };
  auto issue = [&](int64_t it) {
    if (it < total) {
      int64_t r0, n0;
      tile_of(it / nchunk, r0, n0);
      const int64_t k0 = (it % nchunk) * kKC;
      double* base = sm + (size_t)(it % Cf::NS) * Cf::STAGE;
      stage_x<Cf::ROWS, kKC, kXld>(base, A, lda, r0, M, k0, K, tid);
      stage_b<BN, kKC, kBld>(base + Cf::ROWS * kXld, B, ldb, n0, Nn, k0, K, tid);
    }
    cp_async_commit();
  };
  double2 acc[RG][BN / 8];
#pragma unroll
  for (int r = 0; r < RG; ++r)
#pragma unroll
    for (int t = 0; t < BN / 8; ++t) acc[r][t] = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < Cf::NS - 1; ++i) issue(i);
  for (int64_t it = 0; it < total; ++it) {
    issue(it + Cf::NS - 1);
    cp_async_wait<Cf::NS - 1>();
    __syncthreads();
    const double* xs = sm + (size_t)(it % Cf::NS) * Cf::STAGE;
    const double* bs = xs + Cf::ROWS * kXld;
#pragma unroll
    for (int s = 0; s < kKC / 8; ++s) {
      double2 xa[RG], b[BN / 8];
#pragma unroll
      for (int r = 0; r < RG; ++r)
        xa[r] = *reinterpret_cast<const double2*>(xs + ((w * RG + r) * 8 + g) * kXld + 8 * s + 2 * q);
#pragma unroll
      for (int t = 0; t < BN / 8; ++t)
        b[t] = *reinterpret_cast<const double2*>(bs + (t * 8 + g) * kBld + 8 * s + 2 * q);
      // the two K halves of an accumulator are separated by all other accumulators' MMAs
#pragma unroll
      for (int t = 0; t < BN / 8; ++t)
#pragma unroll
        for (int r = 0; r < RG; ++r) dmma(acc[r][t], xa[r].x, b[t].x);
#pragma unroll
      for (int t = 0; t < BN / 8; ++t)
#pragma unroll
        for (int r = 0; r < RG; ++r) dmma(acc[r][t], xa[r].y, b[t].y);
    }
    if (it % nchunk == nchunk - 1) {   // tile done: write, reset
      int64_t r0, n0;
      tile_of(it / nchunk, r0, n0);
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        const int64_t row = r0 + (w * RG + r) * 8 + g;
        if (row < M) {
          double* crow = C + row * ldc + col0;
#pragma unroll
          for (int t = 0; t < BN / 8; ++t) {
            const int64_t j = n0 + t * 8 + 2 * q;
            if (j < Nn) crow[j] = acc[r][t].x;
            if (j + 1 < Nn) crow[j + 1] = acc[r][t].y;
          }
        }
#pragma unroll
        for (int t = 0; t < BN / 8; ++t) acc[r][t] = make_double2(0.0, 0.0);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------
// X(rows, :) -= P(rows, :b') Q_b ; d(rows) = ||x||^2.  P = L[:, k : k+b'].
// Persistent CTAs, flattened (tile, chunk) cp.async pipeline; the next tile's P rows
// (the A fragments) are fetched into registers one chunk before the tile switch.
// Requirements: d % 8 == 0, ldx % 2 == 0, 16-byte aligned X and Qt.
// ---------------------------------------------------------------------------------
template <int BP, int RG_, int KC_>
__global__ void __launch_bounds__(32 * kMmaWarps, 1) k_update_mma(double* __restrict__ X, int64_t ldx,
                                                                  const double* __restrict__ Qt,
                                                                  const double* __restrict__ L,
                                                                  int64_t ldl, int64_t n, int64_t d,
                                                                  double* __restrict__ dvec,
                                                                  DevState* st) {
  using Cf = PCfg<BP, RG_, KC_, true>;
  constexpr int RG = Cf::RG, kKC = Cf::KC, kXld = Cf::XLD, kQld = Cf::BLD;
  extern __shared__ __align__(16) double sm[];
  if (st->stop) return;
  const int bp = st->b_prime;
  if (bp <= 0 || bucket_of(bp) != BP) return;
  const int64_t k0 = st->k;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int64_t ntiles = (n + Cf::ROWS - 1) / Cf::ROWS;
  const int nchunk = (int)((d + kKC - 1) / kKC);
  const int64_t nmine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = nmine * nchunk;
  auto r0_of = [&](int64_t j) { return (blockIdx.x + j * gridDim.x) * (int64_t)Cf::ROWS; };
  auto issue = [&](int64_t it) {
    if (it < total) {
      double* base = sm + (size_t)(it % Cf::NS) * Cf::STAGE;
      const int64_t c0 = (it % nchunk) * kKC;
      stage_x<Cf::ROWS, kKC, kXld>(base, X, ldx, r0_of(it / nchunk), n, c0, d, tid);
      stage_b<BP, kKC, kQld>(base + Cf::ROWS * kXld, Qt, d, 0, bp, c0, d, tid);
    }
    cp_async_commit();
  };
  // A fragments: -P[row][4 jc + q] for the warp's RG row groups
  double a[RG][BP / 4], an[RG][BP / 4];
  auto load_a = [&](double (&dst)[RG][BP / 4], int64_t j) {
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      const int64_t row = r0_of(j) + (w * RG + r) * 8 + g;
      const bool rok = row < n;
      const double* lrow = L + (rok ? row : 0) * ldl + k0;
#pragma unroll
      for (int jc = 0; jc < BP / 4; ++jc) {
        const int jj = jc * 4 + q;
        dst[r][jc] = (rok && jj < bp) ? -lrow[jj] : 0.0;
      }
    }
  };
#pragma unroll
  for (int i = 0; i < Cf::NS - 1; ++i) issue(i);
  if (total > 0) load_a(a, 0);
  double nrm[RG];
#pragma unroll
  for (int r = 0; r < RG; ++r) nrm[r] = 0.0;
  for (int64_t it = 0; it < total; ++it) {
    const int64_t j = it / nchunk;
    const int ch = (int)(it % nchunk);
    issue(it + Cf::NS - 1);
    if (ch == nchunk - 1 && j + 1 < nmine) load_a(an, j + 1);
    cp_async_wait<Cf::NS - 1>();
    __syncthreads();
    const double* xs = sm + (size_t)(it % Cf::NS) * Cf::STAGE;
    const double* qb = xs + Cf::ROWS * kXld;
    const int64_t c0 = (int64_t)ch * kKC;
    double2 xd[RG][kKC / 8];
#pragma unroll
    for (int r = 0; r < RG; ++r)
#pragma unroll
      for (int s = 0; s < kKC / 8; ++s)
        xd[r][s] = *reinterpret_cast<const double2*>(xs + ((w * RG + r) * 8 + g) * kXld + 8 * s + 2 * q);
#pragma unroll
    for (int jc = 0; jc < BP / 4; ++jc) {
#pragma unroll
      for (int s = 0; s < kKC / 8; ++s) {
        const double bq = qb[(jc * 4 + q) * kQld + 8 * s + g];
#pragma unroll
        for (int r = 0; r < RG; ++r) dmma(xd[r][s], a[r][jc], bq);
      }
    }
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      const int64_t row = r0_of(j) + (w * RG + r) * 8 + g;
      const bool rok = row < n;
      double* xrow = X + (rok ? row : 0) * ldx;
#pragma unroll
      for (int s = 0; s < kKC / 8; ++s) {
        const int64_t c = c0 + 8 * s + 2 * q;
        if (rok && c < d) {
          __stcs(reinterpret_cast<double2*>(xrow + c), xd[r][s]);
          nrm[r] += xd[r][s].x * xd[r][s].x + xd[r][s].y * xd[r][s].y;
        }
      }
      if (ch == nchunk - 1) {
        double v = nrm[r];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (rok && q == 0) dvec[row] = v;
        nrm[r] = 0.0;
      }
    }
    if (ch == nchunk - 1) {
#pragma unroll
      for (int r = 0; r < RG; ++r)
#pragma unroll
        for (int jc = 0; jc < BP / 4; ++jc) a[r][jc] = an[r][jc];
    }
    __syncthreads();
  }
  proj_end_stamp(st);
}

static int num_sms() { return device_sms(); }

static bool mma_ok(const void* p, int64_t ld, int64_t K) {
  return (K % 8 == 0) && (ld % 2 == 0) && ((uintptr_t)p % 16 == 0);
}

bool projection_mma_supported(const void* X, int64_t ldx, const void* Qt, int64_t d) {
  return mma_ok(X, ldx, d) && ((uintptr_t)Qt % 16 == 0);
}

// projection tile variant: RBRP_PROJ_VARIANT = 0: (RG 1, KC 64)  1: (RG 2, KC 32)
// 2: (RG 2, KC 64)  3: (RG 1, KC 32); default 0.  (RG 1 for b' > 64 in every variant.)
static int proj_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RBRP_PROJ_VARIANT");
    v = e ? atoi(e) : 0;
    if (v < 0 || v > 3) v = 0;
  }
  return v;
}

template <int BN, int RG, int KC>
static void go_lhat(const double* Xres, int64_t ldx, const double* Qt, int64_t n, int64_t d, double* L,
                    int64_t ldl, DevState* st, cudaStream_t s) {
  using Cf = PCfg<BN, RG, KC, false>;
  auto kern = k_nt_mma<BN, RG, KC>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
  kern<<<num_sms(), 32 * kMmaWarps, Cf::SMEM, s>>>(Xres, ldx, Qt, d, L, ldl, n, 0, d, st, 1);
}
template <int BP, int RG, int KC>
static void go_upd(double* Xres, int64_t ldx, const double* Qt, const double* L, int64_t ldl, int64_t n,
                   int64_t d, double* dvec, DevState* st, cudaStream_t s) {
  using Cf = PCfg<BP, RG, KC, true>;
  auto kern = k_update_mma<BP, RG, KC>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
  kern<<<num_sms(), 32 * kMmaWarps, Cf::SMEM, s>>>(Xres, ldx, Qt, L, ldl, n, d, dvec, st);
}

#define RBRP_VARIANTS(GO, B, ...)                         \
  switch (proj_variant()) {                              \
    case 1: GO<B, 2, 32>(__VA_ARGS__); break;            \
    case 2: GO<B, 2, 64>(__VA_ARGS__); break;            \
    case 3: GO<B, 1, 32>(__VA_ARGS__); break;            \
    default: GO<B, 1, 64>(__VA_ARGS__); break;           \
  }

cudaError_t launch_lhat_mma(const double* Xres, int64_t ldx, const double* Qt, int64_t n, int64_t d,
                            double* L, int64_t ldl, DevState* st, int bucket, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  switch (bucket) {
    case 16: RBRP_VARIANTS(go_lhat, 16, Xres, ldx, Qt, n, d, L, ldl, st, s); break;
    case 32: RBRP_VARIANTS(go_lhat, 32, Xres, ldx, Qt, n, d, L, ldl, st, s); break;
    case 64: RBRP_VARIANTS(go_lhat, 64, Xres, ldx, Qt, n, d, L, ldl, st, s); break;
    default: go_lhat<128, 1, 32>(Xres, ldx, Qt, n, d, L, ldl, st, s); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_update_mma(double* Xres, int64_t ldx, const double* Qt, const double* L,
                              int64_t ldl, int64_t n, int64_t d, double* dvec, DevState* st,
                              int bucket, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  switch (bucket) {
    case 16: RBRP_VARIANTS(go_upd, 16, Xres, ldx, Qt, L, ldl, n, d, dvec, st, s); break;
    case 32: RBRP_VARIANTS(go_upd, 32, Xres, ldx, Qt, L, ldl, n, d, dvec, st, s); break;
    case 64: RBRP_VARIANTS(go_upd, 64, Xres, ldx, Qt, L, ldl, n, d, dvec, st, s); break;
    default: go_upd<128, 1, 32>(Xres, ldx, Qt, L, ldl, n, d, dvec, st, s); break;
  }
  return cudaGetLastError();
}

// W = A B^T with N = k columns (B = L_1^{-T}), DMMA path when shapes allow
bool gemm_nt_mma(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                 int64_t M, int64_t N, int64_t K, cudaStream_t s, cudaError_t* err) {
  if (!mma_ok(A, lda, K) || !mma_ok(B, ldb, K)) return false;
  dim3 grid((unsigned)num_sms(), 1);
  using Cf = PCfg<128, 1, 32, false>;
  static PerDevice attr;
  const cudaError_t ae = attr.once(
      [] { return cudaFuncSetAttribute(k_nt_mma<128, 1, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM); });
  if (ae != cudaSuccess) {
    *err = ae;
    return true;
  }
  k_nt_mma<128, 1, 32><<<grid, 32 * kMmaWarps, Cf::SMEM, s>>>(A, lda, B, ldb, C, ldc, M, N, K, nullptr, 0);
  *err = cudaGetLastError();
  return true;
}

}  // namespace rbrp
