// k_sketch.cu — sketchy pivoting with LUPP and the oversampled sketchy interpolation
// matrix, SkLUPP-OSID (section 3.2; Alg. 4, P:611-622;
// Eq. 5.3).  fp64.
//
//   k_embedding  Omega^T (l x d), iid N(0, 1/l) by Philox4x32-10 + Box-Muller
//                (reading R25).
//   Y = X Omega  the FP64 tensor-path GEMM of k_project_mma.cu (gemm_nt_mma).
//   k_lupp       partial-pivoting LU on Y, first k pivots (reading R26): one
//                cooperative kernel, rows split over the CTAs (one per SM), columns in
//                panels of PW held in shared memory.  Per step: every CTA proposes its
//                best active row (|A(i, c)|, ties to the lower row) with its panel values,
//                one grid barrier, every CTA picks the same winner and updates its rows.
//                At a panel start the earlier pivots' U rows for the panel columns are
//                rebuilt by forward substitution from Y and the stored multipliers, and
//                each active row applies them in pivot order -- every entry sees exactly
//                the updates a - l*u (product rounded, then the difference, as the
//                unblocked loop) in the same order, so pivots and multipliers equal the
//                textbook loop's bit for bit.
//   OSID         Z = Y(S,:) (k x l); CholQR2 of Z^T: G1 = Z Z^T = C1 C1^T, P1 = C1^{-1} Z,
//                G2 = P1 P1^T = C2 C2^T, Q^T = C2^{-1} P1; M^T = (R2 R1)^{-1} Q^T with
//                R = C2^T C1^T, so W = Y M = (Y Q) R^{-T} (Alg. 4 l.4) = Y Y_S^+; then
//                W(S,:) = I_k (l.3).  The k x k / k x l steps (Gram, blocked Cholesky,
//                triangular products) are CUDA-core kernels;
//                W = Y M is the FP64 tensor-path GEMM again.
#include <cooperative_groups.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "../../include/rbrp_sketch.h"
#include "launch.cuh"
#include "philox.cuh"

namespace cg = cooperative_groups;

namespace rbrp {
namespace sk {
constexpr int kThreads = 512;   // >= RBRP_SK_MAX_K: one U row per thread in (1)
constexpr int kCandPerLane = 5;   // winner search: 160 candidates per pass of warp 0
constexpr int kSmemMax = 227 * 1024;
constexpr uint32_t kOmegaTag = 0x4F4D4547u;   // reading R25
static_assert(kThreads >= RBRP_SK_MAX_K, "k_lupp step (1) holds one U row per thread");
}  // namespace sk

// ------------------------------------------------------------------------------------
// Gaussian embedding (reading R25)
// ------------------------------------------------------------------------------------
__global__ void k_embedding(int64_t d, int64_t l, uint2 key, double* __restrict__ OmT, int64_t ldo) {
  const int64_t total = d * l, nq = (total + 1) / 2;
  const double sl = sqrt((double)l);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)q, (uint32_t)(q >> 32), 0u, sk::kOmegaTag), key);
    const double u1 = u53(w);
    const double u2 = u53(make_uint4(w.z, w.w, 0u, 0u));
    const double r = sqrt(-2.0 * log(1.0 - u1));
    const double a = (2.0 * M_PI) * u2;
    const double z0 = r * cos(a), z1 = r * sin(a);
    const int64_t e0 = 2 * q;
    {
      const int64_t j = e0 / d, i = e0 - j * d;
      OmT[j * ldo + i] = z0 / sl;
    }
    if (e0 + 1 < total) {
      const int64_t j = (e0 + 1) / d, i = (e0 + 1) - j * d;
      OmT[j * ldo + i] = z1 / sl;
    }
  }
}

// ------------------------------------------------------------------------------------
// LUPP (reading R26)
// ------------------------------------------------------------------------------------
struct LuArgs {
  const double* Y;
  int64_t n, l, ldy;
  int k, R;
  double* Lm;       // k x n multipliers, column-major: L(i, m) at Lm[m * n + i]
  double* Lp;       // k x k row-major: the pivot rows' multipliers, Lp[m * k + mm] = L(p_m, mm)
  double* cand;     // [2][G][PW + 2]: |v|, row (bits), panel values of each CTA's candidate
  int64_t* piv;     // k
  int64_t* pcol;    // k
  int* out;         // [0] pivots found
};

__device__ __forceinline__ bool lu_better(double v, long long r, double bv, long long br) {
  return v > bv || (v == bv && r < br);
}

// warp argmax of (v, r) with owner tag `who` (< 0: no candidate); result in every lane
__device__ __forceinline__ void lu_warp_best(double& v, long long& r, int& who) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const long long orr = __shfl_xor_sync(0xffffffffu, r, o);
    const int og = __shfl_xor_sync(0xffffffffu, who, o);
    if (og >= 0 && (who < 0 || lu_better(ov, orr, v, r))) {
      v = ov;
      r = orr;
      who = og;
    }
  }
}

#ifdef LU_TRACE   // phase cycle counts of CTA 0 (debug builds: -DLU_TRACE)
__device__ long long g_lu_trace[8];
#define LU_T0() long long lu_t = clock64()
#define LU_T(i)                                                  \
  do {                                                           \
    const long long lu_n = clock64();                            \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_lu_trace[i] += lu_n - lu_t; \
    lu_t = lu_n;                                                 \
  } while (0)
#else
#define LU_T0()
#define LU_T(i)
#endif

template <int PW>
__global__ void __launch_bounds__(sk::kThreads, 1) k_lupp(LuArgs a) {
  cg::grid_group grid = cg::this_grid();
  constexpr int LD = PW + 1, CS = PW + 2, NW = sk::kThreads / 32;
  constexpr int LA1 = PW >= 32 ? 4 : 8, LA = 8;   // multipliers loaded per batch in (1), (2)
  constexpr int HW = PW > 16 ? 16 : PW, NH = PW / HW;   // (2): columns per work item
  extern __shared__ __align__(16) double smd[];
  const int R = a.R, k = a.k, G = gridDim.x;
  double* A = smd;                                       // R x LD: own rows, panel columns
  double* Us = A + (size_t)R * LD;                       // k x PW: U rows of earlier pivots
  double* Up = Us + (size_t)k * PW;                      // PW: the current pivot row
  long long* spiv = reinterpret_cast<long long*>(Up + PW);   // k: pivot rows so far
  unsigned char* act = reinterpret_cast<unsigned char*>(spiv + k);   // R: row still active
  __shared__ double s_wv[NW];
  __shared__ long long s_wr[NW];
  __shared__ int s_wg[NW];
  __shared__ double s_bv;
  __shared__ int s_win;
  __shared__ long long s_br;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * R;
  const int nr = (int)max((int64_t)0, min((int64_t)R, a.n - r0));
  for (int i = tid; i < R; i += sk::kThreads) act[i] = i < nr ? 1 : 0;
  __syncthreads();
  int npiv = 0, par = 0;
  int64_t c = 0;
  LU_T0();
  while (npiv < k && c < a.l) {
    const int64_t c0 = c;
    const int pw = (int)min((int64_t)PW, a.l - c0);
    const int np0 = npiv;
    // (1) U(m, c0 + j), m < np0: Y(p_m, .) minus the earlier pivots' updates, in order.
    // Thread m holds U row m in registers; step mm publishes the (final) row mm in smem,
    // then every row m > mm subtracts L(p_m, mm) U(mm, .).  The multipliers of row m are
    // read LA1 steps ahead (one batch of loads in flight while the previous 8 steps run).
    {
      double u[PW];
      const bool own = tid < np0;
      const int64_t prow = own ? spiv[tid] : 0;   // U row tid = Y(p_tid, .) - ...
      if (own) {
        const double* yr = a.Y + prow * a.ldy + c0;
#pragma unroll
        for (int j = 0; j < PW; ++j) u[j] = j < pw ? yr[j] : 0.0;
      }
      const double* lr = a.Lp + (own ? tid : 0) * k;
      double lcur[LA1], lnext[LA1];
#pragma unroll
      for (int t = 0; t < LA1; ++t) lcur[t] = (own && t < tid) ? lr[t] : 0.0;
      for (int mg = 0; mg < np0; mg += LA1) {
#pragma unroll
        for (int t = 0; t < LA1; ++t) lnext[t] = (own && mg + LA1 + t < tid) ? lr[mg + LA1 + t] : 0.0;
#pragma unroll
        for (int t = 0; t < LA1; ++t) {
          const int mm = mg + t;
          if (mm >= np0) break;
          if (tid == mm) {
#pragma unroll
            for (int j = 0; j < PW; ++j) Us[mm * PW + j] = u[j];
          }
          __syncthreads();
          if (own && tid > mm) {
            const double lm = lcur[t];
            const double* ur = Us + mm * PW;
#pragma unroll
            for (int j = 0; j < PW; ++j) u[j] = __dsub_rn(u[j], __dmul_rn(lm, ur[j]));
          }
        }
#pragma unroll
        for (int t = 0; t < LA1; ++t) lcur[t] = lnext[t];
      }
      __syncthreads();
    }
    LU_T(0);
    // (2) own active rows: panel columns of Y, then the earlier pivots' updates in order,
    // held in registers (columns >= pw carry unused values).  Work items are (row, group
    // of HW columns): every entry's update sequence is its own, so the split is exact.
    for (int e = tid; e < nr * NH; e += sk::kThreads) {
      const int i = e / NH, h = e - i * NH;
      if (!act[i]) continue;
      const int j0 = h * HW;
      const double* yr = a.Y + (r0 + i) * a.ldy + c0 + j0;
      double rv[HW];
#pragma unroll
      for (int j = 0; j < HW; ++j) rv[j] = j0 + j < pw ? yr[j] : 0.0;
      const double* lr = a.Lm + r0 + i;   // column-major: coalesced over the CTA's rows
      for (int mg = 0; mg < np0; mg += LA) {
        double lb[LA];
#pragma unroll
        for (int t = 0; t < LA; ++t) lb[t] = mg + t < np0 ? lr[(size_t)(mg + t) * a.n] : 0.0;
#pragma unroll
        for (int t = 0; t < LA; ++t) {
          if (mg + t >= np0) break;
          const double* u = Us + (mg + t) * PW + j0;
#pragma unroll
          for (int j = 0; j < HW; ++j) rv[j] = __dsub_rn(rv[j], __dmul_rn(lb[t], u[j]));
        }
      }
      double* ar = A + (size_t)i * LD + j0;
#pragma unroll
      for (int j = 0; j < HW; ++j) ar[j] = rv[j];
    }
    __syncthreads();
    LU_T(1);
    // (3) the panel's steps
    int s = 0;
    for (; s < pw && npiv < k; ++s) {
      double bv = -1.0;
      long long br = LLONG_MAX;
      int bl = -1;
      for (int i = tid; i < nr; i += sk::kThreads)
        if (act[i]) {
          const double v = fabs(A[(size_t)i * LD + s]);
          if (v > bv) {   // rows visited in increasing order: ties keep the lower row
            bv = v;
            bl = i;
            br = r0 + i;
          }
        }
      lu_warp_best(bv, br, bl);
      if (lane == 0) {
        s_wv[w] = bv;
        s_wr[w] = br;
        s_wg[w] = bl;
      }
      __syncthreads();
      // warp 0: the CTA's candidate (|v|, row, its pw <= 32 panel values); the grid barrier
      // below starts with a CTA barrier
      if (w == 0) {
        double v = lane < NW ? s_wv[lane] : -1.0;
        long long r = lane < NW ? s_wr[lane] : LLONG_MAX;
        int li = lane < NW ? s_wg[lane] : -1;
        lu_warp_best(v, r, li);
        double* cr = a.cand + ((size_t)par * G + blockIdx.x) * CS;
        if (li >= 0 && lane < pw) cr[2 + lane] = A[(size_t)li * LD + lane];
        if (lane == 0) {
          cr[0] = v;
          cr[1] = __longlong_as_double(li >= 0 ? (long long)(r0 + li) : -1ll);
        }
      }
      LU_T(2);
      grid.sync();
      LU_T(3);
      // the winner, identical in every CTA: warp 0 reads every candidate through L2 (lane
      // l takes candidates l, l + 32, ...; all loads issued before the compares), then a
      // warp argmax
      if (w == 0) {
        double v = -1.0;
        long long r = LLONG_MAX;
        int who = -1;
        for (int gb = 0; gb < G; gb += 32 * sk::kCandPerLane) {
          double qv[sk::kCandPerLane];
          long long qr[sk::kCandPerLane];
#pragma unroll
          for (int u = 0; u < sk::kCandPerLane; ++u) {
            const int g = gb + lane + 32 * u;
            const double* q = a.cand + ((size_t)par * G + g) * CS;
            qv[u] = g < G ? __ldcg(q) : -1.0;
            qr[u] = g < G ? __double_as_longlong(__ldcg(q + 1)) : -1ll;
          }
#pragma unroll
          for (int u = 0; u < sk::kCandPerLane; ++u)
            if (qr[u] >= 0 && lu_better(qv[u], qr[u], v, r)) {
              v = qv[u];
              r = qr[u];
              who = gb + lane + 32 * u;
            }
        }
        lu_warp_best(v, r, who);
        // the winner's panel values and the bookkeeping, before the CTA barrier
        if (who >= 0 && v > 0.0) {
          const double* q = a.cand + ((size_t)par * G + who) * CS;
          if (lane < pw) Up[lane] = __ldcg(q + 2 + lane);
          if (lane == 0) {
            spiv[npiv] = r;
            if (r >= r0 && r < r0 + nr) act[r - r0] = 0;
            if (blockIdx.x == 0) {
              a.piv[npiv] = r;
              a.pcol[npiv] = c0 + s;
            }
          }
        }
        if (lane == 0) {
          s_bv = v;
          s_br = r;
          s_win = who;
        }
      }
      __syncthreads();
      LU_T(4);
      par ^= 1;
      if (s_win < 0) {   // no active row left anywhere
        c = a.l;
        break;
      }
      if (!(s_bv > 0.0)) continue;   // exactly zero active column: skipped (no pivot)
      const long long prow = s_br;
      const int m = npiv++;
      // the owner files the new pivot row's multipliers for (1) of later panels
      if (prow >= r0 && prow < r0 + nr)
        for (int mm = tid; mm < m; mm += sk::kThreads) a.Lp[(size_t)m * k + mm] = a.Lm[(size_t)mm * a.n + prow];
      const double pv = Up[s];
      for (int i = tid; i < nr; i += sk::kThreads) {
        if (!act[i]) continue;
        double* ar = A + (size_t)i * LD;
        const double lv = ar[s] / pv;
        a.Lm[(size_t)m * a.n + r0 + i] = lv;
        for (int j = s + 1; j < pw; ++j) ar[j] = __dsub_rn(ar[j], __dmul_rn(lv, Up[j]));
      }
      __syncthreads();
      LU_T(5);
    }
    if (c < a.l) c = c0 + s;
    grid.sync();   // this panel's multipliers are read by every CTA in (1) of the next
    LU_T(6);
  }
  if (blockIdx.x == 0 && tid == 0) a.out[0] = npiv;
}

static int sk_num_sms() {
  const int v = device_sms();
  return v;
}

static size_t lupp_smem(int PW, int R, int k) {
  return (size_t)R * (PW + 1) * 8 + (size_t)k * PW * 8 + PW * 8 + (size_t)k * 8 + R + 64;
}

// grid and panel width for n rows: one CTA per SM, the widest panel that fits
static bool lupp_plan(int64_t n, int k, int* G, int* R, int* PW) {
  const int sms = sk_num_sms();
  *G = (int)std::min<int64_t>(sms, n);
  *R = (int)((n + *G - 1) / *G);
  const char* cap = getenv("RBRP_LUPP_PW");   // test knob: largest panel width tried
  const int pw_max = cap ? atoi(cap) : 32;
  for (int pw : {32, 16, 8})
    if (pw <= pw_max && lupp_smem(pw, *R, k) <= (size_t)sk::kSmemMax) {
      *PW = pw;
      return true;
    }
  return false;
}

template <int PW>
static cudaError_t go_lupp(LuArgs a, int G, cudaStream_t s) {
  const size_t smem = lupp_smem(PW, a.R, a.k);
  cudaError_t e = cudaFuncSetAttribute(k_lupp<PW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(sk::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeCooperative;
  la[0].val.cooperative = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_lupp<PW>, a);
}

static cudaError_t launch_lupp(LuArgs a, int G, int PW, cudaStream_t s) {
  switch (PW) {
    case 32: return go_lupp<32>(a, G, s);
    case 16: return go_lupp<16>(a, G, s);
    default: return go_lupp<8>(a, G, s);
  }
}

// B (cols x rows, row-major) = A^T, A rows x cols row-major; 32 x 32 tiles through smem
__global__ void k_transpose(const double* __restrict__ A, int64_t rows, int64_t cols, double* __restrict__ B) {
  __shared__ double t[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int64_t r = r0 + y, c = c0 + threadIdx.x;
    t[y][threadIdx.x] = (r < rows && c < cols) ? A[r * cols + c] : 0.0;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int64_t c = c0 + y, r = r0 + threadIdx.x;
    if (c < cols && r < rows) B[c * rows + r] = t[threadIdx.x][y];
  }
}

// ------------------------------------------------------------------------------------
// OSID helpers (small k x k and k x l steps)
// ------------------------------------------------------------------------------------
__global__ void k_gather_rows(const double* __restrict__ Y, int64_t ldy, const int64_t* __restrict__ S, int k,
                              int64_t lp, double* __restrict__ Z) {
  const int i = blockIdx.x;
  if (i >= k) return;
  const double* y = Y + S[i] * ldy;
  for (int64_t c = threadIdx.x; c < lp; c += blockDim.x) Z[(int64_t)i * lp + c] = y[c];
}

// C (M x N, ldc) = sum_t A(i, t) B(t, j) with A(i, t) = A[i sa0 + t sa1], B(t, j) =
// B[t sb0 + j sb1] (any transposition); tri = 1: A(i, t) = 0 for t > i, tri = 2: for t < i
// (the zero triangle is neither read nor trusted); lower_only: tiles above the diagonal
// of C skipped (a Gram matrix whose lower part is used).  32 x 32 tiles, K in chunks of 32
// through smem, 2 x 2 outputs per thread; for the k x k and k x l steps of OSID.
__global__ void __launch_bounds__(256) k_dgemm_small(const double* __restrict__ A, int64_t sa0, int64_t sa1,
                                                     const double* __restrict__ B, int64_t sb0, int64_t sb1,
                                                     double* __restrict__ C, int64_t ldc, int M, int N, int K,
                                                     int tri, int lower_only) {
  __shared__ double As[32][33], Bs[32][33];   // As[r][q] = A(i0 + r, t0 + q), Bs[r][q] = B(t0 + r, j0 + q)
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (lower_only && bj > bi) return;
  const int i0 = bi * 32, j0 = bj * 32;
  const int t_lo = tri == 2 ? i0 : 0, t_hi = tri == 1 ? min(K, i0 + 32) : K;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const bool a_row = sa1 == 1, b_row = sb1 == 1;   // the contiguous index runs over the lanes
  double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
  for (int t0 = t_lo; t0 < t_hi; t0 += 32) {
    for (int e = threadIdx.x; e < 1024; e += 256) {
      const int f = e >> 5, g = e & 31;
      {
        const int r = a_row ? f : g, q = a_row ? g : f;
        const int i = i0 + r, t = t0 + q;
        const bool z = i >= M || t >= t_hi || (tri == 1 && t > i) || (tri == 2 && t < i);
        As[r][q] = z ? 0.0 : A[(int64_t)i * sa0 + (int64_t)t * sa1];
      }
      {
        const int r = b_row ? f : g, q = b_row ? g : f;
        const int t = t0 + r, j = j0 + q;
        Bs[r][q] = (t >= t_hi || j >= N) ? 0.0 : B[(int64_t)t * sb0 + (int64_t)j * sb1];
      }
    }
    __syncthreads();
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
      const double a0 = As[ty][q], a1 = As[ty + 16][q], b0 = Bs[q][tx], b1 = Bs[q][tx + 16];
      c00 = fma(a0, b0, c00);
      c01 = fma(a0, b1, c01);
      c10 = fma(a1, b0, c10);
      c11 = fma(a1, b1, c11);
    }
    __syncthreads();
  }
  const int i = i0 + ty, j = j0 + tx;
  if (i < M && j < N) C[(int64_t)i * ldc + j] = c00;
  if (i < M && j + 16 < N) C[(int64_t)i * ldc + j + 16] = c01;
  if (i + 16 < M && j < N) C[(int64_t)(i + 16) * ldc + j] = c10;
  if (i + 16 < M && j + 16 < N) C[(int64_t)(i + 16) * ldc + j + 16] = c11;
}

static void dgemm_small(const double* A, int64_t sa0, int64_t sa1, const double* B, int64_t sb0, int64_t sb1,
                        double* C, int64_t ldc, int M, int N, int K, int tri, int lower_only, cudaStream_t s) {
  k_dgemm_small<<<dim3((unsigned)((N + 31) / 32), (unsigned)((M + 31) / 32)), 256, 0, s>>>(
      A, sa0, sa1, B, sb0, sb1, C, ldc, M, N, K, tri, lower_only);
}

// Blocked right-looking Cholesky (C = G's lower factor, in place in C after a copy of G):
// per 32-column panel, k_chol_panel factors the diagonal block and solves the rows below
// it (a warp per row), then k_chol_update applies C_below C_below^T to the trailing
// matrix, a CTA per 32 x 32 lower block.
constexpr int kCholNB = 32;

// Panel j0: warp 0 of every CTA factors the diagonal block (lane i holds row i in
// registers, column j's multipliers broadcast by shuffles), then each warp solves one row
// below it: x D^T = g, x_q = (g_q - sum_{t<q} x_t D(q, t)) / D(q, q), t ascending.  The
// diagonal block is read by every CTA, so the factor goes to Dbuf (copied into C after
// the last panel) and C's diagonal block stays untouched until then; CTA 0 zeroes the
// panel rows right of the block.
__global__ void __launch_bounds__(256) k_chol_panel(double* __restrict__ C, int k, int j0,
                                                    double* __restrict__ Dbuf, int* __restrict__ info) {
  __shared__ double D[kCholNB][kCholNB + 1];
  __shared__ double Dinv[kCholNB];
  const int jb = min(kCholNB, k - j0), lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w == 0) {
    double r[kCholNB];
    const double* src = C + (size_t)(j0 + min(lane, jb - 1)) * k + j0;
#pragma unroll
    for (int q = 0; q < kCholNB; ++q) r[q] = (lane < jb && q <= lane) ? src[q] : 0.0;
    bool bad = false;
#pragma unroll
    for (int j = 0; j < kCholNB; ++j) {
      if (j < jb) {
        double djj = __shfl_sync(0xffffffffu, r[j], j);
        if (!(djj > 0.0)) {
          bad = true;
          djj = 1.0;
        }
        const double rs = rsqrt(djj);   // one reciprocal square root per step: the
        r[j] = lane > j ? r[j] * rs : (lane == j ? djj * rs : 0.0);   // chain is 32 steps long
#pragma unroll
        for (int q = j + 1; q < kCholNB; ++q) {
          const double lqj = __shfl_sync(0xffffffffu, r[j], q);
          if (lane >= q) r[q] = fma(-r[j], lqj, r[q]);
        }
      }
    }
    if (blockIdx.x == 0 && lane == 0 && bad) *info = 1;
#pragma unroll
    for (int q = 0; q < kCholNB; ++q) D[lane][q] = (lane < jb && q <= lane) ? r[q] : 0.0;
    __syncwarp();
    Dinv[lane] = lane < jb ? 1.0 / D[lane][lane] : 0.0;
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    double* db = Dbuf + (size_t)(j0 / kCholNB) * kCholNB * kCholNB;
    for (int e = threadIdx.x; e < kCholNB * kCholNB; e += blockDim.x) db[e] = D[e >> 5][e & 31];
    const int wr = k - j0 - jb;
    for (int e = threadIdx.x; e < jb * wr; e += blockDim.x) {
      const int i = e / wr, q = e - i * wr;
      C[(size_t)(j0 + i) * k + j0 + jb + q] = 0.0;
    }
  }
  const int i = j0 + kCholNB + blockIdx.x * 8 + w;
  if (i >= k) return;
  double* row = C + (size_t)i * k + j0;
  double acc = row[lane];
  double x = 0.0;
#pragma unroll
  for (int t = 0; t < kCholNB; ++t) {
    if (lane == t) x = acc * Dinv[t];
    const double xt = __shfl_sync(0xffffffffu, x, t);
    if (lane > t) acc = fma(-xt, D[lane][t], acc);
  }
  row[lane] = x;
}

// the factored diagonal blocks from Dbuf into C (block b per CTA)
__global__ void k_chol_diag_store(double* __restrict__ C, int k, const double* __restrict__ Dbuf) {
  const int b = blockIdx.x, j0 = b * kCholNB, jb = min(kCholNB, k - j0);
  for (int e = threadIdx.x; e < kCholNB * kCholNB; e += blockDim.x) {
    const int r = e >> 5, q = e & 31;
    if (r < jb && q < jb) C[(size_t)(j0 + r) * k + j0 + q] = Dbuf[(size_t)b * kCholNB * kCholNB + e];
  }
}

// trailing update C(i, q) -= sum_t C(i, j0 + t) C(q, j0 + t), j1 = j0 + 32 <= q <= i < k;
// one 32 x 32 block of (i, q) per CTA (lower blocks only), panel rows staged in smem
__global__ void __launch_bounds__(1024) k_chol_update(double* __restrict__ C, int k, int j0) {
  __shared__ double Pi[kCholNB][kCholNB + 1], Pq[kCholNB][kCholNB + 1];
  const int j1 = j0 + kCholNB;
  const int bi = blockIdx.y, bq = blockIdx.x;
  if (bq > bi) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int i0 = j1 + bi * kCholNB, q0 = j1 + bq * kCholNB;
  {
    const int ri = i0 + ty, rq = q0 + ty;
    Pi[ty][tx] = ri < k ? C[(size_t)ri * k + j0 + tx] : 0.0;
    Pq[ty][tx] = rq < k ? C[(size_t)rq * k + j0 + tx] : 0.0;
  }
  __syncthreads();
  const int i = i0 + ty, q = q0 + tx;
  if (i >= k || q > i) return;
  double v = C[(size_t)i * k + q];
#pragma unroll
  for (int t = 0; t < kCholNB; ++t) v = fma(-Pi[ty][t], Pq[tx][t], v);
  C[(size_t)i * k + q] = v;
}

// G (k x k) = C C^T, C lower with zeros above the diagonal; info = 1 if not positive
// definite.  Dbuf: ceil(k / 32) blocks of 32 x 32 doubles.
static cudaError_t chol_blocked(const double* G, int k, double* C, double* Dbuf, int* info, cudaStream_t s,
                                int* launches) {
  cudaError_t e = cudaMemcpyAsync(C, G, (size_t)k * k * 8, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return e;
  for (int j0 = 0; j0 < k; j0 += kCholNB) {
    const int m = k - j0 - kCholNB;   // rows below the diagonal block
    k_chol_panel<<<m > 0 ? (m + 7) / 8 : 1, 256, 0, s>>>(C, k, j0, Dbuf, info);
    ++*launches;
    if (m > 0) {
      const int nb = (m + kCholNB - 1) / kCholNB;
      k_chol_update<<<dim3(nb, nb), dim3(kCholNB, kCholNB), 0, s>>>(C, k, j0);
      ++*launches;
    }
  }
  k_chol_diag_store<<<(k + kCholNB - 1) / kCholNB, 256, 0, s>>>(C, k, Dbuf);
  ++*launches;
  return cudaGetLastError();
}


}  // namespace rbrp

using namespace rbrp;

namespace {

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
int64_t round8(int64_t x) { return (x + 7) & ~int64_t(7); }

struct LuLayout {
  size_t Lm, Lp, cand, piv, pcol, out, total;
};
LuLayout lu_layout(int64_t n, int64_t k, int G) {
  LuLayout L{};
  size_t o = 0;
  L.Lm = o;
  o += al256((size_t)n * k * 8);
  L.Lp = o;
  o += al256((size_t)k * k * 8);
  L.cand = o;
  o += al256((size_t)2 * G * (32 + 2) * 8);
  L.piv = o;
  o += al256((size_t)k * 8);
  L.pcol = o;
  o += al256((size_t)k * 8);
  L.out = o;
  o += 256;
  L.total = o;
  return L;
}

int lupp_check(int64_t n, int64_t l, int64_t ldy, int64_t k) {
  if (n < 1 || l < 1 || ldy < l || k < 1 || k > n || k > l || k > RBRP_SK_MAX_K) return RBRP_EINVAL;
  return RBRP_OK;
}

// run the LUPP kernel; pivots copied to the host (synchronises the stream)
// L_out (n x k row-major, optional): the multipliers, zero where a row was not active
int run_lupp(const double* Y, int64_t n, int64_t l, int64_t ldy, int64_t k, char* ws, double* L_out,
             cudaStream_t s, int64_t* piv_h, int64_t* pcol_h, int64_t* npiv_h, int64_t** piv_dev) {
  int G, R, PW;
  if (!lupp_plan(n, (int)k, &G, &R, &PW)) return RBRP_ENOTSUP;
  LuLayout Ly = lu_layout(n, k, G);
  double* Lm = (double*)(ws + Ly.Lm);
  // the kernel reads only multipliers it wrote; zeros matter for the exported L only
  if (L_out && cudaMemsetAsync(Lm, 0, (size_t)n * k * 8, s) != cudaSuccess) return RBRP_ECUDA;
  LuArgs a;
  a.Y = Y;
  a.n = n;
  a.l = l;
  a.ldy = ldy;
  a.k = (int)k;
  a.R = R;
  a.Lm = Lm;
  a.Lp = (double*)(ws + Ly.Lp);
  a.cand = (double*)(ws + Ly.cand);
  a.piv = (int64_t*)(ws + Ly.piv);
  a.pcol = (int64_t*)(ws + Ly.pcol);
  a.out = (int*)(ws + Ly.out);
  if (launch_lupp(a, G, PW, s) != cudaSuccess) return RBRP_ECUDA;
  if (L_out) {
    k_transpose<<<dim3((unsigned)((n + 31) / 32), (unsigned)((k + 31) / 32)), dim3(32, 8), 0, s>>>(Lm, k, n, L_out);
    if (cudaGetLastError() != cudaSuccess) return RBRP_ECUDA;
  }
  int np = 0;
  if (cudaMemcpyAsync(&np, a.out, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess) return RBRP_ECUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return RBRP_ECUDA;
  *npiv_h = np;
  if (np > 0 && piv_h && cudaMemcpy(piv_h, a.piv, np * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return RBRP_ECUDA;
  if (np > 0 && pcol_h && cudaMemcpy(pcol_h, a.pcol, np * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
    return RBRP_ECUDA;
  if (piv_dev) *piv_dev = a.piv;
  return RBRP_OK;
}

struct SkLayout {
  size_t OmT, Y, lu, Z, P, G, C1, C2, A1T, A2T, st, gsc, Db, info, total;
  int64_t lp;
};
SkLayout sk_layout(int64_t n, int64_t d, int64_t k, int64_t l) {
  SkLayout L{};
  L.lp = round8(l);
  int G = (int)std::min<int64_t>(sk_num_sms(), n);
  size_t o = 0;
  L.OmT = o;
  o += al256((size_t)L.lp * d * 8);
  L.Y = o;
  o += al256((size_t)n * L.lp * 8);
  L.lu = o;
  o += lu_layout(n, k, G).total;
  L.Z = o;
  o += al256((size_t)k * L.lp * 8);
  L.P = o;
  o += al256((size_t)k * L.lp * 8);
  L.A1T = o;
  o += al256((size_t)k * k * 8);
  L.A2T = o;
  o += al256((size_t)k * k * 8);
  L.st = o;
  o += al256(sizeof(DevState));
  L.gsc = o;
  o += al256(std::max(gemm_lp_scratch_bytes(L.lp, d), gemm_lp_scratch_bytes(k, L.lp)));
  L.G = o;
  o += al256((size_t)k * k * 8);
  L.C1 = o;
  o += al256((size_t)k * k * 8);
  L.C2 = o;
  o += al256((size_t)k * k * 8);
  L.Db = o;
  o += al256((size_t)((k + 31) / 32) * 32 * 32 * 8);
  L.info = o;
  o += 256;
  L.total = o;
  return L;
}

int sk_check(int64_t n, int64_t d, int64_t ldx, int64_t k, int64_t l) {
  if (n < 1 || d < 1 || ldx < d || k < 1 || k > n || k > RBRP_SK_MAX_K || l < k || l > 4 * k)
    return RBRP_EINVAL;
  return RBRP_OK;
}

struct Ev {
  cudaEvent_t e[2] = {nullptr, nullptr};
  bool on = false;
  void begin(bool p, cudaStream_t s) {
    on = p;
    if (!on) return;
    cudaEventCreate(&e[0]);
    cudaEventCreate(&e[1]);
    cudaEventRecord(e[0], s);
  }
  float end(cudaStream_t s) {
    if (!on) return 0.f;
    float ms = 0.f;
    cudaEventRecord(e[1], s);
    cudaEventSynchronize(e[1]);
    cudaEventElapsedTime(&ms, e[0], e[1]);
    cudaEventDestroy(e[0]);
    cudaEventDestroy(e[1]);
    return ms;
  }
};

}  // namespace

extern "C" {

#ifdef LU_TRACE
int rbrp_debug_lu_trace(long long* out, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, g_lu_trace, sizeof(long long) * 8) != cudaSuccess) return RBRP_ECUDA;
  if (reset) {
    long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_lu_trace, z, sizeof(z));
  }
  return RBRP_OK;
}
#endif

int rbrp_gaussian_embedding(int64_t d, int64_t l, uint64_t seed, double* OmegaT, int64_t ldo, void* stream) {
  if (d < 1 || l < 1 || ldo < d || !OmegaT) return RBRP_EINVAL;
  const int64_t nq = (d * l + 1) / 2;
  const int blocks = (int)std::min<int64_t>((nq + 255) / 256, 148 * 16);
  k_embedding<<<blocks, 256, 0, (cudaStream_t)stream>>>(d, l, make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)),
                                                         OmegaT, ldo);
  return cudaGetLastError() == cudaSuccess ? RBRP_OK : RBRP_ECUDA;
}

int rbrp_lupp_workspace_size(int64_t n, int64_t l, int64_t k, size_t* bytes) {
  int rc = lupp_check(n, l, l, k);
  if (rc) return rc;
  if (!bytes) return RBRP_EINVAL;
  *bytes = lu_layout(n, k, (int)std::min<int64_t>(sk_num_sms(), n)).total;
  return RBRP_OK;
}

int rbrp_lupp(const double* Y, int64_t n, int64_t l, int64_t ldy, int64_t k, void* workspace, size_t ws_bytes,
              void* stream, int64_t* piv_out, int64_t* pcol_out, int64_t* npiv_out, double* L_out) {
  int rc = lupp_check(n, l, ldy, k);
  if (rc) return rc;
  if (!Y || !workspace || !piv_out || !npiv_out || ((uintptr_t)workspace % 256)) return RBRP_EINVAL;
  size_t need = 0;
  rbrp_lupp_workspace_size(n, l, k, &need);
  if (ws_bytes < need) return RBRP_ENOMEM;
  return run_lupp(Y, n, l, ldy, k, (char*)workspace, L_out, (cudaStream_t)stream, piv_out, pcol_out, npiv_out,
                  nullptr);
}

int rbrp_sketch_workspace_size(int64_t n, int64_t d, int64_t k, int64_t l, size_t* bytes) {
  int rc = sk_check(n, d, d, k, l);
  if (rc) return rc;
  if (!bytes) return RBRP_EINVAL;
  *bytes = sk_layout(n, d, k, l).total;
  return RBRP_OK;
}

int rbrp_sketch_id(const double* X, int64_t n, int64_t d, int64_t ldx, int64_t k, int64_t l, uint64_t seed,
                   const double* OmegaT, void* workspace, size_t ws_bytes, void* stream, int64_t* S_out,
                   double* W_out, rbrp_sketch_report* rep) {
  int rc = sk_check(n, d, ldx, k, l);
  if (rc) return rc;
  if (!X || !workspace || !S_out || ((uintptr_t)workspace % 256)) return RBRP_EINVAL;
  if (d % 8 || ldx % 2 || ((uintptr_t)X % 16)) return RBRP_ENOTSUP;
  SkLayout Ly = sk_layout(n, d, k, l);
  if (ws_bytes < Ly.total) return RBRP_ENOMEM;
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  const int64_t lp = Ly.lp;
  double* OmT = (double*)(ws + Ly.OmT);
  double* Y = (double*)(ws + Ly.Y);
  double* Z = (double*)(ws + Ly.Z);
  double* Gm = (double*)(ws + Ly.G);
  double* C1 = (double*)(ws + Ly.C1);
  double* C2 = (double*)(ws + Ly.C2);
  int* info = (int*)(ws + Ly.info);
  double* Dbuf = (double*)(ws + Ly.Db);
  const bool prof = rep && rep->profile;
  int launches = 0;
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  cudaEventRecord(t0, s);
  float ph[4] = {0, 0, 0, 0};
  Ev ev;
#define SK(x)                                   \
  do {                                          \
    if ((x) != cudaSuccess) return RBRP_ECUDA;  \
  } while (0)
  // Alg. 4 l.1: Omega (rows l .. lp of Omega^T are zero, so Y's padding columns are 0)
  ev.begin(prof, s);
  SK(cudaMemsetAsync(OmT + l * d, 0, (size_t)(lp - l) * d * 8, s));
  if (OmegaT) {
    SK(cudaMemcpyAsync(OmT, OmegaT, (size_t)l * d * 8, cudaMemcpyDeviceToDevice, s));
  } else {
    if ((rc = rbrp_gaussian_embedding(d, l, seed, OmT, d, stream))) return rc;
    ++launches;
  }
  ph[0] = ev.end(s);
  // Y = X Omega
  ev.begin(prof, s);
  cudaError_t ge = cudaSuccess;
  void* gsc = ws + Ly.gsc;
  if (gemm_lp_supported(X, ldx, OmT, d, d)) {   // 32-column read-only DMMA passes
    SK(gemm_nt_lp(X, ldx, OmT, d, Y, lp, n, lp, d, gsc, s));
    launches += 1 + 2 * (int)((lp + 31) / 32);
  } else {
    if (!gemm_nt_mma(X, ldx, OmT, d, Y, lp, n, lp, d, s, &ge)) return RBRP_ENOTSUP;
    SK(ge);
    ++launches;
  }
  ph[1] = ev.end(s);
  // S = the first k LUPP pivots of Y
  ev.begin(prof, s);
  int64_t np = 0;
  int64_t* Sdev = nullptr;
  rc = run_lupp(Y, n, l, lp, k, ws + Ly.lu, nullptr, s, S_out, nullptr, &np, &Sdev);
  if (rc) return rc;
  launches += 1;
  ph[2] = ev.end(s);
  uint32_t flags = np < k ? RBRP_SK_SHORT : 0;
  // OSID (Alg. 4 l.2-4): W = Y Y_S^+ = Y M, M^T = G1^{-1} Z via CholQR2 of Z^T
  ev.begin(prof, s);
  if (np > 0 && W_out) {
    const int kk = (int)np;
    double* P = (double*)(ws + Ly.P);
    double* A1T = (double*)(ws + Ly.A1T);
    double* A2T = (double*)(ws + Ly.A2T);
    DevState* dst = (DevState*)(ws + Ly.st);
    SK(cudaMemsetAsync(info, 0, sizeof(int), s));
    SK(cudaMemsetAsync(dst, 0, sizeof(DevState), s));
    auto chol = [&](double* Cout) -> cudaError_t {   // Gm = Cout Cout^T
      return chol_blocked(Gm, kk, Cout, Dbuf, info, s, &launches);
    };
    k_gather_rows<<<kk, 256, 0, s>>>(Y, lp, Sdev, kk, lp, Z);          // Z = Y(S,:)
    dgemm_small(Z, lp, 1, Z, 1, lp, Gm, kk, kk, kk, (int)lp, 0, 1, s);   // G1 = Z Z^T (lower part)
    SK(chol(C1));                                                       // G1 = C1 C1^T (R1 = C1^T)
    SK(launch_trinv<double>(C1, kk, A1T, kk, dst, s));                 // A1T = C1^{-T}
    dgemm_small(A1T, 1, kk, Z, lp, 1, P, lp, kk, (int)lp, kk, 1, 0, s);  // P1 = C1^{-1} Z = A1T^T Z = Q1^T
    dgemm_small(P, lp, 1, P, 1, lp, Gm, kk, kk, kk, (int)lp, 0, 1, s);   // G2 = P1 P1^T
    SK(chol(C2));                                                       // G2 = C2 C2^T (R2 = C2^T)
    SK(launch_trinv<double>(C2, kk, A2T, kk, dst, s));                 // A2T = C2^{-T}
    dgemm_small(A2T, 1, kk, P, lp, 1, Z, lp, kk, (int)lp, kk, 1, 0, s);  // Q^T = C2^{-1} P1
    dgemm_small(A2T, kk, 1, Z, lp, 1, P, lp, kk, (int)lp, kk, 2, 0, s);  // R2^{-1} Q^T (A2T upper)
    dgemm_small(A1T, kk, 1, P, lp, 1, Z, lp, kk, (int)lp, kk, 2, 0, s);  // M^T = R1^{-1} R2^{-1} Q^T
    SK(cudaGetLastError());
    launches += 9;
    if (gemm_lp_supported(Y, lp, Z, lp, lp, 256)) {                                   // W = Y M
      SK(gemm_nt_lp(Y, lp, Z, lp, W_out, k, n, kk, lp, gsc, s, false, 256));
      launches += 2 * (kk + 31) / 32;
    } else {
      if (!gemm_nt_mma(Y, lp, Z, lp, W_out, k, n, kk, lp, s, &ge)) return RBRP_ENOTSUP;
      SK(ge);
    }
    SK(launch_w_identity<double>(W_out, k, Sdev, kk, n, 0, s));                         // W(S,:) = I
    launches += 2;
  }
  ph[3] = ev.end(s);
  int hinfo = 0;
  SK(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, s));
  cudaEventRecord(t1, s);
  SK(cudaEventSynchronize(t1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
#undef SK
  if (rep) {
    rep->k = np;
    rep->flags = flags;
    rep->ms_total = ms;
    for (int i = 0; i < 4; ++i) rep->ms_phase[i] = ph[i];
    rep->launches = launches;
  }
  return (np > 0 && W_out && hinfo) ? RBRP_EDEGENERATE : RBRP_OK;
}

}  // extern "C"
