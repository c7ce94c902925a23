// k_formw.cu — a6 interpolation matrix, Alg. 3.
//
// L_1 = L(S,:) is exactly lower-triangular in selection order (reading R13), so
// L_2 L_1^{-1} is a triangular solve (north_star step 6).  We form
// L_1^{-1} once (k_trinv: one warp per column, forward substitution in fp64), then
// W = L L_1^{-1} for all local rows with the tile GEMM (k_gemm_nt, B = L_1^{-T}), and
// finally W(S,:) = I exactly (Alg. 3 l.2).
//
// Remark 5.2: L_1 from (R)BRP "tends to be ill-conditioned", and the paper
// then evaluates L_1^{-1} by a clipped SVD.  Reading R17: when min |diag L_1| <
// 1e-12 max |diag L_1| (the host tests the running min/max k_fixup keeps in DevState, or
// k_diag_test for a standalone rbrp_form_w), W(rest,:) = L_2 pinv_clip(L_1) with the
// singular values below 1e-12 sigma_max discarded, and W_CLIPPED is reported.  The SVD
// is a one-sided (Hestenes) Jacobi SVD of A = L_1^T in fp64 (k_jacobi_svd, cooperative,
// round-robin pairs, high relative accuracy for the small singular values), then
// pinv_clip(L_1)^T = V Sigma^+ U^T = sum_l sigma_l^-2 V_l (A V)_l^T (k_pinv_form).
#include <cooperative_groups.h>
#include <float.h>

#include <algorithm>

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

// Blocked inversion of the lower-triangular L_1 in place, one cooperative kernel (the
// substitution kernels above chain k dependent steps; this one chains log2(k / 32) levels
// of small GEMMs spread over the whole GPU):
//   phase 0  the strictly upper triangle of L_1 is zeroed; every 32 x 32 diagonal block is
//            inverted in place (one warp per block, thread j = column j, substitution)
//   level s  (s = 32, 64, ...) for every pair of inverted diagonal blocks A (rows/cols
//            [2ps, 2ps + s)) and C (the next s or fewer), with B = L_1(C, A):
//            T = B A^{-1} (scratch), then L_1(C, A) <- -C^{-1} T   (= the (C, A) block of L_1^{-1})
//   final    LinvT(j, i) = L_1^{-1}(i, j), zero above the diagonal and in the padding
// GEMM tiles are 32 x 32 outputs per CTA step (256 threads, 4 outputs each, 32-deep smem
// panels), taken grid-stride; one grid barrier after each step.  Triangular factors are
// stored with exact zeros above the diagonal, so the panels need no masks.
constexpr int kTbThreads = 256;
template <typename T>
__global__ void __launch_bounds__(kTbThreads) k_trinv_blk(double* __restrict__ L1, int k, double* __restrict__ Tsc,
                                                          T* __restrict__ LinvT, int64_t ldo) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double Ps[32][33], Qs[32][33];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int64_t kk = k;
  // phase 0a: zero the strictly upper triangle (one warp per row)
  for (int64_t i = (int64_t)blockIdx.x * (kTbThreads / 32) + ty; i < kk; i += (int64_t)gridDim.x * (kTbThreads / 32))
    for (int64_t j = i + 1 + tx; j < kk; j += 32) L1[i * kk + j] = 0.0;
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
  grid.sync();
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
    }
  }
  // final: LinvT (k x ldo) = L_1^{-T}, zero above the diagonal and in the padding
  for (int64_t e = (int64_t)blockIdx.x * kTbThreads + tid; e < kk * ldo; e += (int64_t)gridDim.x * kTbThreads) {
    const int64_t j = e / ldo, i = e - j * ldo;
    LinvT[e] = (i >= j && i < kk) ? (T)L1[i * kk + j] : T(0);
  }
}

// k <= 128: L_1^{-1} in ONE CTA with L_1 resident in shared memory (padded to kp = 8 ceil(k/8)
// rows with an identity block, whose inverse is the identity), by recursive doubling: the 8 x 8
// diagonal blocks by substitution (one thread per column, in registers), then for sb = 8, 16,
// 32, 64 every pair of inverted sb-blocks A = L(a0.., a0..), C = L(c0.., c0..) (c0 = a0 + sb)
// with B = L(C, A) becomes the inverse of [[A, 0], [B, C]] by T = B A^{-1} (scratch) and
// L(C, A) = -C^{-1} T, all pairs of a level together, on the FP64 tensor path (DMMA m8n8k4):
// a warp owns 2 x 2 output tiles (one 8 x 8 tile while sb = 8), so each fragment load feeds two
// MMAs; the K loops skip the zero triangles of A^{-1} (T: k >= the first column) and C^{-1}
// (L: k <= the last row). No grid barriers and no global round trips between the levels; the
// FP64 work on one SM (kp^3 / 3 FMA) is ~3 us at k = 128.
constexpr int kT1K = 128;
constexpr int kT1Threads = 512;
constexpr int kT1Scratch = 64 * 68 + kT1K;   // level scratch (max np sb (sb + 4)) + reciprocals
__host__ __device__ constexpr size_t trinv_one_smem(int k) {
  return ((size_t)((k + 7) & ~7) * (((k + 7) & ~7) + 4) + kT1Scratch) * sizeof(double);
}
__device__ __forceinline__ void t1_dmma(double2& d, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d.x), "+d"(d.y)
      : "d"(a), "d"(b));
}
template <typename T>
__global__ void __launch_bounds__(kT1Threads, 1) k_trinv_one(const double* __restrict__ L1, int k,
                                                              T* __restrict__ LinvT, int64_t ldo) {
  extern __shared__ double t1_[];
  const int kp = (k + 7) & ~7, ld = kp + 4;   // ld = 4 mod 8: conflict-free fragment loads
  double* Ls = t1_;                           // [kp][ld]
  double* Tt = Ls + (size_t)kp * ld;          // level scratch [pair][sb][sb + 4]
  double* Dr = Tt + 64 * 68;                  // 1 / L(i, i)
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, q = lane & 3;
  constexpr int NW = kT1Threads / 32, RPW = kT1K / NW;
  {
    // warp w: rows w + 16 r, lanes over the columns; all loads in flight before the stores
    double v[RPW][4];
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int i = w + NW * r, jj = lane + 32 * t;
        v[r][t] = (i < k && jj <= i) ? L1[(int64_t)i * k + jj] : (i == jj ? 1.0 : 0.0);
      }
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int i = w + NW * r, jj = lane + 32 * t;
        if (i < kp && jj < kp) {
          Ls[i * ld + jj] = v[r][t];
          if (jj == i) Dr[i] = 1.0 / v[r][t];
        }
      }
    // LinvT's zeros (above the diagonal and the padding columns [k, ldo)); every other entry
    // is written once, when it becomes final
    for (int j = w; j < k; j += NW)
      for (int64_t i = lane; i < ldo; i += 32)
        if (i < j || i >= k) LinvT[(int64_t)j * ldo + i] = T(0);
  }
  __syncthreads();
  {
    // 8 x 8 diagonal blocks: thread 8 b + j solves L_bb x = e_j
    const int b = tid >> 3, j = tid & 7;
    double x[8];
    double* Lb = Ls + 8 * b * (ld + 1);
    if (tid < kp) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double sacc = i == j ? 1.0 : 0.0;
#pragma unroll
        for (int m = 0; m < i; ++m) sacc = fma(-Lb[i * ld + m], x[m], sacc);
        x[i] = sacc * Dr[8 * b + i];
      }
    }
    __syncthreads();
    if (tid < kp) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i >= j) {
          Lb[i * ld + j] = x[i];
          if (8 * b + i < k) LinvT[(int64_t)(8 * b + j) * ldo + 8 * b + i] = (T)x[i];
        }
    }
  }
  __syncthreads();
  for (int sb = 8; sb < kp; sb *= 2) {
    const int np = (kp - sb + 2 * sb - 1) / (2 * sb), ntc = sb / 8;
    const int bt = sb >= 16 ? 2 : 1, nub = ntc / bt;   // units of bt x bt tiles, np nub^2 <= 16
    const int tld = sb + 4;
    for (int step = 0; step < 2; ++step) {
      // the coordinate that sets a unit's K extent (T: its first tile column, L: its last tile
      // row) varies across the four warps of each SM sub-partition (w / 4), the rest (w % 4)
      const int hv = (w >> 2) % nub, v = (w & 3) + 4 * (w / (4 * nub));
      const int p = v / nub, ot = v - p * nub;
      const int trb = step == 0 ? ot : hv, tcb = step == 0 ? hv : ot;
      const int a0 = 2 * sb * p, c0 = a0 + sb, cs = min(sb, kp - c0);
      const int tr0 = bt * trb, tc0 = bt * tcb;
      const bool act = p < np && 8 * tr0 < cs;
      const bool row1 = bt == 2 && 8 * (tr0 + 1) < cs;   // second tile row inside the block
      const int rA0 = c0 + 8 * tr0 + g, rA1 = row1 ? rA0 + 8 : rA0;
      if (act) {
        double2 acc[2][2];
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y) acc[x][y] = make_double2(0.0, 0.0);
        if (step == 0) {
          // T(r, c) = sum_{m >= 8 tc0} B(r, m) A^{-1}(m, c)
          const double* a_0 = Ls + rA0 * ld + a0 + q;
          const double* a_1 = Ls + rA1 * ld + a0 + q;
          const double* b_0 = Ls + (a0 + q) * ld + a0 + 8 * tc0 + g;
          for (int s4 = 2 * tc0; s4 < sb / 4; ++s4) {
            const double x0 = a_0[4 * s4], y0 = b_0[4 * s4 * ld];
            t1_dmma(acc[0][0], x0, y0);
            if (bt == 2) {
              const double x1 = a_1[4 * s4], y1 = b_0[4 * s4 * ld + 8];
              t1_dmma(acc[0][1], x0, y1);
              t1_dmma(acc[1][0], x1, y0);
              t1_dmma(acc[1][1], x1, y1);
            }
          }
          double* o = Tt + (size_t)p * sb * tld + (8 * tr0 + g) * tld + 8 * tc0 + 2 * q;
          *reinterpret_cast<double2*>(o) = acc[0][0];
          if (bt == 2) {
            *reinterpret_cast<double2*>(o + 8) = acc[0][1];
            if (row1) {
              *reinterpret_cast<double2*>(o + 8 * tld) = acc[1][0];
              *reinterpret_cast<double2*>(o + 8 * tld + 8) = acc[1][1];
            }
          }
        } else {
          // L(C, A)(r, c) = -sum_{m < 8 (tr0 + bt)} C^{-1}(r, m) T(m, c)
          const double* a_0 = Ls + rA0 * ld + c0 + q;
          const double* a_1 = Ls + rA1 * ld + c0 + q;
          const double* b_0 = Tt + (size_t)p * sb * tld + q * tld + 8 * tc0 + g;
          const int kend = min(cs, 8 * (tr0 + bt)) / 4;
          for (int s4 = 0; s4 < kend; ++s4) {
            const double x0 = a_0[4 * s4], y0 = b_0[4 * s4 * tld];
            t1_dmma(acc[0][0], x0, y0);
            if (bt == 2) {
              const double x1 = a_1[4 * s4], y1 = b_0[4 * s4 * tld + 8];
              t1_dmma(acc[0][1], x0, y1);
              t1_dmma(acc[1][0], x1, y0);
              t1_dmma(acc[1][1], x1, y1);
            }
          }
          // these entries of L_1^{-1} are final: also straight to LinvT (8 consecutive i per
          // store group), overlapping the later levels
#pragma unroll
          for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y) {
              if ((x == 1 || y == 1) && bt == 1) continue;
              if (x == 1 && !row1) continue;
              const double2 r = make_double2(-acc[x][y].x, -acc[x][y].y);
              const int i = rA0 + 8 * x, j = a0 + 8 * (tc0 + y) + 2 * q;
              *reinterpret_cast<double2*>(Ls + i * ld + j) = r;
              if (i < k) {
                LinvT[(int64_t)j * ldo + i] = (T)r.x;
                LinvT[(int64_t)(j + 1) * ldo + i] = (T)r.y;
              }
            }
        }
      }
      __syncthreads();
    }
  }
}

template <typename T>
cudaError_t launch_trinv(const double* L1, int64_t k, T* LinvT, int64_t ldo, DevState* st, cudaStream_t s,
                         void* scratch) {
  if (k <= 0) return cudaSuccess;
  if (k > 32 && k <= kT1K && !getenv("RBRP_TRINV_SUBST") && !getenv("RBRP_TRINV_GRID")) {
    const size_t smem = trinv_one_smem((int)k);
    static PerDevice attr1;
    const cudaError_t ae = attr1.once([] {
      const size_t mx = trinv_one_smem(kT1K);
      cudaError_t r = cudaFuncSetAttribute(k_trinv_one<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
      if (r == cudaSuccess)
        r = cudaFuncSetAttribute(k_trinv_one<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
      return r;
    });
    if (ae != cudaSuccess) return ae;
    k_trinv_one<T><<<1, kT1Threads, smem, s>>>(L1, (int)k, LinvT, ldo);
    return cudaGetLastError();
  }
  if (scratch && k > 32 && !getenv("RBRP_TRINV_SUBST")) {
    // blocked cooperative inversion (L1 is overwritten by L_1^{-1}; scratch >= k^2 / 2 doubles)
    int maxit = (int)((k + 31) / 32);
    for (int64_t sb = 32; sb < k; sb *= 2) {
      int items = 0;
      for (int64_t a0 = 0; a0 + sb < k; a0 += 2 * sb) items += (int)(((std::min<int64_t>(sb, k - a0 - sb) + 31) / 32) * (sb / 32));
      maxit = std::max(maxit, items);
    }
    int per = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_trinv_blk<T>, kTbThreads, 0);
    if (e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(maxit, device_sms() * std::max(per, 1)));
    double* L1w = const_cast<double*>(L1);
    double* Tsc = (double*)scratch;
    int ki = (int)k;
    void* args[] = {&L1w, &ki, &Tsc, &LinvT, &ldo};
    e = cudaLaunchCooperativeKernel((const void*)k_trinv_blk<T>, dim3(grid), dim3(kTbThreads), args, 0, s);
    return e;
  }
  if (k <= kTrinvSmallK) {
    const size_t smem = (size_t)(k * k + k + kTrinvSmallWarps * k) * sizeof(double);
    static PerDevice attr;   // once per device, for the largest k of this path
    const cudaError_t ae = attr.once([] {
      const size_t mx = (size_t)(kTrinvSmallK * kTrinvSmallK + kTrinvSmallK + kTrinvSmallWarps * kTrinvSmallK) * 8;
      return cudaFuncSetAttribute(k_trinv_small<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    });
    if (ae != cudaSuccess) return ae;
    k_trinv_small<T><<<ceil_div(k, kTrinvSmallWarps), 32 * kTrinvSmallWarps, smem, s>>>(L1, k, LinvT, ldo, st);
    return cudaGetLastError();
  }
  size_t smem = (size_t)kTrinvWarps * k * sizeof(double);
  cudaFuncSetAttribute(k_trinv<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_trinv<T><<<ceil_div(k, kTrinvWarps), 32 * kTrinvWarps, smem, s>>>(L1, k, LinvT, ldo, st);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------
// Remark 5.2: clipped pseudo-inverse of L_1 (k x k, row-major fp64)
// ---------------------------------------------------------------------------------

// The Remark 5.2 trigger for a standalone L_1: out[0] = min |L_1(i,i)|, out[1] = max.
__global__ void k_diag_test(const double* __restrict__ L1, int64_t k, double* __restrict__ out) {
  double mx = 0.0, mn = DBL_MAX;
  for (int64_t i = threadIdx.x; i < k; i += 32) {
    const double a = fabs(L1[i * k + i]);
    mx = fmax(mx, a);
    mn = fmin(mn, a);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  if (threadIdx.x == 0) {
    out[0] = mn;
    out[1] = mx;
  }
}

cudaError_t launch_diag_test(const double* L1, int64_t k, double* out, cudaStream_t s) {
  if (k <= 0) return cudaSuccess;
  k_diag_test<<<1, 32, 0, s>>>(L1, k, out);
  return cudaGetLastError();
}

constexpr int kJacWarps = 8;
constexpr int kJacMaxSweeps = 40;

// round-robin (circle method) position -> column: position 0 fixed, the others rotate
__device__ __forceinline__ int jac_col(int pos, int round, int m) {
  return pos == 0 ? 0 : 1 + (pos - 1 + round) % (m - 1);
}

// One-sided Jacobi SVD of A (columns G[j*k .. +k), j < k; A = L_1^T, so column j of A is
// row j of the row-major L_1 buffer, rotated in place): A V = U Sigma.  Every round
// rotates m/2 disjoint column pairs (one warp each) so that the pair is orthogonal;
// m - 1 rounds make a sweep; sweeps repeat until a sweep rotates nothing (|gamma| <=
// 1e-15 sqrt(alpha beta) for every pair) or kJacMaxSweeps.  V (same layout) starts as I.
// cnt[0..1]: rotation counters of the even/odd sweep (zeroed by the launcher).
__global__ void __launch_bounds__(32 * kJacWarps) k_jacobi_svd(double* __restrict__ G, double* __restrict__ V,
                                                               int k, unsigned* cnt) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kJacWarps + (threadIdx.x >> 5), nw = gridDim.x * kJacWarps;
  const int m = k + (k & 1);   // a phantom zero column when k is odd
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)k * k; e += (int64_t)gridDim.x * blockDim.x)
    V[e] = (e / k == e % k) ? 1.0 : 0.0;
  grid.sync();
  for (int sweep = 0; sweep < kJacMaxSweeps; ++sweep) {
    unsigned* c = cnt + (sweep & 1);
    for (int round = 0; round < m - 1; ++round) {
      for (int pr = gw; pr < m / 2; pr += nw) {
        int p = jac_col(pr, round, m), q = jac_col(m - 1 - pr, round, m);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        if (q >= k) continue;   // phantom column
        double* gp = G + (int64_t)p * k;
        double* gq = G + (int64_t)q * k;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int r = lane; r < k; r += 32) {
          const double a = gp[r], b = gq[r];
          al = fma(a, a, al);
          be = fma(b, b, be);
          ga = fma(a, b, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (!(fabs(ga) > 1e-15 * sqrt(al) * sqrt(be))) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int r = lane; r < k; r += 32) {
          const double a = gp[r], b = gq[r];
          gp[r] = cs * a - sn * b;
          gq[r] = sn * a + cs * b;
        }
        double* vp = V + (int64_t)p * k;
        double* vq = V + (int64_t)q * k;
        for (int r = lane; r < k; r += 32) {
          const double a = vp[r], b = vq[r];
          vp[r] = cs * a - sn * b;
          vq[r] = sn * a + cs * b;
        }
        if (lane == 0) atomicAdd(c, 1u);
      }
      grid.sync();
    }
    const unsigned rot = *(volatile unsigned*)c;
    grid.sync();   // everyone has read c before it is reset for sweep + 2
    if (blockIdx.x == 0 && threadIdx.x == 0) *c = 0u;
    if (rot == 0) break;
  }
}

// w[l] = sigma_l^-2 if sigma_l >= 1e-12 sigma_max else 0 (sigma_l = ||G_l||); V_l *= w[l]
// in place; nclip = number of discarded singular values.  One CTA.
__global__ void k_pinv_weights(const double* __restrict__ G, double* __restrict__ V, int k, int* nclip) {
  extern __shared__ double sg[];   // [k]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int l = w; l < k; l += nwarp) {
    double s = 0.0;
    for (int r = lane; r < k; r += 32) s = fma(G[(int64_t)l * k + r], G[(int64_t)l * k + r], s);
    s = warp_sum(s);
    if (lane == 0) sg[l] = sqrt(s);
  }
  __syncthreads();
  __shared__ double smax;
  __shared__ int ncl;
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int l = 0; l < k; ++l) mx = fmax(mx, sg[l]);
    smax = mx;
    ncl = 0;
  }
  __syncthreads();
  for (int l = w; l < k; l += nwarp) {
    const double sl = sg[l];
    const bool keep = sl >= 1e-12 * smax && sl > 0.0;
    const double wl = keep ? 1.0 / (sl * sl) : 0.0;
    for (int r = lane; r < k; r += 32) V[(int64_t)l * k + r] *= wl;
    if (lane == 0 && !keep) atomicAdd(&ncl, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0 && nclip) *nclip = ncl;
}

// out(j, m) = sum_l Vw[l][j] G[l][m]  (= pinv_clip(L_1)^T), out k x ldo, columns [k, ldo) 0.
// 32 x 32 output tile per CTA, l in chunks of 32 through shared memory.
template <typename T>
__global__ void __launch_bounds__(256) k_pinv_form(const double* __restrict__ Vw, const double* __restrict__ G, int k,
                                                   T* __restrict__ out, int64_t ldo) {
  __shared__ double As[32][33], Bs[32][33];
  const int j0 = blockIdx.y * 32, m0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // ty 0..7: rows ty, ty+8, ...
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int l0 = 0; l0 < k; l0 += 32) {
    for (int u = ty; u < 32; u += 8) {
      const int l = l0 + u;
      As[u][tx] = (l < k && j0 + tx < k) ? Vw[(int64_t)l * k + j0 + tx] : 0.0;
      Bs[u][tx] = (l < k && m0 + tx < k) ? G[(int64_t)l * k + m0 + tx] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int u = 0; u < 32; ++u) {
      const double b = Bs[u][tx];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = fma(As[u][ty + 8 * i], b, acc[i]);
    }
    __syncthreads();
  }
  for (int i = 0; i < 4; ++i) {
    const int j = j0 + ty + 8 * i, m = m0 + tx;
    if (j < k && m < ldo) out[(int64_t)j * ldo + m] = m < k ? (T)acc[i] : T(0);
  }
}

size_t pinv_scratch_bytes(int64_t k) { return ((size_t)k * k * 8 + 255) / 256 * 256 + 256; }

// LinvT (k x ldo) = pinv_clip(L_1)^T.  L1 (k x k row-major fp64) is overwritten by the
// rotated columns A V; scratch >= pinv_scratch_bytes(k).  nclip (device, optional):
// number of discarded singular values.
template <typename T>
cudaError_t launch_pinv_clip(double* L1, int64_t k, T* LinvT, int64_t ldo, void* scratch, int* nclip,
                             cudaStream_t s) {
  if (k <= 0) return cudaSuccess;
  double* V = (double*)scratch;
  unsigned* cnt = (unsigned*)((char*)scratch + ((size_t)k * k * 8 + 255) / 256 * 256);
  cudaError_t e = cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi_svd, 32 * kJacWarps, 0);
  if (e != cudaSuccess) return e;
  const int pairs = (int)((k + 1) / 2);
  int grid = ceil_div(pairs, kJacWarps);
  grid = std::max(1, std::min(grid, std::max(1, per_sm) * device_sms()));
  int kk = (int)k;
  void* args[] = {(void*)&L1, (void*)&V, (void*)&kk, (void*)&cnt};
  e = cudaLaunchCooperativeKernel((const void*)k_jacobi_svd, dim3(grid), dim3(32 * kJacWarps), args, 0, s);
  if (e != cudaSuccess) return e;
  const size_t wsm = (size_t)k * 8;
  if (wsm > 48 * 1024) {
    e = cudaFuncSetAttribute(k_pinv_weights, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm);
    if (e != cudaSuccess) return e;
  }
  k_pinv_weights<<<1, 1024, wsm, s>>>(L1, V, kk, nclip);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 g2((unsigned)ceil_div(ldo, 32), (unsigned)ceil_div(k, 32));
  k_pinv_form<T><<<g2, 256, 0, s>>>(V, L1, kk, LinvT, ldo);
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

// W = L L_1^{-T} for small K = kp <= kWsK (Alg. 3): L_1^{-T} (kp x kp, fp64) stays
// in shared memory for the whole launch, 64-row tiles of L stream through (converted to fp64,
// prefetched into registers during the previous tile's MMAs), and the product runs on the FP64
// tensor path (DMMA m8n8k4): 16 warps, warp w owns the tile's rows 8 (w & 7) .. + 7 and one half
// of the groups of four 8-column output tiles (four independent accumulator chains, one A
// fragment per k-step shared by the four).  Output tile t (columns 8t ..) skips the k-steps with k < 8t, where
// L_1^{-T}(n, k) = 0 (L_1^{-1} is lower triangular).  One pass over L, one write of W.
constexpr int kWsK = 128;
constexpr int kWsRows = 64;
constexpr int kWsThreads = 512;
__device__ __forceinline__ void ws_dmma(double2& d, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d.x), "+d"(d.y)
      : "d"(a), "d"(b));
}
template <typename T>
__global__ void __launch_bounds__(kWsThreads, 1)
    k_w_small(const T* __restrict__ L, int64_t ldl, const T* __restrict__ LinvT, int64_t n, int k, int kp,
              T* __restrict__ W, int64_t ldw, int lower) {
  extern __shared__ double ws_[];
  const int ld = kp + 4;                         // conflict-free fragment loads (ld = 4 mod 8)
  double* Bs = ws_;                              // [kp][ld]: Bs[nn][kk] = L_1^{-T}(nn, kk)
  double* As = Bs + (size_t)kp * ld;             // [64][ld]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, q = lane & 3;
  // warp w: row group rg = w & 7 (8 rows of the tile), column half ch = w >> 3 of the groups of
  // four 8-column output tiles, paired from both ends (0 with the last, 1 with the one before,
  // ...) so that both halves carry the same triangular work
  const int rg = w & 7, ch = w >> 3;
  for (int e = tid; e < kp * kp; e += kWsThreads) {
    const int nn = e / kp, kk = e - nn * kp;
    Bs[nn * ld + kk] = (double)LinvT[(int64_t)nn * kp + kk];
  }
  const int64_t ntiles = (n + kWsRows - 1) / kWsRows;
  constexpr int PF = kWsRows * kWsK / kWsThreads;   // prefetched elements per thread (16)
  T pf[PF];
  auto fetch = [&](int64_t tile) {
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int e = tid + u * kWsThreads, r = e / kWsK, c = e - r * kWsK;
      const int64_t row = tile * kWsRows + r;
      pf[u] = (c < k && row < n) ? L[row * ldl + c] : T(0);   // L's columns [k, kp) read as zeros
    }
  };
  int64_t tile = blockIdx.x;
  if (tile < ntiles) fetch(tile);
  const int ntt = kp / 8, ngr = (ntt + 3) / 4, nk4 = kp / 4;
  for (; tile < ntiles; tile += gridDim.x) {
    __syncthreads();   // previous tile's MMAs done with As (and Bs complete, first time)
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int e = tid + u * kWsThreads, r = e / kWsK, c = e - r * kWsK;
      if (c < kp) As[r * ld + c] = (double)pf[u];
    }
    __syncthreads();
    if (tile + gridDim.x < ntiles) fetch(tile + gridDim.x);   // in flight during the MMAs
    const double* Ar = As + (8 * rg + g) * ld + q;
    const int64_t row = tile * kWsRows + 8 * rg + g;
    for (int grp = 0; grp < ngr; ++grp) {
      // half 0 takes the groups 0, 3, 4, 7, ... and half 1 the groups 1, 2, 5, 6, ...: with the
      // triangular k ranges shrinking by 8 per group, both halves get the same work
      const int m4 = grp & 3;
      if ((m4 == 0 || m4 == 3) != (ch == 0)) continue;
      const int t0 = 4 * grp;
      double2 acc[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0),
                        make_double2(0.0, 0.0)};
      const double* B0 = Bs + (8 * t0 + g) * ld + q;
      const int nj = min(4, ntt - t0);
      int s4 = lower ? 2 * t0 : 0;   // k-steps of 4 below 8 t0 hold only zeros of B
      // diagonal band (lower): tile t0 + j starts at k-step 2 (t0 + j)
      const int sfull = lower ? min(nk4, 2 * t0 + 6) : s4;
      for (; s4 < sfull; ++s4) {
        const double a = Ar[4 * s4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < nj && s4 >= 2 * (t0 + j)) ws_dmma(acc[j], a, B0[8 * j * ld + 4 * s4]);
      }
      if (nj == 4) {
#pragma unroll 2
        for (; s4 < nk4; ++s4) {
          const double a = Ar[4 * s4];
          const double b0 = B0[4 * s4], b1 = B0[8 * ld + 4 * s4], b2 = B0[16 * ld + 4 * s4], b3 = B0[24 * ld + 4 * s4];
          ws_dmma(acc[0], a, b0);
          ws_dmma(acc[1], a, b1);
          ws_dmma(acc[2], a, b2);
          ws_dmma(acc[3], a, b3);
        }
      } else {
        for (; s4 < nk4; ++s4) {
          const double a = Ar[4 * s4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < nj) ws_dmma(acc[j], a, B0[8 * j * ld + 4 * s4]);
        }
      }
      if (row < n) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int col = 8 * (t0 + j) + 2 * q;
          if (j < nj) {
            if (col < k) W[row * ldw + col] = (T)acc[j].x;
            if (col + 1 < k) W[row * ldw + col + 1] = (T)acc[j].y;
          }
        }
      }
    }
  }
}

template <typename T>
bool w_small_supported(int64_t kp) { return kp % 8 == 0 && kp >= 8 && kp <= kWsK; }

template <typename T>
cudaError_t launch_w_small(const T* L, int64_t ldl, const T* LinvT, int64_t n, int64_t k, int64_t kp, T* W,
                           int64_t ldw, bool lower, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (!w_small_supported<T>(kp)) return cudaErrorInvalidValue;
  const size_t smem = (size_t)(kp + kWsRows) * (kp + 4) * sizeof(double);
  static PerDevice attr;
  const cudaError_t ae = attr.once([] {
    return cudaFuncSetAttribute(k_w_small<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)((size_t)(kWsK + kWsRows) * (kWsK + 4) * sizeof(double)));
  });
  if (ae != cudaSuccess) return ae;
  const int64_t ntiles = (n + kWsRows - 1) / kWsRows;
  const int grid = (int)std::min<int64_t>(ntiles, device_sms());
  k_w_small<T><<<grid, kWsThreads, smem, s>>>(L, ldl, LinvT, n, (int)k, (int)kp, W, ldw, lower ? 1 : 0);
  return cudaGetLastError();
}

#define INSTW(T)                                                                                  \
  template cudaError_t launch_gather_L1<T>(const T*, int64_t, const int64_t*, int64_t, int64_t,  \
                                           int64_t, double*, cudaStream_t);                      \
  template cudaError_t launch_trinv<T>(const double*, int64_t, T*, int64_t, DevState*, cudaStream_t, void*); \
  template cudaError_t launch_w_identity<T>(T*, int64_t, const int64_t*, int64_t, int64_t,       \
                                            int64_t, cudaStream_t);                              \
  template cudaError_t launch_pinv_clip<T>(double*, int64_t, T*, int64_t, void*, int*, cudaStream_t); \
  template bool w_small_supported<T>(int64_t);                                                   \
  template cudaError_t launch_w_small<T>(const T*, int64_t, const T*, int64_t, int64_t, int64_t, T*, int64_t, \
                                         bool, cudaStream_t);
INSTW(double)
INSTW(float)

}  // namespace rbrp
