// k_filter_coop.cu — a3 in ONE cooperative kernel: gather + local pivoted QR + robust
// filter + CholQR2 basis (Alg. 2 l.6-9; Remark 4.1).
//
// Grid = ceil(d / 32) CTAs; CTA c owns columns [32c, 32c+32) of V = X_res(S_t,:)^T and of
// every basis built from it, kept in shared memory for the whole kernel.
//   A  gather V(:, cols) (fp64) and its partial Gram                    -> Gpart[c]
//   B  G = sum_c Gpart[c] in a fixed order (element slices)              -> G
//   C  every CTA (redundantly, bit-identical, so nothing is broadcast): right-looking
//      pivoted Cholesky of G with logical pivoting.  The Schur diagonal is the
//      Householder CPQR residual column norm^2 (reading R10), so mass[i] =
//      ||R_V(i:b,i:b)||_F^2 and b' = max{i : mass[i] >= tau_b mass[0]} (l.8);
//      pivot = max, ties -> lowest draw position (R9).  Then T11 = R11^{-1}.
//   D  Q1(:, cols) = V(:, pi(1:b')) T11 (parallel dot products); partial Gram of Q1
//   E  G2 = sum_c Gpart[c]
//   F  every CTA: Cholesky G2 = R2^T R2 (CholQR2) with T2 = R2^{-1}; CTA 0: R_total = R2 R11
//   G  Q_b(:, cols) = Q1 T2 -> Qt (rows >= b' zero up to bp_pad)
// Four grid-wide barriers.
#include <atomic>
#include <cooperative_groups.h>
#include <float.h>

#include "launch.cuh"

namespace cg = cooperative_groups;

namespace rbrp {

constexpr int kFiltThreads = 256;
constexpr int kFiltCW = 32;         // columns per CTA
constexpr int kFiltLd = kFiltCW + 1;
constexpr int kSmallNb = 64;        // nb <= 64: G, R, T, R11 all in shared memory

// Right-looking pivoted (mode 1) or plain (mode 2) Cholesky of the symmetric nb x nb
// matrix A (shared memory, stride lda, destroyed), all threads of the CTA, logical
// pivoting (no row/column swaps):
//   step i: p = argmax of the unchosen Schur diagonal dg (ties -> lowest original index,
//   reading R9; mode 2: p = i; replay: forced[i]); R(i, l) = A(p, l) / sqrt(dg(p)) for
//   the unchosen l; A(r, c) -= R(i, r) R(i, c) on the unchosen block.
// dg is the Householder CPQR residual column norm^2 (reading R10), so in mode 1
// mass[i] = sum of the unchosen dg before step i = ||R_V(i:b,i:b)||_F^2 and the loop
// stops at the first i with mass[i] < tau_b mass[0] (l.8; the masses are
// non-increasing), or at a non-positive pivot (numerical rank).  R: row = step, column =
// original index (ldr).  Returns the number of kept steps.
__device__ int cta_pivchol(double* A, int lda, int nb, int mode, const int32_t* forced, double tau_b,
                           double* R, int ldr, int* perm, double* mass, double* dg, int* chosen,
                           int* rank_def) {
  __shared__ int s_p, s_cut;
  __shared__ double s_thr;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int l = tid; l < nb; l += blockDim.x) {
    dg[l] = A[l * lda + l];
    chosen[l] = 0;
  }
  if (tid == 0) *rank_def = 0;
  __syncthreads();
  int kept = nb;
  for (int i = 0; i < nb; ++i) {
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
      if (lane == 0) {
        int cut = 0;
        if (mode == 1) {
          mass[i] = ms;
          if (i == 0) s_thr = tau_b * ms;
          if (!(ms > 0.0) || ms < s_thr) cut = 1;                  // l.8 cut
        }
        int p = bl;
        if (mode == 2) p = i;
        if (mode == 1 && forced) p = forced[i];
        if (!cut && !(dg[p] > 0.0)) cut = 2;                      // non-positive pivot
        s_p = p;
        s_cut = cut;
        if (!cut) perm[i] = p;
      }
    }
    __syncthreads();
    if (s_cut) {
      if (tid == 0 && s_cut == 2) *rank_def = 1;
      kept = i;
      break;
    }
    const int p = s_p;
    const double rii = sqrt(dg[p]);
    for (int l = tid; l < nb; l += blockDim.x) {
      double v;
      if (l == p) v = rii;
      else if (chosen[l]) v = 0.0;
      else v = A[p * lda + l] / rii;
      R[i * ldr + l] = v;
    }
    __syncthreads();
    if (tid == 0) chosen[p] = 1;
    for (int e = tid; e < nb * nb; e += blockDim.x) {
      const int r = e / nb, c = e % nb;
      if (r == p || c == p) continue;
      const double rr = R[i * ldr + r], rc = R[i * ldr + c];
      if (rr == 0.0 && rc == 0.0) continue;   // chosen rows/columns carry zeros
      const double a = fma(-rr, rc, A[r * lda + c]);
      A[r * lda + c] = a;
      if (r == c) dg[r] = a;
    }
    __syncthreads();
  }
  __syncthreads();
  return kept;
}

// Fast path for nb <= 64: pivoted (mode 1) or plain (mode 2) Cholesky AND T = R11^{-1},
// right-looking, logical pivoting, each thread owning EPT fixed elements (r, c) of
//   A(r, c)    the Schur complement (in registers), and
//   acc(j, l)  sum_{q < i} T(j, q) R(q, l)  (in registers),
// so that at step i with pivot p:  R(i, l) = A(p, l) / sqrt(A(p,p)) by the owners of row
// p, T(j, i) = -acc(j, p) / R(i, p) (j < i) by the owners of column p, then the rank-1
// update A -= R(i,.)^T R(i,.) and acc(j, .) += T(j, i) R(i, .).  Every warp finds the
// pivot itself from its register copy of the Schur diagonal (identical, deterministic),
// so a step costs one barrier.  Pivot / mass / cut rules as cta_pivchol.  R: [step][orig] (ld), T:
// [step][step] (ldt).
template <int EPT>
__device__ int cta_chol_inv(const double* __restrict__ Gg, int nb, int mode, const int32_t* forced,
                            double tau_b, double* R, int ld, double* Tm, int ldt, int* perm,
                            double* mass, double* dg, int* chosen_unused, int* rank_def) {
  const int tid = threadIdx.x, lane = tid & 31;
  __builtin_assume(__isShared(R));    // both in shared memory at every call site
  __builtin_assume(__isShared(Tm));
  // element map (blockDim = kFiltThreads): thread t owns column c = t % NBX of rows
  // t / NBX + (256 / NBX) k, NBX = 32 (EPT 4) or 64 (EPT 16); a warp shares its rows (the
  // row loads are broadcasts) and a thread its column (R(i, c) loaded once per step)
  constexpr int NBX = EPT == 4 ? 32 : 64, RSTEP = kFiltThreads / NBX;
  static_assert(NBX * NBX == EPT * kFiltThreads, "element map");
  const int ec0 = tid % NBX;
  double a[EPT], ta[EPT];
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int r = tid / NBX + RSTEP * k;
    a[k] = (r < nb && ec0 < nb) ? Gg[r * kMaxB + ec0] : 0.0;
    if (r == ec0 && r < nb) dg[r] = a[k];
    ta[k] = 0.0;
  }
  for (int e = tid; e < nb * ldt; e += blockDim.x) Tm[e] = 0.0;
  if (tid == 0) *rank_def = 0;
  __syncthreads();
  // the Schur-complement diagonal, in registers of every warp (entries lane, lane + 32):
  // updated redundantly with the same fma as the matrix entry it mirrors, so the pivot
  // search needs no barrier after the update -- one __syncthreads per step
  double dg0 = lane < nb ? dg[lane] : 0.0, dg1 = lane + 32 < nb ? dg[lane + 32] : 0.0;
  unsigned long long chosen = 0ull;   // identical in every thread
  double thr = 0.0;
  int kept = nb;
  for (int i = 0; i < nb; ++i) {
    // every warp: residual mass (fixed order) and pivot (max, ties -> lowest index)
    double ms = 0.0, best = -DBL_MAX;
    int bl = 1 << 30;
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int l = lane + 32 * m;
      if (l < nb && !((chosen >> l) & 1ull)) {
        const double x = m ? dg1 : dg0;
        ms += fmax(x, 0.0);
        if (x > best) { best = x; bl = l; }
      }
    }
    int p;
    double dp;
    if (mode == 1 && !forced) {
      // pivot search as three warp REDUX ops: a positive double orders as its bit pattern,
      // so max of the high words, then max of the low words among those leaders, then the
      // lowest index holding exactly that value (ties -> lowest index, as a butterfly of
      // (value, index) pairs would give).  A non-positive best maps to key 0: that pivot is
      // cut below whichever index is returned.
      const unsigned long long key = best > 0.0 ? (unsigned long long)__double_as_longlong(best) : 0ull;
      const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      p = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bl : (1 << 30));
      dp = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    } else {
      p = mode == 2 ? i : forced[i];
      const double dq0 = __shfl_sync(0xffffffffu, dg0, p & 31), dq1 = __shfl_sync(0xffffffffu, dg1, p & 31);
      dp = p < 32 ? dq0 : dq1;
    }
    int cut = 0;
    if (mode == 1) {
      ms = warp_sum(ms);   // fixed butterfly order
      if (i == 0) thr = tau_b * ms;
      if (!(ms > 0.0) || ms < thr) cut = 1;                         // l.8 cut
    }
    if (!cut && !(dp > 0.0)) cut = 2;                               // non-positive pivot
    if (tid == 0 && mode == 1) mass[i] = ms;
    if (cut) {
      if (tid == 0 && cut == 2) *rank_def = 1;
      kept = i;
      break;
    }
    const double rii = sqrt(dp);
    const double inv = 1.0 / rii;
    if (tid == 0) {
      perm[i] = p;
      Tm[i * ldt + i] = inv;
    }
    const int c = ec0;
    {
      // only the owners write: row p of R is element k = (p - tid / NBX) / RSTEP of the
      // threads of column c (selected without indexing the register array), column p of
      // T (rows < i) belongs to the threads with c == p
      const int rp = p - tid / NBX;
      if (c < nb && rp >= 0 && rp % RSTEP == 0) {
        const int kp = rp / RSTEP;
        double av = a[0];
#pragma unroll
        for (int k = 1; k < EPT; ++k)
          if (k == kp) av = a[k];
        R[i * ld + c] = (c == p) ? rii : (((chosen >> c) & 1ull) ? 0.0 : av * inv);
      }
      if (c == p) {
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
          const int r = tid / NBX + RSTEP * k;
          if (r < i) Tm[r * ldt + i] = -ta[k] * inv;
        }
      }
    }
    chosen |= 1ull << p;
    __syncthreads();   // row i of R and column i of T complete; step i+1 writes row / column i+1
    {
      // branch-free (the loads pipeline): rows r < NBX <= ld exist in R and Tm; an inactive
      // element (r or c >= nb) only ever updates its own, never-read register, and
      // T(r, i) = 0 for r > i (zeroed above, written only for r <= i), so the r <= i
      // guard of the T update is implicit
      const double ric = R[i * ld + c];
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int r = tid / NBX + RSTEP * k;
        a[k] = fma(-R[i * ld + r], ric, a[k]);
        ta[k] = fma(Tm[r * ldt + i], ric, ta[k]);
      }
    }
    if (lane < nb) {
      const double rl = R[i * ld + lane];
      dg0 = fma(-rl, rl, dg0);
    }
    if (lane + 32 < nb) {
      const double rl = R[i * ld + lane + 32];
      dg1 = fma(-rl, rl, dg1);
    }
  }
  __syncthreads();
  return kept;
}

// 64 < nb <= kMaxB = 128, blockDim = 256: cta_pivchol with the Schur complement in
// registers (thread t: column c = t & 127, rows 64 (t >> 7) .. +64) and its diagonal
// mirrored in registers of every warp (entries lane + 32 m).  The update a -= R(i,r) R(i,c)
// runs over every element: for a chosen row or column one factor is exactly zero (or the
// element is never read again), so the kept entries equal cta_pivchol's bit for bit; the
// row loads are warp-uniform broadcasts.  One barrier per step, no memory traffic.
__device__ int cta_pivchol_reg(const double* __restrict__ Gg, int nb, int mode, const int32_t* forced,
                               double tau_b, double* R, int ldr, int* perm, double* mass, int* rank_def) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int c = tid & 127, r0 = 64 * (tid >> 7);
  double a[64];
#pragma unroll
  for (int k = 0; k < 64; ++k) a[k] = (r0 + k < nb && c < nb) ? Gg[(r0 + k) * kMaxB + c] : 0.0;
  double dgv[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int l = lane + 32 * m;
    dgv[m] = l < nb ? Gg[l * kMaxB + l] : 0.0;
  }
  if (tid == 0) *rank_def = 0;
  unsigned long long ch0 = 0ull, ch1 = 0ull;   // chosen columns (identical in every thread)
  auto chosen = [&](int l) { return ((l < 64 ? ch0 >> l : ch1 >> (l - 64)) & 1ull) != 0ull; };
  double thr = 0.0;
  int kept = nb;
  for (int i = 0; i < nb; ++i) {
    double ms = 0.0, best = -DBL_MAX;
    int bl = 1 << 30;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int l = lane + 32 * m;
      if (l < nb && !chosen(l)) {
        const double x = dgv[m];
        ms += fmax(x, 0.0);
        if (x > best) { best = x; bl = l; }
      }
    }
    int p;
    double dp;
    if (mode == 1 && !forced) {   // REDUX pivot search (as cta_chol_inv)
      const unsigned long long key = best > 0.0 ? (unsigned long long)__double_as_longlong(best) : 0ull;
      const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      p = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bl : (1 << 30));
      dp = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    } else {
      p = mode == 2 ? i : forced[i];
      const double q0 = __shfl_sync(0xffffffffu, dgv[0], p & 31), q1 = __shfl_sync(0xffffffffu, dgv[1], p & 31);
      const double q2 = __shfl_sync(0xffffffffu, dgv[2], p & 31), q3 = __shfl_sync(0xffffffffu, dgv[3], p & 31);
      const int pm = (p >> 5) & 3;
      dp = pm == 0 ? q0 : (pm == 1 ? q1 : (pm == 2 ? q2 : q3));
    }
    int cut = 0;
    if (mode == 1) {
      ms = warp_sum(ms);
      if (tid == 0) mass[i] = ms;
      if (i == 0) thr = tau_b * ms;
      if (!(ms > 0.0) || ms < thr) cut = 1;                        // l.8 cut
    }
    if (!cut && !(dp > 0.0)) cut = 2;                               // non-positive pivot
    if (cut) {
      if (tid == 0 && cut == 2) *rank_def = 1;
      kept = i;
      break;
    }
    if (tid == 0) perm[i] = p;
    const double rii = sqrt(dp);
    if ((p >> 6) == (tid >> 7)) {   // this thread holds A(p, c)
      double v = 0.0;
#pragma unroll
      for (int k = 0; k < 64; ++k)
        if (r0 + k == p) v = a[k];
      R[i * ldr + c] = c >= nb ? 0.0 : ((c == p) ? rii : (chosen(c) ? 0.0 : v / rii));
    }
    if (p < 64) ch0 |= 1ull << p;
    else ch1 |= 1ull << (p - 64);
    __syncthreads();   // row i of R complete; step i+1 writes row i+1
    const double* Ri = R + i * ldr;
    const double rc = Ri[c];
#pragma unroll
    for (int k = 0; k < 64; ++k) a[k] = fma(-Ri[r0 + k], rc, a[k]);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int l = lane + 32 * m;
      if (l < nb && l != p) {
        const double rl = Ri[l];
        if (rl != 0.0) dgv[m] = fma(-rl, rl, dgv[m]);
      }
    }
  }
  __syncthreads();
  return kept;
}

// small dense helpers on n x n shared-memory matrices (stride ld), all threads
__device__ void sm_upper_phi(const double* M, double* U, int n, int ld) {   // U = Phi(M)
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - (e / n) * n;
    U[i * ld + j] = i < j ? M[i * ld + j] : (i == j ? 0.5 * M[i * ld + j] : 0.0);
  }
}
// C = E - U^T U  (U upper)
__device__ void sm_e_minus_utu(const double* E, const double* U, double* C, int n, int ld) {
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - (e / n) * n;
    const int m = i < j ? i : j;
    double s = 0.0;
    for (int k = 0; k <= m; ++k) s = fma(U[k * ld + i], U[k * ld + j], s);
    C[i * ld + j] = E[i * ld + j] - s;
  }
}
// C = A B (A, B upper)
__device__ void sm_upper_mul(const double* A, const double* B, double* C, int n, int ld) {
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - (e / n) * n;
    double s = 0.0;
    for (int k = i; k <= j; ++k) s = fma(A[i * ld + k], B[k * ld + j], s);
    C[i * ld + j] = i <= j ? s : 0.0;
  }
}

// CholQR2 second pass for G2 = I + E with small E: R2 = I + U, U the fixed point of
// U = Phi(E - U^T U) (iterated from Phi(E)), T2 = R2^{-1} = I - U + U^2 - ...; the number
// of fixed-point steps and series terms is the smallest that leaves an error below the
// rounding of R2 and T2 (usually none and one: |E| ~ 1e-14 after the first pass).
// Parallel; used when n max|E| < 1e-4, otherwise the caller runs the exact Cholesky.  E (destroyed), R, Tm, W: n x n, stride ld; R
// doubles as scratch.  Writes R2 (upper) into R and T2 into Tm.
__device__ void cholqr2_perturb(double* E, double* R, double* Tm, double* W, int n, int ld, double eta) {
  // eta = n max|E| >= ||E||_2.  Fixed-point error after s steps ~ 2^s eta^(s+2); series
  // truncation after U^m ~ eta^(m+1): both taken below 1e-17 (rounding level of R2, T2)
  const double e2 = eta * eta, e3 = e2 * eta, e4 = e3 * eta;
  const int steps = e2 < 1e-17 ? 0 : (2 * e3 < 1e-17 ? 1 : (4 * e4 < 1e-17 ? 2 : 3));
  const int terms = e2 < 1e-17 ? 1 : (e3 < 1e-17 ? 2 : (e4 < 1e-17 ? 3 : 4));
  sm_upper_phi(E, W, n, ld);                  // U0
  __syncthreads();
  for (int it = 0; it < steps; ++it) {
    sm_e_minus_utu(E, W, R, n, ld);
    __syncthreads();
    sm_upper_phi(R, W, n, ld);                // U_{it+1}
    __syncthreads();
  }
  // T2 = I - U + U^2 - ... (-U)^terms, Horner: P <- I - U P
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - (e / n) * n;
    Tm[i * ld + j] = (i == j ? 1.0 : 0.0) - W[i * ld + j];
  }
  for (int t = 2; t <= terms; ++t) {
    __syncthreads();
    sm_upper_mul(W, Tm, E, n, ld);            // U P (E is free now)
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = e / n, j = e - (e / n) * n;
      Tm[i * ld + j] = (i == j ? 1.0 : 0.0) - E[i * ld + j];
    }
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e - (e / n) * n;
    R[i * ld + j] = (i == j ? 1.0 : 0.0) + W[i * ld + j];
  }
  __syncthreads();
}

// T = R11^{-1} (bp <= 128), one warp per column c of T: back substitution in column form,
// R11 x = e_c from q = c down to 0, x_q = (delta_qc - s_q) / R11(q,q) by its owner lane
// (rows lane + 32 m in registers), broadcast by one shuffle, then s_j += R11(j,q) x_q for
// j < q.  R11(j, q) = R(j, perm[q]) in shared memory; T written once per column.
__device__ void cta_trinv_warp(const double* R, int ldr, const int* perm, int bp, double* Tm, int ldt) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ double rinv[kMaxB];   // 1 / R11(q, q), off the dependent chain
  for (int q = threadIdx.x; q < bp; q += blockDim.x) rinv[q] = 1.0 / R[q * ldr + perm[q]];
  __syncthreads();
  for (int c = w; c < bp; c += nw) {
    double sacc[4] = {0.0, 0.0, 0.0, 0.0}, xr[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = c; q >= 0; --q) {
      const int pq = perm[q], mq = q >> 5;
      double xq = 0.0;
      if (lane == (q & 31)) {
        double sq = sacc[0];
#pragma unroll
        for (int m = 1; m < 4; ++m)
          if (m == mq) sq = sacc[m];
        xq = ((q == c ? 1.0 : 0.0) - sq) * rinv[q];
#pragma unroll
        for (int m = 0; m < 4; ++m)
          if (m == mq) xr[m] = xq;
      }
      xq = __shfl_sync(0xffffffffu, xq, q & 31);
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int j = lane + 32 * m;
        if (j < q) sacc[m] = fma(R[j * ldr + pq], xq, sacc[m]);
      }
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int j = lane + 32 * m;
      if (j < bp) Tm[j * ldt + c] = j <= c ? xr[m] : 0.0;
    }
  }
  __syncthreads();
}

// partial Gram of the nb x 32 slice S (stride kFiltLd) -> out (kMaxB x kMaxB)
// partial Gram of this CTA's 32 columns: out(i, j) = sum_c S(i, c) S(j, c), i, j < nb, in
// 4 x 4 register tiles (8 shared loads per 16 fmas, 16 independent chains per thread)
__device__ void slice_gram(const double* S, int nb, double* out, int ldo = kMaxB) {
  const int nt = (nb + 3) >> 2;   // 4-row tiles per side
  for (int t = threadIdx.x; t < nt * nt; t += blockDim.x) {
    const int ti = t / nt, tj = t - ti * nt;
    const int i0 = 4 * ti, j0 = 4 * tj;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
#pragma unroll 4
    for (int c = 0; c < kFiltCW; ++c) {
      double x[4], y[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {   // rows past nb (< kMaxB) feed only unwritten outputs
        x[a] = S[(i0 + a) * kFiltLd + c];
        y[a] = S[(j0 + a) * kFiltLd + c];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(x[a], y[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (i0 + a < nb && j0 + b < nb) out[(i0 + a) * ldo + j0 + b] = acc[a][b];
  }
}
__device__ void reduce_slices(const double* Gpart, int nsplit, int nb, double* G) {
  const int64_t per = (int64_t)nb * nb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < per;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / nb), j = (int)(e % nb);
    const double* src = Gpart + i * kMaxB + j;
    double s = 0.0;
    int q = 0;
    for (; q + 8 <= nsplit; q += 8) {   // 8 independent loads in flight, summed in order
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = src[(int64_t)(q + u) * kMaxB * kMaxB];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += x[u];
    }
    for (; q < nsplit; ++q) s += src[(int64_t)q * kMaxB * kMaxB];
    G[i * kMaxB + j] = s;
  }
}

// cluster mode, nb <= 32: every CTA sums the nsplit partial Grams (nb x nb, stride 32, in
// the shared memory of the cluster's CTAs, read over DSMEM) in rank order -- the order of
// reduce_slices -- into its own copy G (stride kMaxB); no second barrier
__device__ void reduce_dsmem(double* part, int nsplit, int nb, double* G) {
  cg::cluster_group cl = cg::this_cluster();
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e - (e / nb) * nb;
    double x[8];
    double s = 0.0;
    int q = 0;
    for (; q + 8 <= nsplit; q += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = cl.map_shared_rank(part, q + u)[i * 32 + j];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += x[u];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = q + u < nsplit ? cl.map_shared_rank(part, q + u)[i * 32 + j] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (q + u < nsplit) s += x[u];
    G[i * kMaxB + j] = s;
  }
}

// Out(i, c) = sum_{j <= i} T(j, i) In(src(j), c), i < rows (parallel dot products)
__device__ void apply_T(const double* Tm, int ldt, int rows, const double* In, const int* src,
                        double* Out) {
  // Out(i, c) = sum_{j <= i} T(j, i) In(src(j), c): thread (ty, tx) = column tx of the rows
  // ty + 8u of a 64-row half, eight independent chains; T(j, i) is a warp-wide broadcast
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // blockDim = kFiltThreads = 256
  for (int base = 0; base < rows; base += 64) {
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    const int jmax = min(rows, base + 64);
    for (int j = 0; j < jmax; ++j) {
      const double x = In[(src ? src[j] : j) * kFiltLd + tx];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + ty + 8 * u;
        if (i < rows && j <= i) acc[u] = fma(Tm[j * ldt + i], x, acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + ty + 8 * u;
      if (i < rows) Out[i * kFiltLd + tx] = acc[u];
    }
  }
}

// dynamic shared memory: V, Q1, R (and, nb <= 64, G, T, R11) -- then, cluster mode, two
// 32 x 32 partial Grams read by the other CTAs of the cluster
constexpr size_t filter_smem_small = 2 * kMaxB * kFiltLd + 4 * kSmallNb * (kSmallNb + 1);
constexpr size_t filter_smem_large = 2 * kMaxB * kFiltLd + kMaxB * (kMaxB + 1);
constexpr size_t filter_smem_base =
    sizeof(double) * (filter_smem_small > filter_smem_large ? filter_smem_small : filter_smem_large);

__device__ __forceinline__ void stamp(long long* dbg, int k) {
  if (dbg && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    dbg[k] = (long long)t;
  }
}

template <typename T>
__global__ void __launch_bounds__(kFiltThreads, 1) k_filter_coop(FilterArgs F) {
  cg::grid_group grid = cg::this_grid();
  // the grid barrier: a cooperative launch's grid.sync(), or for d <= 8 * 32 a thread-block
  // cluster of the whole grid and its hardware barrier (release / acquire at cluster scope;
  // the partial Grams go through global memory either way)
  auto gsync = [&]() {
    if (F.cluster) {
      __threadfence();
      cg::this_cluster().sync();
    } else {
      grid.sync();
    }
  };
  stamp(F.dbg, 0);
  extern __shared__ double smd[];
  __shared__ int perm[kMaxB], perm2[kMaxB], s_ch[kMaxB];
  __shared__ double s_mass[kMaxB], s_dg[kMaxB];
  __shared__ int s_nb, s_stop, s_kept, s_rd;
  __shared__ long long s_k;
  DevState* st = F.st;
  const int tid = threadIdx.x;
  __shared__ int s_first;
  __shared__ int64_t s_rows[kMaxB];   // S_t (local rows), loaded together with the state
  if (tid == 0) {
    s_stop = st->stop;
    s_nb = st->b_t;
    s_k = st->k;
    s_first = (F.X0 != nullptr && st->t == 1) ? 1 : 0;   // lazy X_res: block 1 reads X
  }
  if (!F.Vg && tid < kMaxB) s_rows[tid] = F.S_t[tid] - F.row_offset;   // entries >= b_t unused
  __syncthreads();
  if (s_stop || s_nb <= 0) return;   // uniform over the grid
  const int nb = s_nb;
  const bool small = nb <= kSmallNb;
  double* Vs = smd;                          // [kMaxB][33]
  double* Q1s = Vs + kMaxB * kFiltLd;        // [kMaxB][33]
  double* Rs = Q1s + kMaxB * kFiltLd;        // R: [nb][ldr]
  const int ldr = small ? kSmallNb + 1 : kMaxB + 1;
  // small: G, T, R11 copies in shared memory too; large: global scratch (L2)
  double* Gs = small ? Rs + kSmallNb * ldr : F.G;
  const int ldg = small ? ldr : kMaxB;
  double* Ts = small ? Gs + kSmallNb * ldr : F.Tg;
  const int ldt = small ? ldr : kMaxB;
  double* R11s = small ? Ts + kSmallNb * ldr : F.R11;
  const int ld11 = small ? ldr : kMaxB;
  const int64_t c0 = (int64_t)blockIdx.x * kFiltCW;
  const int64_t d = F.d;
  const int nsplit = gridDim.x;
  double* Gp = F.Gpart + (int64_t)blockIdx.x * kMaxB * kMaxB;

  // A: gather + partial Gram.  All of a thread's loads (rows S_t(i), scattered in HBM) are
  // issued before any is stored: one memory latency instead of one per element.
  {
    constexpr int GPT = kMaxB * kFiltCW / kFiltThreads;   // elements per thread (16)
    double v[GPT];
#pragma unroll
    for (int u = 0; u < GPT; ++u) {
      const int e = tid + u * kFiltThreads, i = e / kFiltCW, c = e % kFiltCW;
      double x = 0.0;
      if (i < nb && c0 + c < d) {
        if (F.Vg) {
          x = F.Vg[(int64_t)i * d + c0 + c];
        } else {
          const int64_t r = s_rows[i];
          x = s_first ? (double)((const T*)F.X0)[r * F.ldx0 + c0 + c] : (double)((const T*)F.X)[r * F.ldx + c0 + c];
        }
      }
      v[u] = x;
    }
#pragma unroll
    for (int u = 0; u < GPT; ++u) {
      const int e = tid + u * kFiltThreads, i = e / kFiltCW, c = e % kFiltCW;
      if (i < nb) Vs[i * kFiltLd + c] = v[u];
    }
  }
  __syncthreads();
  // cluster mode with nb <= 32: partial Grams in shared memory, reduced over DSMEM by every
  // CTA into its own slot of Gpart (no global round trip between CTAs, one barrier per
  // reduction instead of two)
  const bool dsm = F.cluster && nb <= 32;
  double* Gl = smd + filter_smem_base / sizeof(double);   // [2][32 x 32]
  const double* Gr = dsm ? Gp : F.G;                        // the reduced Gram, stride kMaxB
  slice_gram(Vs, nb, dsm ? Gl : Gp, dsm ? 32 : kMaxB);
  stamp(F.dbg, 1);
  gsync();
  stamp(F.dbg, 2);
  // B
  if (dsm) {
    reduce_dsmem(Gl, nsplit, nb, Gp);
    __syncthreads();
  } else {
    reduce_slices(F.Gpart, nsplit, nb, F.G);
    gsync();
  }
  stamp(F.dbg, 3);
  // C: pivoted Cholesky + filter + T11 = R11^{-1} (redundant in every CTA).  b_t <= 64:
  // register-resident fast path; larger blocks: shared/L2 path + column-parallel inverse.
  if (!small) {
    Ts = F.Tg + (int64_t)blockIdx.x * kMaxB * kMaxB;
    Gs = F.Ag + (int64_t)blockIdx.x * kMaxB * kMaxB;
  }
  {
    const double tb = st->tau_b < 0.0 ? 1.0 / nb : st->tau_b;
    int kept;
    if (nb <= 32) {
      kept = cta_chol_inv<4>(Gr, nb, 1, F.forced, tb, Rs, ldr, Ts, ldt, perm, s_mass, s_dg, s_ch, &s_rd);
    } else if (small) {
      kept = cta_chol_inv<16>(Gr, nb, 1, F.forced, tb, Rs, ldr, Ts, ldt, perm, s_mass, s_dg, s_ch, &s_rd);
    } else {
      kept = cta_pivchol_reg(F.G, nb, 1, F.forced, tb, Rs, ldr, perm, s_mass, &s_rd);
      __syncthreads();
      stamp(F.dbg, 10);
      cta_trinv_warp(Rs, ldr, perm, kept, Ts, ldt);
    }
    if (tid == 0) s_kept = kept;
  }
  __syncthreads();
  const int bp = s_kept;
  stamp(F.dbg, 4);
  // R11 (step order) and the bookkeeping of l.8-9
  for (int e = tid; e < bp * bp; e += kFiltThreads) {
    const int i = e / bp, j = e % bp;
    const double v = (i <= j) ? Rs[i * ldr + perm[j]] : 0.0;
    if (small) R11s[i * ld11 + j] = v;
    else if (blockIdx.x == 0) F.R11[i * kMaxB + j] = v;
  }
  if (blockIdx.x == 0) {
    for (int i = tid; i < bp; i += kFiltThreads) {
      F.piv[i] = perm[i];
      F.S[s_k + i] = F.S_t[perm[i]];                                  // l.9
    }
    for (int i = tid; i < kMaxB; i += kFiltThreads) F.mass[i] = (i < nb && i <= bp) ? s_mass[i] : 0.0;
    if (tid == 0) {
      st->b_prime = bp;
      if (s_rd) st->rank_def = 1;
      if (bp == 0) {
        st->flags |= RBRP_F_ZERO_BLOCK;
        st->stop = 1;
      }
    }
  }
  if (bp == 0) {   // uniform
    if (dsm) cg::this_cluster().sync();   // the peers are done reading this CTA's partial Gram
    return;
  }
  __syncthreads();
  // D: Q1(:, cols) = V(:, pi(1:b')) T11, partial Gram of Q1
  apply_T(Ts, ldt, bp, Vs, perm, Q1s);
  __syncthreads();
  slice_gram(Q1s, bp, dsm ? Gl + 32 * 32 : Gp, dsm ? 32 : kMaxB);
  stamp(F.dbg, 5);
  gsync();
  stamp(F.dbg, 6);
  // E
  if (dsm) {
    reduce_dsmem(Gl + 32 * 32, nsplit, bp, Gp);
    // this CTA is done reading its peers' shared memory; it may not exit before they are
    // done reading its own (cluster_done() before every exit below)
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    __syncthreads();
  } else {
    reduce_slices(F.Gpart, nsplit, bp, F.G);
    gsync();
  }
  stamp(F.dbg, 7);
  // F: CholQR2 pass (R2 into Rs, T2 = R2^{-1} into Ts).  G2 = I + E: if max|E| is small
  // (the usual case) a parallel perturbation expansion, else the exact Cholesky.
  __shared__ double s_emax;
  {
    double em = 0.0;
    for (int e = tid; e < bp * bp; e += kFiltThreads) {
      const int i = e / bp, j = e - (e / bp) * bp;
      const double x = Gr[i * kMaxB + j] - (i == j ? 1.0 : 0.0);
      Gs[i * ldg + j] = x;
      em = fmax(em, fabs(x));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) em = fmax(em, __shfl_xor_sync(0xffffffffu, em, o));
    if (tid == 0) s_emax = 0.0;
    __syncthreads();
    if ((tid & 31) == 0) atomicMax((unsigned long long*)&s_emax, (unsigned long long)__double_as_longlong(em));
    __syncthreads();
  }
  if (small && bp * s_emax < 1e-4) {
    cholqr2_perturb(Gs, Rs, Ts, Vs, bp, ldr, bp * s_emax);
    if (tid == 0) s_kept = bp;
  } else if (!small && bp * s_emax < 3e-9) {
    // large block, eta^2 < 1e-17: cholqr2_perturb with no fixed-point step and one series
    // term, elementwise: U = Phi(E), R2 = I + U, T2 = I - U
    for (int e = tid; e < bp * bp; e += kFiltThreads) {
      const int i = e / bp, j = e - (e / bp) * bp;
      const double x = Gs[i * ldg + j];
      const double u = i < j ? x : (i == j ? 0.5 * x : 0.0), id = (i == j ? 1.0 : 0.0);
      Ts[i * ldt + j] = id - u;
      Rs[i * ldr + j] = id + u;
    }
    __syncthreads();
    if (tid == 0) s_kept = bp;
  } else {
    int rd2, kept;
    if (bp <= 32 && small) {
      kept = cta_chol_inv<4>(Gr, bp, 2, nullptr, 0.0, Rs, ldr, Ts, ldt, perm2, nullptr, s_dg, s_ch, &rd2);
    } else if (small) {
      kept = cta_chol_inv<16>(Gr, bp, 2, nullptr, 0.0, Rs, ldr, Ts, ldt, perm2, nullptr, s_dg, s_ch, &rd2);
    } else {
      for (int e = tid; e < bp * bp; e += kFiltThreads) Gs[(e / bp) * ldg + e % bp] = F.G[(e / bp) * kMaxB + e % bp];
      __syncthreads();
      kept = cta_pivchol(Gs, ldg, bp, 2, nullptr, 0.0, Rs, ldr, perm2, nullptr, s_dg, s_ch, &rd2);
      __syncthreads();
      cta_trinv_warp(Rs, ldr, perm2, kept, Ts, ldt);
    }
    if (tid == 0) s_kept = kept;
  }
  __syncthreads();
  const int bq = s_kept;   // normally bp; smaller only if G2 lost definiteness
  stamp(F.dbg, 8);
  // R_total = R2 R11 (every CTA holds both factors: the entries are spread over the grid,
  // each dot product in two chains)
  for (int64_t e = (int64_t)blockIdx.x * kFiltThreads + tid; e < (int64_t)bq * bq;
       e += (int64_t)gridDim.x * kFiltThreads) {
    const int i = (int)(e / bq), j = (int)(e % bq);
    double s0 = 0.0, s1 = 0.0;
    if (i <= j) {
      int m = i;
      for (; m + 1 <= j; m += 2) {
        s0 = fma(Rs[i * ldr + m], R11s[m * ld11 + j], s0);
        s1 = fma(Rs[i * ldr + m + 1], R11s[(m + 1) * ld11 + j], s1);
      }
      if (m <= j) s0 = fma(Rs[i * ldr + m], R11s[m * ld11 + j], s0);
    }
    F.Rtot[i * kMaxB + j] = (i <= j) ? s0 + s1 : 0.0;
  }
  if (blockIdx.x == 0) {
    if (tid == 0 && bq < bp) {
      st->b_prime = bq;
      st->rank_def = 1;
      if (bq == 0) st->stop = 1;
    }
  }
  auto cluster_done = [&]() {
    if (dsm) asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  };
  if (bq == 0) {
    cluster_done();
    return;
  }
  // G: Q_b(:, cols) = Q1 T2 -> Vs (free now) -> Qt
  apply_T(Ts, ldt, bq, Q1s, nullptr, Vs);
  __syncthreads();
  T* Qt = (T*)F.Qt;
  const int rows = bq > F.bp_pad ? bq : F.bp_pad;
  for (int e = tid; e < rows * kFiltCW; e += kFiltThreads) {
    const int i = e / kFiltCW, c = e % kFiltCW;
    if (c0 + c >= d) continue;
    Qt[(int64_t)i * d + c0 + c] = (T)(i < bq ? Vs[i * kFiltLd + c] : 0.0);
  }
  if (F.Qp && bq <= 64) {
    // Q_b's two packed images for the 64-row-tile projection (k_pack_q's layout, which the
    // projection would otherwise build in a launch of its own): this CTA's 32 columns, zero
    // rows [b', 64), and (last CTA, at a chunk start) the zero columns of its chunk past d
    const int64_t nc = (d + 63) / 64;
    double* Q2 = F.Qp + nc * 64 * 64;
    const int cw = (blockIdx.x == gridDim.x - 1 && c0 % 64 == 0) ? 64 : kFiltCW;
    for (int e = tid; e < 64 * cw; e += kFiltThreads) {
      const int j = e / cw, cl = e - (e / cw) * cw;
      const int64_t gc = c0 + cl, ch = gc / 64;
      const int col = (int)(gc - ch * 64), pr = j >> 1;
      const double v = (j < bq && cl < kFiltCW && gc < d) ? Vs[j * kFiltLd + cl] : 0.0;
      F.Qp[(ch * 64 + j) * 64 + pack_qswz(j, col)] = v;
      Q2[ch * 64 * 64 + (pr * 64 + (col ^ (2 * (pr & 3)))) * 2 + (j & 1)] = v;
    }
  }
  cluster_done();
  stamp(F.dbg, 9);
}

static size_t filter_smem() { return filter_smem_base + 2 * 32 * 32 * sizeof(double); }

// can a cluster of nc CTAs of the filter be resident (one GPC with nc free SMs)?  Cached per
// device and cluster size; no: the cooperative launch
template <typename T>
bool cluster_fits(int nc, size_t smem) {
  static std::atomic<int> cache[256][9];   // 0 unknown, 1 yes, 2 no
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& c = cache[dev & 255][nc];
  int v = c.load(std::memory_order_relaxed);
  if (v == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nc);
    cfg.blockDim = dim3(kFiltThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = (unsigned)nc;
    la[0].val.clusterDim.y = 1;
    la[0].val.clusterDim.z = 1;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_filter_coop<T>, &cfg);
    if (e != cudaSuccess) cudaGetLastError();   // clear; fall back to the cooperative launch
    v = (e == cudaSuccess && n >= 1) ? 1 : 2;
    c.store(v, std::memory_order_relaxed);
  }
  return v == 1;
}

template <typename T>
cudaError_t launch_filter_coop(const FilterArgs& a, cudaStream_t s) {
  const int nsplit = ceil_div(a.d, kFiltCW);
  const size_t smem = filter_smem();
  static PerDevice attr;
  cudaError_t ae = attr.once(
      [&] { return cudaFuncSetAttribute(k_filter_coop<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
  if (ae != cudaSuccess) return ae;
  // cooperative launch through cudaLaunchKernelEx so that it can be captured in a graph; a
  // grid of at most 8 CTAs runs as one thread-block cluster instead (hardware cluster barrier
  // in place of the cooperative grid barrier; RBRP_FILTER_COOP=1 keeps the cooperative launch)
  const char* ec = getenv("RBRP_FILTER_COOP");
  const bool coop_only = ec && ec[0] == '1';
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nsplit);
  cfg.blockDim = dim3(kFiltThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  FilterArgs b = a;
  b.cluster = !coop_only && nsplit <= 8 && cluster_fits<T>(nsplit, smem);
  if (b.cluster) {
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = (unsigned)nsplit;
    la[0].val.clusterDim.y = 1;
    la[0].val.clusterDim.z = 1;
  } else {
    la[0].id = cudaLaunchAttributeCooperative;
    la[0].val.cooperative = 1;
  }
  cfg.attrs = la;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_filter_coop<T>, b);
}

int filter_coop_nsplit(int64_t d) { return ceil_div(d, kFiltCW); }

template cudaError_t launch_filter_coop<double>(const FilterArgs&, cudaStream_t);
template cudaError_t launch_filter_coop<float>(const FilterArgs&, cudaStream_t);

}  // namespace rbrp
