// mb_chol.cu — per-step cost of the filter's register-resident pivoted Cholesky
// (cta_chol_inv in csrc/k_filter_coop.cu), one CTA of 256 threads, nb = 32 / 64, and a
// variant whose pivot search is three warp REDUX ops (max of the high word, max of the low
// word among the leaders, min index among the exact maxima) instead of a five-level
// shuffle butterfly.  Both must give bit-identical R, T, perm.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_chol scripts/mb_chol.cu
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

constexpr int kMaxB = 128;
constexpr int kThreads = 256;

template <int EPT, bool REDUX>
__device__ int chol_inv(const double* __restrict__ Gg, int nb, double tau_b, double* R, int ld, double* Tm,
                        int ldt, int* perm, double* mass, double* dg, long long* cyc) {
  const int tid = threadIdx.x, lane = tid & 31;
  __builtin_assume(__isShared(R));
  __builtin_assume(__isShared(Tm));
  constexpr int NBX = EPT == 4 ? 32 : 64, RSTEP = kThreads / NBX;
  const int ec0 = tid % NBX;
  int er[EPT];
  double a[EPT], ta[EPT];
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int r = tid / NBX + RSTEP * k;
    if (r < nb && ec0 < nb) {
      er[k] = r;
      a[k] = Gg[r * kMaxB + ec0];
      if (r == ec0) dg[r] = a[k];
    } else {
      er[k] = -1;
      a[k] = 0.0;
    }
    ta[k] = 0.0;
  }
  for (int e = tid; e < nb * ldt; e += blockDim.x) Tm[e] = 0.0;
  __syncthreads();
  double dg0 = lane < nb ? dg[lane] : 0.0, dg1 = lane + 32 < nb ? dg[lane + 32] : 0.0;
  unsigned long long chosen = 0ull;
  double thr = 0.0;
  int kept = nb;
  long long t_red = 0, t_piv = 0, t_wr = 0, t_upd = 0;
  for (int i = 0; i < nb; ++i) {
    long long c0 = clock64();
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
    double dp;
    int p;
    if (REDUX) {
      // non-negative doubles order as their bit patterns; a non-positive best maps to key 0
      // (any such pivot is cut below, whichever index is picked)
      const unsigned long long key = best > 0.0 ? (unsigned long long)__double_as_longlong(best) : 0ull;
      const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      p = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bl : (1 << 30));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ms += __shfl_xor_sync(0xffffffffu, ms, o);
      dp = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double om = __shfl_xor_sync(0xffffffffu, ms, o);
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        ms += om;
        if (ob > best || (ob == best && ol < bl)) { best = ob; bl = ol; }
      }
      p = bl;
      const double dq0 = __shfl_sync(0xffffffffu, dg0, p & 31), dq1 = __shfl_sync(0xffffffffu, dg1, p & 31);
      dp = p < 32 ? dq0 : dq1;
    }
    long long c1 = clock64();
    if (i == 0) thr = tau_b * ms;
    int cut = 0;
    if (!(ms > 0.0) || ms < thr) cut = 1;
    if (!cut && !(dp > 0.0)) cut = 2;
    if (tid == 0) mass[i] = ms;
    if (cut) {
      kept = i;
      break;
    }
    const double rii = sqrt(dp);
    const double inv = 1.0 / rii;
    if (tid == 0) {
      perm[i] = p;
      Tm[i * ldt + i] = inv;
    }
    long long c2 = clock64();
    const int c = ec0;
    {
      const int rp = p - tid / NBX;   // row p is this thread's element k = rp / RSTEP
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
    __syncthreads();
    long long c3 = clock64();
    {
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
    long long c4 = clock64();
    t_red += c1 - c0;
    t_piv += c2 - c1;
    t_wr += c3 - c2;
    t_upd += c4 - c3;
  }
  __syncthreads();
  if (tid == 0) {
    cyc[1] = t_red;
    cyc[2] = t_piv;
    cyc[3] = t_wr;
    cyc[4] = t_upd;
  }
  return kept;
}

template <int EPT>
__device__ int chol_fast(const double* __restrict__ Gg, int nb, double tau_b, double* R, int ld, double* Tm,
                        int ldt, int* perm, double* mass, double* dg, long long* cyc) {
  const int tid = threadIdx.x, lane = tid & 31;
  __builtin_assume(__isShared(R));
  __builtin_assume(__isShared(Tm));
  constexpr int NBX = EPT == 4 ? 32 : 64, RSTEP = kThreads / NBX;
  const int ec0 = tid % NBX;
  int er[EPT];
  double a[EPT], ta[EPT];
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int r = tid / NBX + RSTEP * k;
    if (r < nb && ec0 < nb) {
      er[k] = r;
      a[k] = Gg[r * kMaxB + ec0];
      if (r == ec0) dg[r] = a[k];
    } else {
      er[k] = -1;
      a[k] = 0.0;
    }
    ta[k] = 0.0;
  }
  for (int e = tid; e < nb * ldt; e += blockDim.x) Tm[e] = 0.0;
  __syncthreads();
  double dg0 = lane < nb ? dg[lane] : 0.0, dg1 = lane + 32 < nb ? dg[lane + 32] : 0.0;
  unsigned long long chosen = 0ull;
  double thr = 0.0;
  int kept = nb;
  long long t_red = 0, t_piv = 0, t_wr = 0, t_upd = 0;
  for (int i = 0; i < nb; ++i) {
    long long c0 = clock64();
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
    double dp;
    int p;
    {
      const unsigned long long key = best > 0.0 ? (unsigned long long)__double_as_longlong(best) : 0ull;
      const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      p = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bl : (1 << 30));
      dp = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    }
    const double rii = sqrt(dp);
    const double inv = 1.0 / rii;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ms += __shfl_xor_sync(0xffffffffu, ms, o);
    long long c1 = clock64();
    if (tid == 0) {
      perm[i] = p;
      Tm[i * ldt + i] = inv;
    }
    long long c2 = clock64();
    const int c = ec0;
    {
      const int rp = p - tid / NBX;   // row p is this thread's element k = rp / RSTEP
      if (c < nb && rp >= 0 && rp % RSTEP == 0) {
        const int kp = rp / RSTEP;
        double av = a[0];
#pragma unroll
        for (int k = 1; k < EPT; ++k)
          if (k == kp) av = a[k];
        R[i * ld + c] = (c == p) ? rii : (((chosen >> c) & 1ull) ? 0.0 : av * inv);
      }
    }
    chosen |= 1ull << p;
    __syncthreads();
    if (i == 0) thr = tau_b * ms;
    int cut = 0;
    if (!(ms > 0.0) || ms < thr) cut = 1;
    if (!cut && !(dp > 0.0)) cut = 2;
    if (tid == 0) mass[i] = ms;
    if (cut) {
      kept = i;
      break;
    }
    long long c3 = clock64();
    if (lane < nb) {
      const double rl = R[i * ld + lane];
      dg0 = fma(-rl, rl, dg0);
    }
    if (lane + 32 < nb) {
      const double rl = R[i * ld + lane + 32];
      dg1 = fma(-rl, rl, dg1);
    }
    {
      const double ric = R[i * ld + c];
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int r = tid / NBX + RSTEP * k;
        a[k] = fma(-R[i * ld + r], ric, a[k]);
      }
    }
    long long c4 = clock64();
    t_red += c1 - c0;
    t_piv += c2 - c1;
    t_wr += c3 - c2;
    t_upd += c4 - c3;
  }
  __syncthreads();
  if (tid == 0) {
    cyc[1] = t_red;
    cyc[2] = t_piv;
    cyc[3] = t_wr;
    cyc[4] = t_upd;
  }
  return kept;
}

template <int EPT, bool REDUX>
__global__ void __launch_bounds__(kThreads, 1) k(const double* G, int nb, double* Rout, double* Tout, int* pout,
                                                 long long* cyc) {
  extern __shared__ double sm[];
  double* R = sm;
  double* T = sm + 64 * 65;
  __shared__ double mass[128], dg[128];
  __shared__ int perm[128];
  for (int e = threadIdx.x; e < 64 * 65; e += blockDim.x) R[e] = T[e] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  const int kept = REDUX ? chol_inv<EPT, true>(G, nb, 1e-30, R, 65, T, 65, perm, mass, dg, cyc) : chol_fast<EPT>(G, nb, 1e-30, R, 65, T, 65, perm, mass, dg, cyc);
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[5] = kept;
  }
  for (int e = threadIdx.x; e < 64 * 65; e += blockDim.x) {
    Rout[e] = R[e];
    Tout[e] = T[e];
  }
  if (threadIdx.x < 128) pout[threadIdx.x] = threadIdx.x < kept ? perm[threadIdx.x] : -1;
}

// strided 2-D ownership: thread (br, bc) = (tid / 16, tid % 16) owns rows br + 16 jr and
// columns bc + 16 jc, jr, jc < J (J = 2 for nb <= 32, 4 for nb <= 64): a step loads
// J R(i, r) + J T(r, i) + J R(i, c) instead of EPT + EPT + 1
template <int J>
__device__ int chol_blk(const double* __restrict__ Gg, int nb, double tau_b, double* R, int ld, double* Tm,
                        int ldt, int* perm, double* mass, double* dg, long long* cyc) {
  const int tid = threadIdx.x, lane = tid & 31;
  __builtin_assume(__isShared(R));
  __builtin_assume(__isShared(Tm));
  const int br = tid >> 4, bc = tid & 15;
  double a[J][J], ta[J][J];
#pragma unroll
  for (int jr = 0; jr < J; ++jr)
#pragma unroll
    for (int jc = 0; jc < J; ++jc) {
      const int r = br + 16 * jr, c = bc + 16 * jc;
      a[jr][jc] = (r < nb && c < nb) ? Gg[r * kMaxB + c] : 0.0;
      ta[jr][jc] = 0.0;
      if (r == c && r < nb) dg[r] = a[jr][jc];
    }
  for (int e = tid; e < nb * ldt; e += blockDim.x) Tm[e] = 0.0;
  __syncthreads();
  double dg0 = lane < nb ? dg[lane] : 0.0, dg1 = lane + 32 < nb ? dg[lane + 32] : 0.0;
  unsigned long long chosen = 0ull;
  double thr = 0.0;
  int kept = nb;
  long long t_red = 0, t_piv = 0, t_wr = 0, t_upd = 0;
  for (int i = 0; i < nb; ++i) {
    long long c0 = clock64();
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
    const unsigned long long key = best > 0.0 ? (unsigned long long)__double_as_longlong(best) : 0ull;
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    const int p = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bl : (1 << 30));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ms += __shfl_xor_sync(0xffffffffu, ms, o);
    const double dp = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    long long c1 = clock64();
    if (i == 0) thr = tau_b * ms;
    int cut = 0;
    if (!(ms > 0.0) || ms < thr) cut = 1;
    if (!cut && !(dp > 0.0)) cut = 2;
    if (tid == 0) mass[i] = ms;
    if (cut) {
      kept = i;
      break;
    }
    const double rii = sqrt(dp);
    const double inv = 1.0 / rii;
    if (tid == 0) {
      perm[i] = p;
      Tm[i * ldt + i] = inv;
    }
    long long c2 = clock64();
    const int pr = p & 15, pj = p >> 4;
    if (br == pr) {   // row p: R(i, c) for this thread's columns
#pragma unroll
      for (int jc = 0; jc < J; ++jc) {
        const int c = bc + 16 * jc;
        double av = a[0][jc];
#pragma unroll
        for (int jr = 1; jr < J; ++jr)
          if (jr == pj) av = a[jr][jc];
        if (c < nb) R[i * ld + c] = (c == p) ? rii : (((chosen >> c) & 1ull) ? 0.0 : av * inv);
      }
    }
    if (bc == pr) {   // column p: T(r, i) = -acc(r, p) / R(i, p), r < i
#pragma unroll
      for (int jr = 0; jr < J; ++jr) {
        const int r = br + 16 * jr;
        double tv = ta[jr][0];
#pragma unroll
        for (int jc = 1; jc < J; ++jc)
          if (jc == pj) tv = ta[jr][jc];
        if (r < i) Tm[r * ldt + i] = -tv * inv;
      }
    }
    chosen |= 1ull << p;
    __syncthreads();
    long long c3 = clock64();
    {
      double rr[J], tr[J], rc[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        rr[j] = R[i * ld + br + 16 * j];
        tr[j] = Tm[(br + 16 * j) * ldt + i];
        rc[j] = R[i * ld + bc + 16 * j];
      }
#pragma unroll
      for (int jr = 0; jr < J; ++jr)
#pragma unroll
        for (int jc = 0; jc < J; ++jc) {
          a[jr][jc] = fma(-rr[jr], rc[jc], a[jr][jc]);
          ta[jr][jc] = fma(tr[jr], rc[jc], ta[jr][jc]);
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
    long long c4 = clock64();
    t_red += c1 - c0;
    t_piv += c2 - c1;
    t_wr += c3 - c2;
    t_upd += c4 - c3;
  }
  __syncthreads();
  if (tid == 0) {
    cyc[1] = t_red;
    cyc[2] = t_piv;
    cyc[3] = t_wr;
    cyc[4] = t_upd;
  }
  return kept;
}

template <int J>
__global__ void __launch_bounds__(kThreads, 1) kb(const double* G, int nb, double* Rout, double* Tout, int* pout,
                                                  long long* cyc) {
  extern __shared__ double sm[];
  double* R = sm;
  double* T = sm + 64 * 65;
  __shared__ double mass[128], dg[128];
  __shared__ int perm[128];
  for (int e = threadIdx.x; e < 64 * 65; e += blockDim.x) R[e] = T[e] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  const int kept = chol_blk<J>(G, nb, 1e-30, R, 65, T, 65, perm, mass, dg, cyc);
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[5] = kept;
  }
  for (int e = threadIdx.x; e < 64 * 65; e += blockDim.x) {
    Rout[e] = R[e];
    Tout[e] = T[e];
  }
  if (threadIdx.x < 128) pout[threadIdx.x] = threadIdx.x < kept ? perm[threadIdx.x] : -1;
}

// one warp, nb <= NBW (16 or 32): lane j owns column j of the Schur complement (a[r]) and of
// acc(r, j) = sum_{q < i} T(r, q) R(q, j) (ta[r]) in registers; no CTA barrier per step.
// Same fma operands and order as chol_inv<4, true>: bit-identical R, T, perm.
template <int NBW>
__device__ int warp_chol(const double* __restrict__ Gg, int nb, double tau_b, double* R, int ld, double* Tm,
                         int ldt, int* perm, double* mass, double* stage, long long* cyc) {
  const int tid = threadIdx.x, lane = tid & 31;
  __builtin_assume(__isShared(R));
  __builtin_assume(__isShared(Tm));
  __builtin_assume(__isShared(stage));
  int kept = nb;
  if (tid < 32) {
    double a[NBW], ta[NBW];
#pragma unroll
    for (int r = 0; r < NBW; ++r) {
      a[r] = (r < nb && lane < nb) ? Gg[r * kMaxB + lane] : 0.0;
      ta[r] = 0.0;
    }
    double dg = lane < nb ? Gg[lane * kMaxB + lane] : 0.0;
    for (int e = lane; e < nb * ldt; e += 32) Tm[e] = 0.0;
    double* rrow = stage;        // [32] R(i, .)
    double* tcol = stage + 32;   // [32] T(., i)
    bool chosen = false;
    double thr = 0.0;
    long long t_red = 0, t_piv = 0, t_wr = 0, t_upd = 0;
    for (int i = 0; i < nb; ++i) {
      long long c0 = clock64();
      const bool live = lane < nb && !chosen;
      const double ms0 = live ? fmax(dg, 0.0) : 0.0;
      const double best = live ? dg : -DBL_MAX;
      const int bl = live ? lane : (1 << 30);
      const unsigned long long key = best > 0.0 ? (unsigned long long)__double_as_longlong(best) : 0ull;
      const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      const int p = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bl : (1 << 30));
      const double dp = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
      const double rii = sqrt(dp);
      const double inv = 1.0 / rii;
      double ms = ms0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ms += __shfl_xor_sync(0xffffffffu, ms, o);
      long long c1 = clock64();
      if (i == 0) thr = tau_b * ms;
      int cut = 0;
      if (!(ms > 0.0) || ms < thr) cut = 1;
      if (!cut && !(dp > 0.0)) cut = 2;
      if (lane == 0) mass[i] = ms;
      if (cut) {
        kept = i;
        break;
      }
      // row p of the Schur complement: a[p] (warp-uniform index)
      double av = 0.0;
#pragma unroll
      for (int r = 0; r < NBW; ++r)
        if (r == p) av = a[r];
      const double rij = (lane == p) ? rii : (chosen ? 0.0 : av * inv);
      long long c2 = clock64();
      if (lane < nb) R[i * ld + lane] = rij;
      rrow[lane] = rij;
      if (lane == p) {
#pragma unroll
        for (int r = 0; r < NBW; ++r) {
          const double tv = r < i ? -ta[r] * inv : (r == i ? inv : 0.0);
          tcol[r] = tv;
          if (r <= i) Tm[r * ldt + i] = tv;
        }
        chosen = true;
      }
      if (lane == 0) perm[i] = p;
      dg = fma(-rij, rij, dg);
      __syncwarp();
      long long c3 = clock64();
#pragma unroll
      for (int r = 0; r < NBW; r += 2) {
        const double2 rr = *reinterpret_cast<const double2*>(rrow + r);
        const double2 tt = *reinterpret_cast<const double2*>(tcol + r);
        a[r] = fma(-rr.x, rij, a[r]);
        a[r + 1] = fma(-rr.y, rij, a[r + 1]);
        ta[r] = fma(tt.x, rij, ta[r]);
        ta[r + 1] = fma(tt.y, rij, ta[r + 1]);
      }
      __syncwarp();
      long long c4 = clock64();
      t_red += c1 - c0;
      t_piv += c2 - c1;
      t_wr += c3 - c2;
      t_upd += c4 - c3;
    }
    if (lane == 0) {
      cyc[1] = t_red;
      cyc[2] = t_piv;
      cyc[3] = t_wr;
      cyc[4] = t_upd;
    }
  }
  __syncthreads();
  return kept;
}

template <int NBW>
__global__ void __launch_bounds__(kThreads, 1) kw(const double* G, int nb, double* Rout, double* Tout, int* pout,
                                                  long long* cyc) {
  extern __shared__ double sm[];
  double* R = sm;
  double* T = sm + 64 * 65;
  __shared__ double mass[128];
  __shared__ __align__(16) double stage[64];
  __shared__ int perm[128];
  __shared__ int s_kept;
  for (int e = threadIdx.x; e < 64 * 65; e += blockDim.x) R[e] = T[e] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  const int kept = warp_chol<NBW>(G, nb, 1e-30, R, 65, T, 65, perm, mass, stage, cyc);
  if (threadIdx.x == 0) s_kept = kept;
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[5] = s_kept;
  }
  for (int e = threadIdx.x; e < 64 * 65; e += blockDim.x) {
    Rout[e] = R[e];
    Tout[e] = T[e];
  }
  if (threadIdx.x < 128) pout[threadIdx.x] = threadIdx.x < s_kept ? perm[threadIdx.x] : -1;
}

// one warp, nb <= 16, no shared-memory exchange inside the loop: lane l owns column c = l & 15
// and rows rg + 2 k (rg = l >> 4, k < 8) of the Schur complement A and of acc = T R;
// R(i, .) and T(., i) move by shuffles.  Same fma operands and order as chol_inv<4, true>.
template <bool FAST>
__device__ int warp16_chol(const double* __restrict__ Gg, int nb, double tau_b, double* R, int ld, double* Tm,
                           int ldt, int* perm, double* mass, long long* cyc) {
  const int tid = threadIdx.x, lane = tid & 31;
  __shared__ int s_kept16;
  if (tid < 32) {
    const int c = lane & 15, rg = lane >> 4;
    double a[8], ta[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = rg + 2 * k;
      a[k] = (r < nb && c < nb) ? Gg[r * kMaxB + c] : 0.0;
      ta[k] = 0.0;
    }
    double dg = c < nb ? Gg[c * kMaxB + c] : 0.0;
    for (int e = lane; e < nb * ldt; e += 32) Tm[e] = 0.0;
    __syncwarp();
    unsigned chosen = 0u;
    double thr = 0.0;
    int kept = nb;
    for (int i = 0; i < nb; ++i) {
      const bool live = c < nb && !((chosen >> c) & 1u);
      const double best = live ? dg : -DBL_MAX;
      const int bl = live ? c : (1 << 30);
      const unsigned long long key = best > 0.0 ? (unsigned long long)__double_as_longlong(best) : 0ull;
      const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      const int p = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? bl : (1 << 30));
      const double dp = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
      double ms = (rg == 0 && live) ? fmax(dg, 0.0) : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ms += __shfl_xor_sync(0xffffffffu, ms, o);
      const double inv = FAST ? rsqrt(dp) : 1.0 / sqrt(dp);
      const double rii = FAST ? dp * inv : sqrt(dp);
      double av = a[0];
#pragma unroll
      for (int k = 1; k < 8; ++k)
        if (k == (p >> 1)) av = a[k];
      const double rv = (c == p) ? rii : (((chosen >> c) & 1u) ? 0.0 : av * inv);
      const double ric = __shfl_sync(0xffffffffu, rv, c + 16 * (p & 1));
      if (lane < nb) R[i * ld + lane] = ric;
      if (lane == 0) perm[i] = p;
      double tk[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = rg + 2 * k;
        const double t = __shfl_sync(0xffffffffu, ta[k], 16 * rg + p);
        tk[k] = r < i ? -t * inv : (r == i ? inv : 0.0);
        if (c == p && r <= i) Tm[r * ldt + i] = tk[k];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double rr = __shfl_sync(0xffffffffu, ric, rg + 2 * k);
        a[k] = fma(-rr, ric, a[k]);
        ta[k] = fma(tk[k], ric, ta[k]);
      }
      dg = fma(-ric, ric, dg);
      chosen |= 1u << p;
      // the cut of step i (l.8 / a non-positive pivot) is decided here, off the pivot chain:
      // the row / column i just written are then never read (kept = i)
      if (i == 0) thr = tau_b * ms;
      int cut = 0;
      if (!(ms > 0.0) || ms < thr) cut = 1;
      if (!cut && !(dp > 0.0)) cut = 2;
      if (lane == 0) mass[i] = ms;
      if (cut) {
        kept = i;
        break;
      }
    }
    if (lane == 0) s_kept16 = kept;
  }
  __syncthreads();
  return s_kept16;
}

template <bool WFAST>
__global__ void __launch_bounds__(kThreads, 1) kw16(const double* G, int nb, double* Rout, double* Tout, int* pout,
                                                    long long* cyc) {
  extern __shared__ double sm[];
  double* R = sm;
  double* T = sm + 64 * 65;
  __shared__ double mass[128];
  __shared__ int perm[128];
  for (int e = threadIdx.x; e < 64 * 65; e += blockDim.x) R[e] = T[e] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  const int kept = warp16_chol<WFAST>(G, nb, 1e-30, R, 65, T, 65, perm, mass, cyc);
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[5] = kept;
  }
  for (int e = threadIdx.x; e < 64 * 65; e += blockDim.x) {
    Rout[e] = R[e];
    Tout[e] = T[e];
  }
  if (threadIdx.x < 128) pout[threadIdx.x] = threadIdx.x < kept ? perm[threadIdx.x] : -1;
}

int main() {
  // G = V^T V for a random 2nb x nb V with a few duplicate columns (ties)
  double* G;
  double *R, *T;
  int* P;
  long long* cyc;
  cudaMallocManaged(&G, kMaxB * kMaxB * 8);
  cudaMallocManaged(&R, 4 * 64 * 65 * 8);
  cudaMallocManaged(&T, 4 * 64 * 65 * 8);
  cudaMallocManaged(&P, 4 * 128 * 4);
  cudaMallocManaged(&cyc, 4 * 8 * 8);
  for (int nb : {16, 32, 64}) {
    const int m = 2 * nb;
    double* V = (double*)malloc(m * nb * 8);
    srand(7);
    for (int i = 0; i < m * nb; ++i) V[i] = rand() / (double)RAND_MAX - 0.5;
    for (int i = 0; i < m; ++i) V[i * nb + 5] = V[i * nb + 3];   // tie
    memset(G, 0, kMaxB * kMaxB * 8);
    for (int r = 0; r < nb; ++r)
      for (int c = 0; c < nb; ++c) {
        double s = 0;
        for (int i = 0; i < m; ++i) s += V[i * nb + r] * V[i * nb + c];
        G[r * kMaxB + c] = s;
      }
    for (int rep = 0; rep < 3; ++rep) {
      const int sb = 2 * 64 * 65 * 8;
      cudaFuncSetAttribute(k<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      cudaFuncSetAttribute(k<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      cudaFuncSetAttribute(k<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      cudaFuncSetAttribute(k<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      cudaFuncSetAttribute(kb<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      cudaFuncSetAttribute(kb<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      cudaFuncSetAttribute(kw<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      cudaFuncSetAttribute(kw<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      cudaFuncSetAttribute(kw16<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      cudaFuncSetAttribute(kw16<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sb);
      if (nb == 16) kw16<true><<<1, kThreads, sb>>>(G, nb, R + 2 * 64 * 65, T + 2 * 64 * 65, P + 256, cyc + 16);
      if (nb == 16) kw16<false><<<1, kThreads, sb>>>(G, nb, R + 3 * 64 * 65, T + 3 * 64 * 65, P + 384, cyc + 24);
      else if (nb == 32) kw<32><<<1, kThreads, sb>>>(G, nb, R + 3 * 64 * 65, T + 3 * 64 * 65, P + 384, cyc + 24);
      if (nb == 32) kb<2><<<1, kThreads, sb>>>(G, nb, R + 2 * 64 * 65, T + 2 * 64 * 65, P + 256, cyc + 16);
      else if (nb == 64) kb<4><<<1, kThreads, sb>>>(G, nb, R + 2 * 64 * 65, T + 2 * 64 * 65, P + 256, cyc + 16);
      if (nb <= 32) {
        k<4, false><<<1, kThreads, sb>>>(G, nb, R, T, P, cyc);
        k<4, true><<<1, kThreads, sb>>>(G, nb, R + 64 * 65, T + 64 * 65, P + 128, cyc + 8);
      } else {
        k<16, false><<<1, kThreads, sb>>>(G, nb, R, T, P, cyc);
        k<16, true><<<1, kThreads, sb>>>(G, nb, R + 64 * 65, T + 64 * 65, P + 128, cyc + 8);
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
    }
    const bool same = !memcmp(R, R + 64 * 65, 64 * 65 * 8) && !memcmp(T, T + 64 * 65, 64 * 65 * 8) &&
                      !memcmp(P, P + 128, 128 * 4);
    const bool same3 = !memcmp(R, R + 2 * 64 * 65, 64 * 65 * 8) && !memcmp(T, T + 2 * 64 * 65, 64 * 65 * 8) &&
                       !memcmp(P, P + 256, 128 * 4);
    printf("nb=%d blocked variant bit-identical: %s\n", nb, same3 ? "yes" : "NO");
    if (nb <= 32) {
      const bool same4 = !memcmp(R + 64 * 65, R + 3 * 64 * 65, 64 * 65 * 8) && !memcmp(T + 64 * 65, T + 3 * 64 * 65, 64 * 65 * 8) &&
                         !memcmp(P + 128, P + 384, 128 * 4);
      const long long* c = cyc + 24;
      const double st = (double)c[5];
      printf("nb=%d warp    kept=%lld total %lld cyc = %.0f/step: reduce %.0f pivot %.0f write %.0f update %.0f; bit-identical to redux: %s\n",
             nb, c[5], c[0], c[0] / st, c[1] / st, c[2] / st, c[3] / st, c[4] / st, same4 ? "yes" : "NO");
      if (!same4) {
        int nd = 0;
        for (int e = 0; e < 64 * 65 && nd < 5; ++e)
          if (R[64 * 65 + e] != R[3 * 64 * 65 + e] || T[64 * 65 + e] != T[3 * 64 * 65 + e]) {
            printf("  diff at %d: R %g vs %g  T %g vs %g\n", e, R[64 * 65 + e], R[3 * 64 * 65 + e], T[64 * 65 + e], T[3 * 64 * 65 + e]);
            ++nd;
          }
        for (int e = 0; e < nb; ++e) if (P[128 + e] != P[384 + e]) { printf("  perm diff at %d\n", e); break; }
      }
    }
    for (int v = 0; v < 3; ++v) {
      const long long* c = cyc + 8 * v;
      const double st = (double)c[5];
      printf("nb=%d %s kept=%lld total %lld cyc = %.0f/step: reduce %.0f pivot %.0f write+bar %.0f update %.0f\n", nb,
             v == 2 ? "blocked" : v ? "redux  " : "noT    ", c[5], c[0], c[0] / st, c[1] / st, c[2] / st, c[3] / st, c[4] / st);
    }
    double md = 0.0;
    for (int e = 0; e < 64 * 65; ++e) {
      const double x = fabs(R[e] - R[64 * 65 + e]) / (fabs(R[64 * 65 + e]) + 1e-300), y = fabs(T[e] - T[64 * 65 + e]) / (fabs(T[64 * 65 + e]) + 1e-300);
      if (R[64 * 65 + e] != 0.0 && x > md) md = x;
      if (T[64 * 65 + e] != 0.0 && y > md) md = y;
    }
    printf("nb=%d fast vs redux: perm same %s, max rel diff %.3g\n", nb, !memcmp(P, P + 128, 128 * 4) ? "yes" : "NO", md);
    free(V);
  }
  return 0;
}
