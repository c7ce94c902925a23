// mb_chol.cu — per-step cost of the filter's register-resident pivoted Cholesky
// (cta_chol_inv in csrc/k_filter_coop.cu), one CTA of 256 threads, nb = 32 / 64, and a
// variant whose pivot search is three warp REDUX ops (max of the high word, max of the low
// word among the leaders, min index among the exact maxima) instead of a five-level
// shuffle butterfly.  Both must give bit-identical R, T, perm.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_chol scripts/mb_chol.cu
#include <cfloat>
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
  const int kept = chol_inv<EPT, REDUX>(G, nb, 1e-30, R, 65, T, 65, perm, mass, dg, cyc);
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

int main() {
  // G = V^T V for a random 2nb x nb V with a few duplicate columns (ties)
  double* G;
  double *R, *T;
  int* P;
  long long* cyc;
  cudaMallocManaged(&G, kMaxB * kMaxB * 8);
  cudaMallocManaged(&R, 3 * 64 * 65 * 8);
  cudaMallocManaged(&T, 3 * 64 * 65 * 8);
  cudaMallocManaged(&P, 3 * 128 * 4);
  cudaMallocManaged(&cyc, 3 * 8 * 8);
  for (int nb : {32, 64}) {
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
      if (nb == 32) kb<2><<<1, kThreads, sb>>>(G, nb, R + 2 * 64 * 65, T + 2 * 64 * 65, P + 256, cyc + 16);
      else kb<4><<<1, kThreads, sb>>>(G, nb, R + 2 * 64 * 65, T + 2 * 64 * 65, P + 256, cyc + 16);
      if (nb == 32) {
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
    for (int v = 0; v < 3; ++v) {
      const long long* c = cyc + 8 * v;
      const double st = (double)c[5];
      printf("nb=%d %s kept=%lld total %lld cyc = %.0f/step: reduce %.0f pivot %.0f write+bar %.0f update %.0f\n", nb,
             v == 2 ? "blocked" : v ? "redux  " : "shuffle", c[5], c[0], c[0] / st, c[1] / st, c[2] / st, c[3] / st, c[4] / st);
    }
    printf("nb=%d bit-identical: %s (perm0 %d %d %d %d)\n", nb, same ? "yes" : "NO", P[0], P[1], P[2], P[3]);
    free(V);
  }
  return 0;
}
