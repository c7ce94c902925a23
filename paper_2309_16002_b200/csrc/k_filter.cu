// k_filter.cu — a3: gather + local pivoted QR + robust filter (Alg. 2 l.6-9, P:405-408;
// Remark 4.1).
//
// V = X_res(S_t,:)^T (l.6 in residual form: the residual rows already exclude
// span(Q^(t-1))).  Its pivoted QR (l.7) is taken through the fp64 Gram G = V^T V and a
// pivoted Cholesky G(pi,pi) = R^T R: the Schur-complement diagonal at step i is the
// residual column norm^2 of Householder CPQR, so mass[i] = ||R_V(i:b,i:b)||_F^2 exactly
// as in l.8 (reading R10).  Pivot = max Schur diagonal, ties to the lowest draw
// position (R9).  b' from l.8 with tau_b = 1/b_t (R4/R5).  Q_b = V(:,pi(1:b')) R11^-1,
// re-orthonormalised once (CholQR2): Q_b <- Q_b R2^-1, R_total = R2 R11, so that
// L-hat(S'_t,:) = R_total^T (reading R13).
//
// Kernels: k_gram (partial Grams over column splits, gathers V), k_gram_reduce
// (fixed-order sum of the partials), k_factor (one CTA: pivoted Cholesky + filter, or
// plain Cholesky; triangular inverse), k_apply_tinv (rows of T^-T V).
#include <float.h>

#include "launch.cuh"

namespace rbrp {

constexpr int kGramThreads = 256;

// V rows: Vg(i,:) = X_res(S_t[i],:) in fp64 when this rank owns the row, else 0
// (multi-GPU: an allreduce(sum) then gives every rank the full V).
template <typename T>
__global__ void __launch_bounds__(256) k_gather_rows(const T* __restrict__ X, int64_t ldx,
                                                     const int64_t* __restrict__ rows,
                                                     int64_t n_local, int64_t row_offset,
                                                     const DevState* st, int64_t d,
                                                     double* __restrict__ Vg) {
  if (st->stop) return;
  const int i = blockIdx.x;
  if (i >= st->b_t) return;
  const int64_t r = rows[i] - row_offset;
  const bool own = r >= 0 && r < n_local;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x)
    Vg[(int64_t)i * d + c] = own ? (double)X[r * ldx + c] : 0.0;
}

template <typename T>
cudaError_t launch_gather_rows(const T* X, int64_t ldx, const int64_t* rows, int64_t n_local,
                               int64_t row_offset, const DevState* st, int64_t d, double* Vg,
                               cudaStream_t s) {
  k_gather_rows<T><<<kMaxB, 256, 0, s>>>(X, ldx, rows, n_local, row_offset, st, d, Vg);
  return cudaGetLastError();
}
template cudaError_t launch_gather_rows<double>(const double*, int64_t, const int64_t*, int64_t,
                                                int64_t, const DevState*, int64_t, double*,
                                                cudaStream_t);
template cudaError_t launch_gather_rows<float>(const float*, int64_t, const int64_t*, int64_t,
                                               int64_t, const DevState*, int64_t, double*,
                                               cudaStream_t);

template <typename TS>
__global__ void __launch_bounds__(kGramThreads) k_gram(const TS* __restrict__ src, int64_t ld,
                                                       const int64_t* __restrict__ rows,
                                                       int64_t row_offset, const DevState* st,
                                                       int use_bprime, int64_t d,
                                                       double* __restrict__ Vout,
                                                       double* __restrict__ Gpart, int cw) {
  extern __shared__ double tile[];   // [nb][cw + 1]
  const int nb = use_bprime ? st->b_prime : st->b_t;
  if (st->stop || nb <= 0) return;
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * cw;
  const int ldt = cw + 1;
  for (int e = tid; e < nb * cw; e += kGramThreads) {
    const int i = e / cw, c = e % cw;
    double v = 0.0;
    if (c0 + c < d) {
      const int64_t r = rows ? rows[i] - row_offset : i;
      v = (double)src[r * ld + c0 + c];
      if (Vout) Vout[(int64_t)i * d + c0 + c] = v;
    }
    tile[i * ldt + c] = v;
  }
  __syncthreads();
  double* G = Gpart + (int64_t)blockIdx.x * kMaxB * kMaxB;
  for (int p = tid; p < nb * nb; p += kGramThreads) {
    const int i = p / nb, j = p % nb;
    if (i > j) continue;
    double s = 0.0;
    for (int c = 0; c < cw; ++c) s += tile[i * ldt + c] * tile[j * ldt + c];
    G[i * kMaxB + j] = s;
    G[j * kMaxB + i] = s;
  }
}

template <typename TS>
cudaError_t launch_gram(const TS* src, int64_t ld, const int64_t* rows, int64_t row_offset,
                        const DevState* st, int use_bprime, int64_t d, double* Vout, double* Gpart,
                        int nsplit, int cw, cudaStream_t s) {
  size_t smem = (size_t)kMaxB * (cw + 1) * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_gram<TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  k_gram<TS><<<nsplit, kGramThreads, smem, s>>>(src, ld, rows, row_offset, st, use_bprime, d,
                                               Vout, Gpart, cw);
  return cudaGetLastError();
}

__global__ void k_gram_reduce(const double* __restrict__ Gpart, int nsplit, double* __restrict__ G) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= kMaxB * kMaxB) return;
  double s = 0.0;
  for (int q = 0; q < nsplit; ++q) s += Gpart[(int64_t)q * kMaxB * kMaxB + e];
  G[e] = s;
}

cudaError_t launch_gram_reduce(const double* Gpart, int nsplit, double* G, cudaStream_t s) {
  k_gram_reduce<<<kMaxB * kMaxB / 256, 256, 0, s>>>(Gpart, nsplit, G);
  return cudaGetLastError();
}

constexpr int kFactorThreads = 512;

__global__ void __launch_bounds__(kFactorThreads) k_factor(FactorArgs F) {
  extern __shared__ double A[];   // [nb][nb]
  __shared__ int perm[kMaxB];
  __shared__ double s_mass[kMaxB];
  __shared__ int s_p, s_rankdef, s_nb, s_bp;
  DevState* st = F.st;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    s_nb = (st->stop) ? 0 : (F.mode == 1 ? st->b_t : st->b_prime);
    s_rankdef = -1;
  }
  __syncthreads();
  const int nb = s_nb;
  if (nb <= 0) return;
  for (int e = tid; e < nb * nb; e += kFactorThreads) A[e] = F.G[(e / nb) * kMaxB + (e % nb)];
  if (tid < nb) perm[tid] = tid;
  __syncthreads();
  for (int i = 0; i < nb; ++i) {
    if (w == 0) {
      double m = 0.0, best = -DBL_MAX;
      int bi = -1, bperm = 1 << 30;
      for (int j = i + lane; j < nb; j += 32) {
        const double a = A[j * nb + j];
        m += fmax(a, 0.0);
        if (a > best || (a == best && perm[j] < bperm)) { best = a; bi = j; bperm = perm[j]; }
      }
      m = warp_sum(m);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const int op = __shfl_xor_sync(0xffffffffu, bperm, o);
        if (ob > best || (ob == best && op < bperm)) { best = ob; bi = oi; bperm = op; }
      }
      if (lane == 0) {
        if (F.mode == 2) bi = i;
        if (F.mode == 1 && F.forced) {
          for (int j = i; j < nb; ++j)
            if (perm[j] == F.forced[i]) bi = j;
        }
        s_mass[i] = m;
        s_p = bi;
      }
    }
    __syncthreads();
    const int p = s_p;
    if (p != i) {
      for (int r = tid; r < nb; r += kFactorThreads) {   // columns i <-> p (all rows)
        const double x = A[r * nb + i];
        A[r * nb + i] = A[r * nb + p];
        A[r * nb + p] = x;
      }
      __syncthreads();
      for (int c = tid; c < nb; c += kFactorThreads) {   // rows i <-> p
        const double x = A[i * nb + c];
        A[i * nb + c] = A[p * nb + c];
        A[p * nb + c] = x;
      }
      if (tid == 0) {
        const int x = perm[i];
        perm[i] = perm[p];
        perm[p] = x;
      }
      __syncthreads();
    }
    const double aii = A[i * nb + i];
    if (!(aii > 0.0)) {   // non-positive pivot: numerical rank exhausted
      if (tid == 0) s_rankdef = i;
      break;
    }
    const double rii = sqrt(aii);
    __syncthreads();
    for (int c = i + 1 + tid; c < nb; c += kFactorThreads) A[i * nb + c] /= rii;
    if (tid == 0) A[i * nb + i] = rii;
    __syncthreads();
    const int m = nb - i - 1;
    for (int e = tid; e < m * m; e += kFactorThreads) {
      const int j = i + 1 + e / m, l = i + 1 + e % m;
      A[j * nb + l] -= A[i * nb + j] * A[i * nb + l];
    }
    __syncthreads();
  }
  __syncthreads();
  const int rd = s_rankdef;
  if (tid == 0) {
    if (rd >= 0)
      for (int i = rd + 1; i < nb; ++i) s_mass[i] = 0.0;
    int bp;
    if (F.mode == 1) {
      const double tb = st->tau_b < 0.0 ? 1.0 / nb : st->tau_b;
      const double thr = tb * s_mass[0];
      bp = 0;
      if (s_mass[0] > 0.0)
        for (int i = 0; i < nb; ++i)
          if (s_mass[i] >= thr) bp = i + 1;                   // l.8
      if (rd >= 0 && bp > rd) bp = rd;
      if (bp == 0) {
        st->flags |= RBRP_F_ZERO_BLOCK;
        st->stop = 1;
      }
      st->b_prime = bp;
      if (rd >= 0) st->rank_def = 1;
    } else {
      bp = nb;
      if (rd >= 0) {   // CholQR2 pass lost definiteness: keep the leading rd columns
        bp = rd;
        st->b_prime = rd;
        st->rank_def = 1;
        if (rd == 0) st->stop = 1;
      }
    }
    s_bp = bp;
  }
  __syncthreads();
  const int bp = s_bp;
  if (F.mode == 1) {
    for (int i = tid; i < nb; i += kFactorThreads) {
      F.piv[i] = perm[i];
      F.mass[i] = s_mass[i];
    }
    const int64_t k = st->k;
    for (int i = tid; i < bp; i += kFactorThreads) F.S[k + i] = F.S_t[perm[i]];   // l.9
    for (int e = tid; e < bp * bp; e += kFactorThreads) {
      const int i = e / bp, j = e % bp;
      F.R11[i * kMaxB + j] = (i <= j) ? A[i * nb + j] : 0.0;
    }
  } else {
    // R_total = R2 R11 (both upper triangular)
    for (int e = tid; e < bp * bp; e += kFactorThreads) {
      const int i = e / bp, j = e % bp;
      double s = 0.0;
      for (int m = i; m <= j; ++m) s += A[i * nb + m] * F.R11[m * kMaxB + j];
      F.Rtot[i * kMaxB + j] = (i <= j) ? s : 0.0;
    }
  }
  // Tinv = R^-1 (upper triangular), in place, column by column:
  // T(j,j) = 1/R(j,j); T(i,j) = -(sum_{i<=m<j} T(i,m) R(m,j)) / R(j,j).
  __shared__ double tmp[kMaxB];
  __syncthreads();
  for (int j = 0; j < bp; ++j) {
    const double inv = 1.0 / A[j * nb + j];
    for (int i = tid; i < j; i += kFactorThreads) {
      double s = 0.0;
      for (int m = i; m < j; ++m) s += A[i * nb + m] * A[m * nb + j];
      tmp[i] = s;
    }
    __syncthreads();
    for (int i = tid; i < j; i += kFactorThreads) A[i * nb + j] = -tmp[i] * inv;
    if (tid == 0) A[j * nb + j] = inv;
    __syncthreads();
  }
  for (int e = tid; e < bp * bp; e += kFactorThreads) {
    const int i = e / bp, j = e % bp;
    F.Tinv[i * kMaxB + j] = (i <= j) ? A[i * nb + j] : 0.0;
  }
}

cudaError_t launch_factor(const FactorArgs& a, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_factor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kMaxB * kMaxB * (int)sizeof(double));
    attr_set = true;
  }
  k_factor<<<1, kFactorThreads, kMaxB * kMaxB * sizeof(double), s>>>(a);
  return cudaGetLastError();
}

// Qout(i,:) = sum_{j<=i} Tinv(j,i) Vsrc(src(j),:), i < b';  rows [b', bp_pad) zeroed.
template <typename TO>
__global__ void __launch_bounds__(128) k_apply_tinv(const double* __restrict__ Tinv,
                                                    const double* __restrict__ Vsrc,
                                                    const int32_t* __restrict__ perm,
                                                    const DevState* st, int64_t d,
                                                    TO* __restrict__ Qout, int bp_pad) {
  __shared__ double Ts[kMaxB][17];
  __shared__ int src[kMaxB];
  if (st->stop) return;
  const int bp = st->b_prime;
  const int i0 = blockIdx.y * 16;
  const int64_t c = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (i0 >= (bp > bp_pad ? bp : bp_pad)) return;
  const int i1 = min(bp, i0 + 16);
  for (int e = threadIdx.x; e < i1 * 16; e += 128) {
    const int j = e / 16, ii = i0 + e % 16;
    Ts[j][e % 16] = (ii < i1 && j <= ii) ? Tinv[j * kMaxB + ii] : 0.0;
  }
  for (int j = threadIdx.x; j < i1; j += 128) src[j] = perm ? perm[j] : j;
  __syncthreads();
  if (c >= d) return;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  for (int j = 0; j < i1; ++j) {
    const double v = Vsrc[(int64_t)src[j] * d + c];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] += Ts[j][q] * v;
  }
  for (int q = 0; q < 16; ++q) {
    const int i = i0 + q;
    if (i < bp) Qout[(int64_t)i * d + c] = (TO)acc[q];
    else if (i < bp_pad) Qout[(int64_t)i * d + c] = (TO)0;
  }
}

template <typename TO>
cudaError_t launch_apply_tinv(const double* Tinv, const double* Vsrc, const int32_t* perm,
                              const DevState* st, int64_t d, TO* Qout, int bp_pad, cudaStream_t s) {
  int rows = bp_pad > 0 ? bp_pad : kMaxB;
  dim3 grid(ceil_div(d, 128), ceil_div(rows, 16));
  k_apply_tinv<TO><<<grid, 128, 0, s>>>(Tinv, Vsrc, perm, st, d, Qout, bp_pad);
  return cudaGetLastError();
}

template cudaError_t launch_gram<double>(const double*, int64_t, const int64_t*, int64_t,
                                         const DevState*, int, int64_t, double*, double*, int, int,
                                         cudaStream_t);
template cudaError_t launch_gram<float>(const float*, int64_t, const int64_t*, int64_t,
                                        const DevState*, int, int64_t, double*, double*, int, int,
                                        cudaStream_t);
template cudaError_t launch_apply_tinv<double>(const double*, const double*, const int32_t*,
                                               const DevState*, int64_t, double*, int, cudaStream_t);
template cudaError_t launch_apply_tinv<float>(const double*, const double*, const int32_t*,
                                              const DevState*, int64_t, float*, int, cudaStream_t);

}  // namespace rbrp
