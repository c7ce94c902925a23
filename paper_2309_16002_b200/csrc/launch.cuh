// launch.cuh — host-side launchers of the librbrp kernels (internal).
#pragma once
#include "common.cuh"

namespace rbrp {

// k_norms.cu — Alg. 2 l.2 and the sampling CDF chunks
template <typename T>
cudaError_t launch_init_norms(const T* X, int64_t ldx, T* Xres, int64_t n, int64_t d, double* dvec,
                              DevState* st, bool copy, cudaStream_t s);
cudaError_t launch_chunk_scan(const double* dvec, int64_t n_local, int64_t chunk0, double* cpre,
                              double* ctot, int32_t* cpos, cudaStream_t s);

// k_sample.cu — Alg. 2 l.3-5
struct SampleArgs {
  DevState* st;
  const double* ctot;     // per-chunk totals (global chunk index)
  const int32_t* cpos;    // per-chunk positive counts
  double* cprefix;        // out: inclusive prefix over chunks
  int nchunks;
  const double* cpre;     // chunk-local inclusive prefix of d (local rows)
  const double* dvec;
  int64_t n_local, row_offset;
  int64_t* S_t;           // out: candidates (global ids)
  int replay_len;         // >= 0: replay (S_t already filled); -1: sample
  uint64_t seed;
  int first;              // 1 on the call right after init (sets D0)
};
cudaError_t launch_sample(const SampleArgs& a, cudaStream_t s);

// k_filter.cu — Alg. 2 l.6-9
template <typename T>
cudaError_t launch_gather_rows(const T* X, int64_t ldx, const int64_t* rows, int64_t n_local,
                               int64_t row_offset, const DevState* st, int64_t d, double* Vg,
                               cudaStream_t s);
template <typename TS>
cudaError_t launch_gram(const TS* src, int64_t ld, const int64_t* rows, int64_t row_offset,
                        const DevState* st, int use_bprime, int64_t d, double* Vout, double* Gpart,
                        int nsplit, int cw, cudaStream_t s);
cudaError_t launch_gram_reduce(const double* Gpart, int nsplit, double* G, cudaStream_t s);
struct FactorArgs {
  DevState* st;
  const double* G;          // kMaxB x kMaxB (ld kMaxB)
  int mode;                 // 1: pivoted Cholesky + filter (l.7-8); 2: Cholesky (CholQR2 pass)
  const int32_t* forced;    // device, forced pivots for this block or null
  int32_t* piv;             // out (mode 1)
  double* mass;             // out (mode 1)
  double* Tinv;             // out: inverse of the triangular factor (upper, ld kMaxB)
  double* R11;              // mode 1 out / mode 2 in: first-pass R (upper, ld kMaxB)
  double* Rtot;             // mode 2 out: R2 * R11
  const int64_t* S_t;       // candidates
  int64_t* S;               // skeleton list (mode 1 appends S'_t at [k, k+b'))
};
cudaError_t launch_factor(const FactorArgs& a, cudaStream_t s);
template <typename TO>
cudaError_t launch_apply_tinv(const double* Tinv, const double* Vsrc, const int32_t* perm,
                              const DevState* st, int64_t d, TO* Qout, int bp_pad, cudaStream_t s);

// k_project.cu — Alg. 2 l.13, l.16 in residual form
template <typename T>
cudaError_t launch_lhat(const T* Xres, int64_t ldx, const T* Qt, int64_t n, int64_t d, T* L,
                        int64_t ldl, const DevState* st, int bucket, cudaStream_t s);
template <typename T>
cudaError_t launch_update(T* Xres, int64_t ldx, const T* Qt, const T* L, int64_t ldl, int64_t n,
                          int64_t d, double* dvec, const DevState* st, int bucket, cudaStream_t s);
template <typename T>
cudaError_t launch_fixup(T* Xres, int64_t ldx, double* dvec, T* L, int64_t ldl, const double* Rtot,
                         const int64_t* S, int64_t n_local, int64_t row_offset, int64_t d,
                         DevState* st, cudaStream_t s);

// k_formw.cu — Alg. 3 by triangular solve
template <typename T>
cudaError_t launch_gather_L1(const T* L, int64_t ldl, const int64_t* S, int64_t k, int64_t n_local,
                             int64_t row_offset, double* L1, cudaStream_t s);
template <typename T>
cudaError_t launch_trinv(const double* L1, int64_t k, T* LinvT, DevState* st, cudaStream_t s);
template <typename T>
cudaError_t launch_gemm_nt(const T* A, int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc,
                           int64_t M, int64_t N, int64_t K, cudaStream_t s);
template <typename T>
cudaError_t launch_w_identity(T* W, int64_t ldw, const int64_t* S, int64_t k, int64_t n_local,
                              int64_t row_offset, cudaStream_t s);

}  // namespace rbrp
