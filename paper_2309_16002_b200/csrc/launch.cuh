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
  double* ctot;           // per-chunk totals (global chunk index; written by a fused scan)
  int32_t* cpos;          // per-chunk positive counts
  double* cprefix;        // out: inclusive prefix over chunks
  int nchunks;
  double* cpre;           // chunk-local inclusive prefix of d (local rows)
  const double* dvec;
  int64_t n_local, row_offset;
  int64_t* S_t;           // out: candidates (global ids)
  const int64_t* S_rep;   // replay: staged candidate ids, copied to S_t
  int replay_len;         // >= 0: replay (ids in S_rep); -1: sample; -2: replay exhausted
  uint64_t seed;
  int first;              // 1 on the call right after init (sets D0)
  const int32_t* piv;     // pivots of the block that just finished (logged)
  BlockLog log;
  unsigned long long cond;   // cudaGraphConditionalHandle of the WHILE node (0: none)
  unsigned long long cond2;  // row-sharded graph loop: handle of the draw-round WHILE node (0: none)
  int dist;               // 1: row-sharded run; this kernel only does the stop test / b_t
  int64_t* cand;          // distributed rounds: candidate rows of kSampleRound draws (-1 = not mine)
  int greedy;             // RBGP (Remark 4.2): S_t = the top b_t rows of d (k_topb), no draw
  const int64_t* S_top;   // greedy: top rows of d, in order
  const int* top_cnt;     // greedy: how many of them have d > 0
  long long* dbg = nullptr;   // optional: %globaltimer stamps of the phases (RBRP_DEBUG_STAMPS)
  int fuse_scan = 0;          // one chunk, single GPU: the sampler scans d itself (no k_chunk_scan)
};
cudaError_t launch_sample(const SampleArgs& a, cudaStream_t s);
// distributed sampling: every rank resolves the draws that land in its
// own chunks; the candidate vectors are combined (max over ranks); every rank then
// accepts in draw order (identical everywhere).  One round = kSampleRound draws.
constexpr int kSampleRound = 256;
cudaError_t launch_draw_resolve(const SampleArgs& a, cudaStream_t s);
cudaError_t launch_draw_accept(const SampleArgs& a, cudaStream_t s);

// k_topb.cu — RBGP candidate block (Remark 4.2): top-B rows of d, ties to the lower row
size_t topb_scratch_bytes(int64_t n, int B);
cudaError_t launch_topb(const double* dvec, int64_t n, int64_t row_offset, int B, void* scratch, int64_t* S_top,
                        int* top_cnt, const DevState* st, cudaStream_t s);

// k_filter.cu — Alg. 2 l.6-9
template <typename T>
cudaError_t launch_gather_rows(const T* X, int64_t ldx, const int64_t* rows, int64_t n_local,
                               int64_t row_offset, const DevState* st, int64_t d, double* Vg,
                               cudaStream_t s, const T* X0 = nullptr, int64_t ldx0 = 0);   // X0: lazy block 1
// k_filter_coop.cu — the whole a3 step in one cooperative kernel
struct FilterArgs {
  DevState* st;
  const void* X;            // X_res (dtype T), used when Vg == nullptr
  int64_t ldx;
  const void* X0;           // lazy X_res copy: block 1 reads V from X itself (or null)
  int64_t ldx0;
  const double* Vg;         // pre-gathered V rows (multi-GPU, after allreduce) or null
  const int64_t* S_t;       // candidates (global ids)
  int64_t row_offset, d;
  double* Gpart;            // nsplit x kMaxB x kMaxB
  double* G;                // kMaxB x kMaxB
  const int32_t* forced;    // forced pivots (device) or null
  int32_t* piv;             // out: pi_V
  double* mass;             // out: ||R_V(i:b,i:b)||_F^2
  double* R11;              // out: first-pass R (upper, ld kMaxB)
  double* Tg;               // scratch: nsplit x kMaxB x kMaxB (b_t > 64 only)
  double* Ag;               // scratch: nsplit x kMaxB x kMaxB (b_t > 64 only)
  double* Rtot;             // out: R2 R11
  int64_t* S;               // skeleton list: S'_t appended at [k, k+b')
  void* Qt;                 // out: Q_b rows (dtype T), ld d; rows [b', bp_pad) zero
  int bp_pad;
  int cluster = 0;          // set by launch_filter_coop: the grid is one thread-block cluster
  double* Qp = nullptr;     // optional: also write Q_b's packed images (k_pack.cu layout) when b' <= 64
  long long* dbg;           // optional: %globaltimer stamps of the phases (CTA 0)
};
template <typename T>
cudaError_t launch_filter_coop(const FilterArgs& a, cudaStream_t s);
int filter_coop_nsplit(int64_t d);

// k_project.cu — Alg. 2 l.13, l.16 in residual form
template <typename T>
cudaError_t launch_lhat(const T* Xres, int64_t ldx, const T* Qt, int64_t n, int64_t d, T* L,
                        int64_t ldl, DevState* st, int bucket, cudaStream_t s);
template <typename T>
cudaError_t launch_update(T* Xres, int64_t ldx, const T* Qt, const T* L, int64_t ldl, int64_t n,
                          int64_t d, double* dvec, DevState* st, int bucket, cudaStream_t s);
template <typename T>
cudaError_t launch_fixup(T* Xres, int64_t ldx, double* dvec, T* L, int64_t ldl, const double* Rtot,
                         const int64_t* S, int64_t n_local, int64_t row_offset, int64_t d,
                         DevState* st, cudaStream_t s);   // Xres == nullptr: leave X (paper form)

// k_project_mma.cu — DMMA (FP64 tensor) projection
bool projection_mma_supported(const void* X, int64_t ldx, const void* Qt, int64_t d);
cudaError_t launch_lhat_mma(const double* Xres, int64_t ldx, const double* Qt, int64_t n, int64_t d,
                            double* L, int64_t ldl, DevState* st, int bucket, cudaStream_t s);
cudaError_t launch_update_mma(double* Xres, int64_t ldx, const double* Qt, const double* L,
                              int64_t ldl, int64_t n, int64_t d, double* dvec, DevState* st,
                              int bucket, cudaStream_t s);
// k_pack.cu — Q_b packed in the shared-memory image of k_lhat_paper (two images)
size_t fused_pack_bytes(int64_t d);
// up to 8 (src, dst, bytes) segments copied by one kernel (4-byte words; bytes % 4 == 0),
// e.g. device -> pinned (host-mapped) memory: one launch instead of one copy per segment
struct CopySeg {
  const void* src;
  void* dst;
  size_t bytes;
};
constexpr int kMaxCopySegs = 8;
cudaError_t launch_copy_segments(const CopySeg* segs, int nseg, cudaStream_t s);
// *st = v, the value travelling as a kernel parameter (no copy, no PCIe read)
cudaError_t launch_set_state(const DevState& v, DevState* st, cudaStream_t s);
// Q_b image 1 of the packed layout (k_pack.cu): row j, column col of a 64-column chunk at
// j * 64 + pack_qswz(j, col) (conflict-free B fragments of the L-hat pass)
__host__ __device__ __forceinline__ int pack_qswz(int j, int col) {
  return col ^ (8 * (j & 1)) ^ (4 * ((j >> 1) & 3));
}
// Qt: rows of Q_b (leading dimension ldq, 0 -> d), d columns packed
// part >= 0: rows of part_range(b', part, pw)
cudaError_t launch_pack_q(const double* Qt, int64_t d, double* Qp, DevState* st, cudaStream_t s, int part = -1,
                          int64_t ldq = 0, int pw = 32);
cudaError_t launch_pack_q(const float* Qt, int64_t d, double* Qp, DevState* st, cudaStream_t s, int part = -1,
                          int64_t ldq = 0, int pw = 32);

// k_lhat_paper.cu — paper form, l.13 + l.16: read-only DMMA pass with 64-row tiles.
// bucket 16 / 32: k_lhat_paper (K-split warps); bucket 64 (fp64): k_lhat64 (N-split warps,
// L-hat tile shared through shared memory).  part >= 0: the rows part_range(b', part, pw) of
// Q_b (b' > pw, pw = 0: the bucket), run only if their count falls in this bucket
int lhat_paper_max_bucket(const void* X, int64_t ldx, int64_t d);
cudaError_t launch_lhat_paper(const double* X, int64_t ldx, const double* Qp, double* L, int64_t ldl,
                              int64_t n, int64_t d, double* dvec, DevState* st, int bucket, bool resid,
                              cudaStream_t s, const double* X0 = nullptr, int64_t ldx0 = 0, int part = -1,
                              int pw = 0);
// fp32 storage (X, X_res, L), fp64 DMMA arithmetic, fp64 norms (R19)
cudaError_t launch_lhat_paper(const float* X, int64_t ldx, const double* Qp, float* L, int64_t ldl,
                              int64_t n, int64_t d, double* dvec, DevState* st, int bucket, bool resid,
                              cudaStream_t s, const float* X0 = nullptr, int64_t ldx0 = 0, int part = -1,
                              int pw = 0);
int lhat_paper_max_bucket_f32(const void* X, int64_t ldx, int64_t d);
// resid: + the update pass (residual form, L2 re-read).  X0 (lazy X_res): in block 1 the
// tile is read from X0 (the input) and the update is written to X (X_res)

// k_proj_tc32.cu — fp32 residual-form projection on tcgen05 (kind::tf32, 3xTF32 split),
// TMEM accumulators; b' <= 64 per launch (part >= 0: 64-column parts of b' > 64)
bool proj_tc32_supported(const void* X, int64_t ldx, int64_t d);
size_t tc32_pack_bytes(int64_t d);
cudaError_t launch_pack_tc32(const float* Qt, int64_t d, float* Qimg, DevState* st, cudaStream_t s, int part);
cudaError_t launch_proj_tc32(float* X, int64_t ldx, const float* Qimg, float* L, int64_t ldl, int64_t n, int64_t d,
                             double* dvec, DevState* st, cudaStream_t s, const float* X0, int64_t ldx0, int part);

// k_paper.cu — left-looking (paper) form of Alg. 2: CGS2 of the candidate rows (l.6),
// Q append (l.10), exact zeros of earlier skeletons' L-hat (R13), d downdate (l.16)
template <typename T>
cudaError_t launch_cgs2_rows(double* Vg, int64_t d, const T* Qall, int64_t k_cap, double* C,
                             const DevState* st, cudaStream_t s);   // C: kMaxB x k_cap scratch
template <typename T>
cudaError_t launch_append_q(const T* Qt, int64_t d, T* Qall, const DevState* st, cudaStream_t s);
template <typename T>
cudaError_t launch_zero_prev(T* L, int64_t ldl, const int64_t* S, int64_t n_local, int64_t row_offset,
                             const DevState* st, cudaStream_t s);
template <typename T>
cudaError_t launch_downdate(const T* L, int64_t ldl, int64_t n, double* dvec, DevState* st,
                            int fused_max, cudaStream_t s);
bool gemm_nt_mma(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                 int64_t M, int64_t N, int64_t K, cudaStream_t s, cudaError_t* err);
// k_lhat_paper.cu: C = A B^T by read-only L-hat passes of 64 (or 32) columns (B: N x K,
// ldb == K); scratch >= gemm_lp_scratch_bytes(N, K), 256-byte aligned
size_t gemm_lp_scratch_bytes(int64_t N, int64_t K);
// min_k: smallest K for which the pass structure beats k_nt_mma (128 for the W GEMMs of
// the ID since k_lhat64 (no K fold), 256 for OSID's W = Y M)
bool gemm_lp_supported(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t K,
                       int64_t min_k = 512);
// Column groups of 64 (k_lhat64; 32 if A's layout only admits k_lhat_paper).  lower_b:
// B(j, m) = 0 for m < j (B = L_1^{-T} of W): each group starts its K range at the 64-column
// chunk holding its first nonzero (about half the work).  nlaunch: + kernels launched
cudaError_t gemm_nt_lp(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                       int64_t M, int64_t N, int64_t K, void* scratch, cudaStream_t s, bool lower_b = false,
                       int64_t min_k = 512, int* nlaunch = nullptr);
// fp32 storage: 32-column groups on k_lhat_paper<32, float> (fp64 DMMA arithmetic)
bool gemm_lp_supported(const float* A, int64_t lda, const float* B, int64_t ldb, int64_t K, int64_t min_k = 512);
cudaError_t gemm_nt_lp(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                       int64_t M, int64_t N, int64_t K, void* scratch, cudaStream_t s, bool lower_b = false,
                       int64_t min_k = 512, int* nlaunch = nullptr);

// k_formw.cu — Alg. 3 by triangular solve
// W = L L_1^{-T} for K = kp <= 128 (kp % 8 == 0): L_1^{-T} resident in shared memory, DMMA;
// lower: skip the zero k-steps of a triangular L_1^{-1}
template <typename T>
bool w_small_supported(int64_t kp);
template <typename T>
cudaError_t launch_w_small(const T* L, int64_t ldl, const T* LinvT, int64_t n, int64_t k, int64_t kp, T* W,
                           int64_t ldw, bool lower, cudaStream_t s);
template <typename T>
cudaError_t launch_gather_L1(const T* L, int64_t ldl, const int64_t* S, int64_t k, int64_t n_local,
                             int64_t row_offset, double* L1, cudaStream_t s);
// LinvT: k x ldo, columns [k, ldo) zero.  scratch (>= k^2/2 doubles, optional): the blocked
// cooperative inversion k_trinv_blk, which overwrites L1 with L_1^{-1}; without: substitution
template <typename T>
cudaError_t launch_trinv(const double* L1, int64_t k, T* LinvT, int64_t ldo, DevState* st,
                         cudaStream_t s, void* scratch = nullptr);
template <typename T>
cudaError_t launch_gemm_nt(const T* A, int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc,
                           int64_t M, int64_t N, int64_t K, cudaStream_t s);
// Remark 5.2 (reading R17): LinvT = pinv_clip(L_1)^T by a one-sided Jacobi SVD (L1 is
// overwritten); scratch >= pinv_scratch_bytes(k); nclip (device, optional) = number of
// singular values below 1e-12 sigma_max that were discarded
size_t pinv_scratch_bytes(int64_t k);
template <typename T>
cudaError_t launch_pinv_clip(double* L1, int64_t k, T* LinvT, int64_t ldo, void* scratch, int* nclip,
                             cudaStream_t s);
cudaError_t launch_diag_test(const double* L1, int64_t k, double* out, cudaStream_t s);   // out: min, max |diag|
template <typename T>
cudaError_t launch_w_identity(T* W, int64_t ldw, const int64_t* S, int64_t k, int64_t n_local,
                              int64_t row_offset, cudaStream_t s);

}  // namespace rbrp
