/*
 * rbrp.h — C ABI of librbrp.so: robust blockwise random pivoting (RBRP) for the
 * row-wise interpolative decomposition X ≈ W·X_S on NVIDIA B200 (sm_100a).
 *
 * Paper: Y. Dong, C. Chen, P.-G. Martinsson, K. Pearce, "Robust blockwise random
 * pivoting: fast and accurate adaptive interpolative decomposition", arXiv 2309.16002.
 * Citations "P:n" are lines of its LaTeX source; "Alg. 2 l.k" is the
 * k-th \State of Algorithm 2.
 *
 *   Problem (Eq. 1.1): given X (n x d), a relative tolerance tau on the
 *   squared Frobenius norm (Remark 1.1) or a fixed rank k, select
 *   skeleton rows S and an interpolation matrix W with
 *       ||X - W X_S||_F^2 = errskel(X; S) <= tau ||X||_F^2      (Prop. 5.1)
 *   Skeleton selection: Alg. 2 with the robust filter tau_b = 1/b
 *   (Remark 4.1).  W: Alg. 3 by triangular solve.
 *
 * Plain C: no C++ or torch types.  Device pointers are CUDA device memory of the
 * calling thread's current device; `stream` is a cudaStream_t passed as void*.
 * Every function returns RBRP_OK (0) or a negative rbrp_status; none throws,
 * aborts or prints.  The library holds no global state besides what a
 * rbrp_comm owns; concurrent calls on distinct workspaces are safe.
 */
#ifndef RBRP_H_
#define RBRP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RBRP_VERSION_MAJOR 0
#define RBRP_VERSION_MINOR 1

typedef enum { RBRP_F32 = 0, RBRP_F64 = 1 } rbrp_dtype;

typedef enum {
  RBRP_OK = 0,
  RBRP_EINVAL = -1,       /* invalid argument (see rbrp_problem) */
  RBRP_ENONFINITE = -2,   /* X contains NaN or Inf */
  RBRP_EDEGENERATE = -3,  /* ||X||_F = 0 */
  RBRP_ENOMEM = -4,       /* workspace smaller than rbrp_workspace_size() */
  RBRP_ECUDA = -5,        /* a CUDA runtime call or kernel launch failed */
  RBRP_ENCCL = -6,        /* an NCCL call failed, or NCCL could not be loaded */
  RBRP_EREPLAY = -7,      /* replay log inconsistent with the problem */
  RBRP_ENOTSUP = -8       /* requested option not built into this library */
} rbrp_status;

/* rbrp_problem.flags */
enum {
  RBRP_INPLACE = 1,    /* X is overwritten by the residual X - L Q^T (saves n*d*w bytes of
                          workspace); X must then be writable */
  RBRP_NO_W = 2,       /* skeleton selection only; W_out is ignored */
  RBRP_FORM_PAPER = 4  /* left-looking form, Alg. 2 exactly as written: X is
                          read only (never copied, never written; INPLACE is ignored);
                          l.6 V = X(S_t,:)^T - Q Q^T X(S_t,:)^T by CGS2; l.13
                          L-hat = X Q_b; l.16 d <- max(0, d - ||L-hat(i,:)||^2)
                          (P:418).  Workspace adds k_cap x d x w for Q.  Without the flag:
                          the residual form of north_star step 4 (X_res updated per block,
                          exact residual norms) */
};

/* rbrp_report.flags (non-fatal) */
enum {
  RBRP_F_TOL_UNREACHED = 1,     /* k_max reached before tau */
  RBRP_F_ZERO_BLOCK = 2,        /* the filter kept no column: V numerically zero */
  RBRP_F_W_CLIPPED = 4,         /* min |diag L_1| < 1e-12 max |diag L_1| (Remark 5.2):
                                   W was formed from the clipped pseudo-inverse of L_1
                                   (singular values < 1e-12 sigma_max discarded) instead of
                                   the triangular solve */
  RBRP_F_SUPPORT_EXHAUSTED = 8, /* fewer than b_t rows had positive weight */
  RBRP_F_NEAR_TIE = 16          /* replay: at least one block ran with forced pivots (blocks
                                   whose logged pivot margin is below the contract's delta,
                                   SURVEY §8(c)); see replay_pivots */
};

/*
 * rbrp_problem — one RBRP call.  All ranks of a multi-GPU call pass identical
 * values except n_local and row_offset.
 *
 *   dtype      element type of X, the residual, L, Q_b and W (RBRP_F32 / RBRP_F64).
 *              Norms, sampling CDF, local pivoted QR, stop sums and the L_1 solve are
 *              always fp64 (reading R19).
 *   n_global   total rows n (>= 1).
 *   n_local    rows of X held by this rank (>= 0).
 *   row_offset global index of this rank's first row; row_offset + n_local <= n_global.
 *              Multi-GPU: rows must be split in contiguous ranges whose boundaries are
 *              multiples of RBRP_CHUNK (except the last rank's end).
 *   d          columns (>= 1).
 *   ld         leading dimension of X in elements (row-major, ld >= d).
 *   tol        tau in (0, 1): stop when ||d||_1 <= tau ||d^(0)||_1 (Alg. 2 l.3).
 *              tol <= 0 selects fixed-rank mode with k = k_max (l.3 "(or |S| < k)").
 *   k_max      fixed rank (tol <= 0), or the cap on |S| in tolerance mode
 *              (0 -> min(n_global, d)).  Buffers L / W / S_out are sized by k_cap =
 *              (k_max ? k_max : min(n_global, d)).
 *   b          block size (>= 1, <= RBRP_MAX_B).
 *   tau_b      filter tolerance (Alg. 2 input (d)): < 0 -> 1/b_t (default,
 *              reading R4); 0 -> plain BRP; must be <= 1.
 *   greedy     0 = RBRP sampling (l.5); 1 = RBGP: S_t = the top-b_t residual norms, ties to
 *              the lower row, positive entries only (Remark 4.2); single GPU only
 *              (a communicator returns RBRP_ENOTSUP).  tau_b = 0 with greedy = 0 is plain BRP.
 *   seed       64-bit sampler seed: Philox4x32-10 key (reading R8).
 *   flags      RBRP_INPLACE | RBRP_NO_W.
 *   replay_blocks / replay_lens / replay_nblocks  (host, optional, may be NULL):
 *              forced candidate blocks S_t (global row ids, concatenated; block t has
 *              replay_lens[t] entries).  The run ends when they are exhausted.
 *   replay_pivots (host, optional): forced local pivot order per block (positions into
 *              the block, concatenated like replay_blocks).  A block whose first entry is
 *              negative is not forced: the GPU's own pivoted QR picks its pivots (the
 *              NEAR_TIE rule: force only the blocks whose pivot margin is below delta).
 */
typedef struct {
  rbrp_dtype dtype;
  int64_t n_global, n_local, row_offset, d, ld;
  double tol;
  int64_t k_max;
  int32_t b;
  double tau_b;
  int32_t greedy;
  uint64_t seed;
  uint32_t flags;
  const int64_t* replay_blocks;
  const int32_t* replay_lens;
  const int32_t* replay_pivots;
  int32_t replay_nblocks;
} rbrp_problem;

#define RBRP_CHUNK 4096   /* rows per sampling chunk (sharding-invariant CDF) */
#define RBRP_MAX_B 128    /* largest supported block size */

/*
 * rbrp_report — host struct filled by rbrp_id.  The per-block arrays are optional
 * caller-owned host arrays of length max_blocks (NULL to skip); blocks beyond
 * max_blocks are counted in nblocks but not logged.
 *   k          |S| at exit.
 *   resid_rel  ||d||_1 / ||d^(0)||_1 at exit = errskel(X; S)/||X||_F^2.
 *   fro2       ||X||_F^2 = ||d^(0)||_1.
 *   nblocks    number of blocks run.
 *   flags      RBRP_F_* bits.
 *   b_t[t], b_prime[t], rho[t]: block size drawn, kept by the filter (l.8), and
 *              ||d^(t)||_1/||d^(0)||_1 after block t.
 *   block_idx  (optional, length max_blocks * b): the candidate block S_t (global row
 *              ids, draw order) of each logged block, -1 padded.
 *   block_piv  (optional, length max_blocks * b): the local pivot order pi_V.
 *   ms_total   device time of the whole call in ms (CUDA events on `stream`).
 *   profile    (in) non-zero: record CUDA events around every phase on `stream` and fill
 *              ms_phase (summed over blocks): [0] init norms + chunk scan, [1] sampler +
 *              stop test, [2] gather + local pivoted QR + filter (a3), [3] projection
 *              L-hat = X_res Q_b, [4] fused update X_res -= L-hat Q_b^T + norms, [5] skeleton
 *              fix-up + chunk scan, [6] W (Alg. 3), [7] collectives.
 *   launches   (out) number of kernels this call launched.
 *   proj_calls (out) number of projection passes that did work (one per block).
 *   proj_ms    (out) device time of the projection passes (a4: L-hat + fused update),
 *              summed over blocks, from %globaltimer stamps taken inside the kernels
 *              (first CTA start of L-hat to last CTA end of the update).
 *   graph      (out) 1 if the block loop ran as one CUDA-graph launch (conditional WHILE
 *              node), 0 if it was launched eagerly (replay, profile, or graphs unusable).
 *   proj_ms_blk (optional, caller array of max_blocks floats, NULL to skip) the projection
 *              device time of each logged block (same stamps as proj_ms).
 *   d_out      (optional, DEVICE array of n_local doubles, NULL to skip) the final
 *              residual squared row norms d^(t)(i) of this rank's rows (Alg. 2 l.16;
 *              0 on skeleton rows).  rbrp_id_sharded: only with one shard.
 */
typedef struct {
  int64_t k;
  double resid_rel;
  double fro2;
  int32_t nblocks;
  uint32_t flags;
  int32_t max_blocks;
  int32_t* b_t;
  int32_t* b_prime;
  double* rho;
  int64_t* block_idx;
  int32_t* block_piv;
  float ms_total;
  int32_t profile;
  float ms_phase[8];
  int32_t launches;
  int32_t proj_calls;
  float proj_ms;
  int32_t graph;
  float* proj_ms_blk;
  double* d_out;
} rbrp_report;

/* Opaque NCCL communicator wrapper; NULL means a single-GPU call. */
typedef struct rbrp_comm rbrp_comm;

/*
 * rbrp_comm_init — create a communicator over `nranks` processes (one GPU each,
 * `device` = this rank's CUDA device).  `nccl_unique_id` is the 128-byte
 * ncclUniqueId produced on rank 0 by rbrp_comm_unique_id and broadcast by the
 * caller (e.g. through torch.distributed).  NCCL is loaded at run time
 * (libnccl.so.2); RBRP_ENCCL if it cannot be.  *c is owned by the caller and
 * released with rbrp_comm_destroy.
 */
int rbrp_comm_unique_id(void* nccl_unique_id_128B);
int rbrp_comm_init(rbrp_comm** c, const void* nccl_unique_id_128B, int nranks, int rank, int device);
int rbrp_comm_destroy(rbrp_comm* c);

/*
 * rbrp_workspace_size — bytes of device workspace rbrp_id needs for problem p
 * (validated as in rbrp_id).  Returns RBRP_EINVAL for an invalid problem.
 */
int rbrp_workspace_size(const rbrp_problem* p, size_t* bytes);

/*
 * rbrp_id — run Alg. 2 (and Alg. 3 unless RBRP_NO_W) on this rank's rows.
 *   X          device, n_local x d row-major with leading dimension ld; read-only
 *              unless RBRP_INPLACE.
 *   workspace  device, >= rbrp_workspace_size() bytes, 256-byte aligned, caller-owned;
 *              contents are scratch on entry and exit.
 *   comm       NULL (single GPU) or a communicator from rbrp_comm_init: this rank's rows are
 *              p->row_offset .. +n_local (row_offset a multiple of RBRP_CHUNK); per block the
 *              chunk totals, the candidate rows of every draw round and the V rows are
 *              combined with NCCL allreduces, and L_1 once for W.
 *   stream     cudaStream_t (as void*); all device work is ordered on it.  The call
 *              blocks the host once per block (the data-dependent stop test, l.3).
 *   S_out      host, int64[k_cap]: skeletons S in selection order (= pi(1:k)), global
 *              row ids; identical on all ranks.  Entries >= k are left untouched.
 *   W_out      device, n_local x k_cap row-major (ld = k_cap) of dtype, or NULL:
 *              W(rest,:) = L_2 L_1^{-1}, W(S_local,:) = I exactly (Alg. 3).  Columns
 *              >= k are left untouched.
 *   rep        host report (may be NULL).
 * Errors: RBRP_EINVAL (b < 1 or > RBRP_MAX_B, tol >= 1 or NaN, tol <= 0 with
 * k_max < 1, tau_b > 1, d < 1, ld < d, n_local < 0, row_offset + n_local > n_global,
 * NULL X with n_local > 0, S_out NULL); RBRP_ENOMEM (ws_bytes too small);
 * RBRP_ENONFINITE; RBRP_EDEGENERATE; RBRP_EREPLAY (replay id outside [0, n_global)
 * or block longer than b); RBRP_ECUDA / RBRP_ENCCL.
 */
int rbrp_id(const rbrp_problem* p, void* X, void* workspace, size_t ws_bytes,
            rbrp_comm* comm, void* stream, int64_t* S_out, void* W_out, rbrp_report* rep);

/*
 * rbrp_id_host — end-to-end call with HOST buffers: copies X (host, n_local x d, leading
 * dimension ld; pinned memory gives full PCIe bandwidth) into a private device copy inside
 * the workspace, runs rbrp_id on it in place (the copy becomes the residual; X_host is
 * never written), and copies W (the first k columns) back into W_host.
 *   X_host     host, n_local x ld elements of dtype.
 *   workspace  device, >= rbrp_workspace_size_host(p) bytes (X copy + W + rbrp_id's
 *              workspace with RBRP_INPLACE), 256-byte aligned.
 *   W_host     host, n_local x k_cap row-major (ld = k_cap) or NULL; columns >= k untouched
 *              (with rep == NULL all k_cap columns are copied).
 *   S_out, comm, stream, rep: as rbrp_id.  Returns after the W copy has completed.
 * Errors as rbrp_id.
 */
int rbrp_workspace_size_host(const rbrp_problem* p, size_t* bytes);
int rbrp_id_host(const rbrp_problem* p, const void* X_host, void* workspace, size_t ws_bytes,
                 rbrp_comm* comm, void* stream, int64_t* S_out, void* W_host, rbrp_report* rep);

/*
 * rbrp_id_sharded — the row-sharded algorithm of a multi-GPU run for
 * `nshards` contiguous row shards held on the CURRENT device by one process: the same
 * kernels and exchange points as `nshards` ranks of rbrp_id with a communicator, with the
 * collectives realised as shared device buffers written by the row owners.  Used to check
 * shard invariance (S, b', rho, W rows identical for any sharding) on one GPU, and to run
 * problems larger than one allocation.
 *   p           problem; n_local / row_offset are ignored (taken from shard_rows).
 *   shard_rows  host int64[nshards]: rows per shard, in order; every shard but the last a
 *               multiple of RBRP_CHUNK; sum = n_global.
 *   X           host array of nshards device pointers (shard h: shard_rows[h] x d, ld).
 *   workspace   host array of nshards device pointers, each >= ws_bytes, where ws_bytes >=
 *               rbrp_workspace_size() of every shard's problem (n_local = shard_rows[h]).
 *   W_out       host array of nshards device pointers (shard_rows[h] x k_cap, ld k_cap), or
 *               NULL; entries may be NULL.
 *   S_out, rep  as rbrp_id (report of shard 0; S is the same for every shard).
 * Errors as rbrp_id, plus RBRP_EINVAL for inconsistent shard sizes.
 */
int rbrp_id_sharded(const rbrp_problem* p, int nshards, const int64_t* shard_rows, void* const* X,
                    void* const* workspace, size_t ws_bytes, void* stream, int64_t* S_out,
                    void* const* W_out, rbrp_report* rep);

/*
 * rbrp_form_w — Alg. 3 on its own: the interpolation matrix from the L and S
 * of a pivoting run.  W(S,:) = I_k (Alg. 3 l.2); W(rest,:) = L_2 L_1^{-1} with L_1 =
 * L(S,:), L_2 = the other rows.
 *   dtype      element type of L and W.  L_1's inverse / pseudo-inverse is computed in fp64.
 *   L          device, n x k row-major with leading dimension ldl >= k (read only).
 *   n          rows of L and W (>= k).
 *   S          host int64[k]: distinct row ids in [0, n), selection order.
 *   method     0 = auto: triangular solve, unless min |diag L_1| < 1e-12 max
 *              |diag L_1| -- then the clipped SVD of Remark 5.2 (reading R17);
 *              1 = triangular solve (L_1 must be lower-triangular, as rbrp_id's L is);
 *              2 = clipped SVD: L_1^{-1} := pinv(L_1) with singular values < 1e-12 sigma_max
 *              discarded (one-sided Jacobi SVD in fp64; any L_1).
 *   W_out      device, n x ldw row-major (ldw >= k); columns >= k untouched.
 *   workspace  device, >= rbrp_form_w_workspace_size() bytes, 256-byte aligned.
 *   stream     cudaStream_t as void*.  The call blocks the host until W is complete.
 *   flags      host (optional): RBRP_F_W_CLIPPED if the clipped SVD was used.
 *   nclip      host (optional): number of singular values discarded (0 for the solve).
 * Errors: RBRP_EINVAL (k < 1, n < k, ldl or ldw < k, S out of range, NULL pointers,
 * method not 0..2, misaligned workspace), RBRP_ENOMEM, RBRP_ECUDA.
 */
int rbrp_form_w_workspace_size(rbrp_dtype dtype, int64_t k, size_t* bytes);
int rbrp_form_w(rbrp_dtype dtype, const void* L, int64_t ldl, int64_t n, const int64_t* S, int64_t k,
                int32_t method, void* W_out, int64_t ldw, void* workspace, size_t ws_bytes, void* stream,
                uint32_t* flags, int32_t* nclip);

/* Human-readable name of a status code (static string; never NULL). */
const char* rbrp_strerror(int status);

/* (major << 16) | minor */
int rbrp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RBRP_H_ */
