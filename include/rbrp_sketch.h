/*
 * rbrp_sketch.h — C ABI of librbrp.so, part 2: sketchy pivoting with LUPP and the
 * oversampled sketchy interpolation matrix (SkLUPP-OSID), the paper's fastest GPU
 * competitor (Table 3) and its gamma-ID-revealing construction (SURVEY §8(f)
 * NEXT-4).  fp64 only.
 *
 *   Sketch (section 3.2; Alg. 4 l.1):  Y = X Omega, Omega (d x l) with
 *       iid N(0, 1/l) entries (Prop. 5.3).
 *   Selection: S = the first k pivot rows of LU with partial pivoting on Y.
 *   Interpolation (Alg. 4; Eq. 5.3): Y_S^T = Q R (economy QR),
 *       W(S,:) = I_k, W(rest,:) = (Y(rest,:) Q) R^{-T}, i.e. W = Y Y_S^+.
 *
 * Conventions as rbrp.h: plain C, device pointers in the calling thread's current
 * device, `stream` a cudaStream_t passed as void*, rbrp_status return codes, no global
 * state.  The readings the paper leaves open are DESIGN.md R25 (embedding generator) and
 * R26 (LUPP: no row swaps, ties to the lowest row, exactly zero columns skipped).
 */
#ifndef RBRP_SKETCH_H_
#define RBRP_SKETCH_H_

#include <stddef.h>
#include <stdint.h>

#include "rbrp.h"

#ifdef __cplusplus
extern "C" {
#endif

#define RBRP_SK_MAX_K 512   /* largest k of rbrp_sketch_id and rbrp_lupp */

/* rbrp_sketch_report.flags */
enum {
  RBRP_SK_SHORT = 1   /* the columns of Y ran out before k pivots (rank of Y < k) */
};

/*
 * rbrp_sketch_report — host struct filled by rbrp_sketch_id.
 *   k          pivots found (= the requested k unless RBRP_SK_SHORT).
 *   flags      RBRP_SK_* bits.
 *   ms_total   device time of the call (CUDA events on `stream`).
 *   profile    (in) non-zero: events around the phases, filling ms_phase:
 *              [0] embedding, [1] sketch Y = X Omega, [2] LUPP, [3] OSID W.
 *   launches   (out) kernels launched.
 */
typedef struct {
  int64_t k;
  uint32_t flags;
  float ms_total;
  int32_t profile;
  float ms_phase[4];
  int32_t launches;
} rbrp_sketch_report;

/*
 * rbrp_gaussian_embedding — Omega^T (l x d, row-major, leading dimension ldo >= d) with
 * iid N(0, 1/l) entries, drawn from `seed` by reading R25: entry (j, i) (e = j d + i) is
 * normal number e % 2 of Philox4x32-10 block q = e / 2, counter (q_lo, q_hi, 0,
 * 0x4F4D4547), key (seed_lo, seed_hi); u1 = U53(w0, w1), u2 = U53(w2, w3),
 * z = sqrt(-2 ln(1 - u1)) (cos | sin)(2 pi u2), entry = z / sqrt(l).
 *   OmegaT   device, written; columns [d, ldo) are left untouched.
 * Errors: RBRP_EINVAL (d < 1, l < 1, ldo < d, NULL OmegaT); RBRP_ECUDA.
 */
int rbrp_gaussian_embedding(int64_t d, int64_t l, uint64_t seed, double* OmegaT, int64_t ldo, void* stream);

/*
 * rbrp_lupp — the first k pivots of partial-pivoting LU on Y (n x l), reading
 * R26.  Blocked (panels of columns), one cooperative kernel; every Schur-complement entry
 * receives its updates a - l*u (product rounded, then the difference; no fused
 * multiply-add) in pivot order, so pivots and multipliers are those of the unblocked
 * textbook loop, bit for bit.
 *   Y          device, n x l row-major, leading dimension ldy >= l; read only.
 *   k          pivots wanted, 1 <= k <= min(n, l, RBRP_SK_MAX_K).
 *   workspace  device, >= rbrp_lupp_workspace_size() bytes, 256-byte aligned.
 *   piv_out    host int64[k]: pivot rows in order (S = piv_out[0 .. *npiv_out)).
 *   pcol_out   host int64[k] or NULL: the column each pivot was taken in (> its index
 *              after a skipped zero column).
 *   npiv_out   host: pivots found (< k only if the columns ran out).
 *   L_out      device n x k (ld k) or NULL: multipliers L(i, m) = l_i of step m for the
 *              rows active at step m, 0 elsewhere.
 * Errors: RBRP_EINVAL; RBRP_ENOMEM; RBRP_ENOTSUP (n above the LUPP row capacity of the
 * device: about 148 x 2800 rows); RBRP_ECUDA.
 */
int rbrp_lupp_workspace_size(int64_t n, int64_t l, int64_t k, size_t* bytes);
int rbrp_lupp(const double* Y, int64_t n, int64_t l, int64_t ldy, int64_t k, void* workspace, size_t ws_bytes,
              void* stream, int64_t* piv_out, int64_t* pcol_out, int64_t* npiv_out, double* L_out);

/*
 * rbrp_sketch_id — SkLUPP-OSID: Y = X Omega (FP64 tensor path), S = LUPP pivots of Y,
 * W = Y Y_S^+ by Alg. 4 (Y_S^T = Q R by CholQR2 on device, W = Y (Q R^{-T})).
 *   X          device, n x d row-major, leading dimension ldx (even, >= d); d % 8 == 0;
 *              16-byte aligned.  Read only.
 *   k, l       skeletons and sketch size, 1 <= k <= min(RBRP_SK_MAX_K, n), k <= l <= 4k
 *              (the paper's oversampling is l = 3k; l may exceed d, as at the
 *              paper's Table 3 ranks k > d/3).
 *   seed       embedding seed (rbrp_gaussian_embedding) when OmegaT is NULL.
 *   OmegaT     device l x d (ld d) or NULL: a caller-supplied Omega^T.
 *   workspace  device, >= rbrp_sketch_workspace_size(), 256-byte aligned.
 *   S_out      host int64[k]: S in pivot order.
 *   W_out      device n x k (ld k) or NULL; W(S,:) = I_k exactly.
 *   rep        host report or NULL.
 * Errors: RBRP_EINVAL (ranges above, NULL X / S_out / workspace); RBRP_ENOMEM;
 * RBRP_ENOTSUP (d % 8 != 0, odd ldx, misaligned X, n above the LUPP capacity);
 * RBRP_EDEGENERATE (Y_S Y_S^T not positive definite: Y_S rank deficient); RBRP_ECUDA.
 */
int rbrp_sketch_workspace_size(int64_t n, int64_t d, int64_t k, int64_t l, size_t* bytes);
int rbrp_sketch_id(const double* X, int64_t n, int64_t d, int64_t ldx, int64_t k, int64_t l, uint64_t seed,
                   const double* OmegaT, void* workspace, size_t ws_bytes, void* stream, int64_t* S_out,
                   double* W_out, rbrp_sketch_report* rep);

#ifdef __cplusplus
}
#endif
#endif /* RBRP_SKETCH_H_ */
