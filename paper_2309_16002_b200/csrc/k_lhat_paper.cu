// k_lhat_paper.cu — l.13 + l.16 of Alg. 2 in the paper-literal form (RBRP_FORM_PAPER,
// SURVEY §8(f) NEXT-1): one read-only pass over X per block,
//
//     L-hat = X Q_b^T  (n x b', written to L[:, k : k+b'])            (l.13)
//     d(i) <- max(0, d(i) - ||L-hat(i,:)||^2)                          (l.16, R14)
//
// on the FP64 tensor path (DMMA).  No tile has to stay resident (nothing is written back),
// so tiles are 64 rows tall: every Q_b chunk fetched from L2 serves 64 rows (4x the reuse
// of the residual-form kernel, whose 16-row tiles are bounded by shared memory).
//
// Persistent CTAs, one per SM; 16 consumer warps = 4 row pairs (16 rows each) x 4 column
// groups (16 columns of every 64-column chunk: a K split); an X-producer warp (four TMA
// boxes of 16 columns x 64 rows, 128-byte swizzle) and a Q-producer warp (one bulk copy of
// the pre-packed chunk, layout of k_pack_q) on mbarrier full/empty rings.  At the end of
// a tile the four K-partials of each row pair are folded in a fixed order
// ((c0 + c2) + (c1 + c3)): bitwise reproducible.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "launch.cuh"

namespace rbrp {

namespace lp {
constexpr int R = 64;            // rows per tile
constexpr int KC = 64;           // columns per chunk
constexpr int NCW = 4;           // column groups (16 columns each)
constexpr int NRP = 4;           // row pairs (16 rows each)
constexpr int NCONS = NCW * NRP; // consumer warps
constexpr int NTH = (NCONS + 2) * 32;
constexpr int SLOT = R * KC;     // doubles per X slot (4 boxes of 64 rows x 16 columns)
constexpr int BOX = R * 16;      // doubles per box
constexpr int PACK_ROWS = 64;    // rows of the packed Q_b buffer (k_pack_q)
constexpr int SMEM_MAX = 232448;
}  // namespace lp

__device__ __forceinline__ void lp_dmma(double2& d, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d.x), "+d"(d.y)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ uint32_t lp_su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void lp_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(lp_su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void lp_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(lp_su32(b)) : "memory");
}
__device__ __forceinline__ void lp_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(lp_su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void lp_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n"
      "}\n" ::"r"(lp_su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ double2 lp_lds2(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(lp_su32(p)));
  return v;
}
__device__ __forceinline__ void lp_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(lp::NCONS * 32) : "memory"); }
// Q chunk layout of k_pack_q: row j, column c at j * 64 + (c ^ f(j))
__device__ __forceinline__ int lp_qswz(int j, int col) { return col ^ (8 * (j & 1)) ^ (4 * ((j >> 1) & 3)); }
// X slot: box (col >> 4) of 64 rows x 16 doubles, 128-byte swizzle of 16-byte chunks by row
__device__ __forceinline__ int lp_xoff(int row, int col) {
  return (col >> 4) * lp::BOX + row * 16 + ((((col & 15) >> 1) ^ (row & 7)) << 1);
}

struct LpRing {
  int i = 0, ph = 0;
  __device__ __forceinline__ void next(int n) {
    if (++i == n) {
      i = 0;
      ph ^= 1;
    }
  }
};

template <int BPB>
struct LpCfg {
  static constexpr int NT = BPB / 8;
  static constexpr int ACC = 2 * NT * 2;          // doubles per lane of a row pair's partial
  static constexpr int QSTAGE = BPB * lp::KC;
  static constexpr int SCR = lp::NRP * 2 * ACC * 32;   // two partial slots per row pair
  static size_t smem(int ns, int nq) {
    return (size_t)ns * lp::SLOT * 8 + (size_t)nq * QSTAGE * 8 + (size_t)(SCR + 2 * lp::NRP * lp::NCW * 16) * 8 +
           (2 * ns + 2 * nq) * 8 + 1024;
  }
  static bool rings(int& ns, int& nq) {
    ns = 4;
    nq = 4;
    if (const char* e = getenv("RBRP_LP_NS")) ns = atoi(e);   // experiments only
    if (const char* e = getenv("RBRP_LP_NQ")) nq = atoi(e);
    while (smem(ns, nq) > (size_t)lp::SMEM_MAX && nq > 2) --nq;
    while (smem(ns, nq) > (size_t)lp::SMEM_MAX && ns > 2) --ns;
    return smem(ns, nq) <= (size_t)lp::SMEM_MAX;
  }
};

template <int BPB>
__global__ void __launch_bounds__(lp::NTH, 1)
    k_lhat_paper(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap xmap0,
                 int lazy, const double* __restrict__ Qp,
                 double* __restrict__ L, int64_t ldl, int64_t n, int d, int nc, int NS, int NQ,
                 double* __restrict__ dvec, DevState* st, double* __restrict__ Xr, int64_t ldx, int resid) {
  using Cf = LpCfg<BPB>;
  constexpr int NT = Cf::NT;
  using namespace lp;
  if (st->stop) return;
  const int bp = st->b_prime;
  if (bp <= 0 || bucket_of(bp) != BPB) return;
  const int64_t k0 = st->k;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->ts0 = gtimer();

  extern __shared__ __align__(1024) double sm_raw[];
  double* sm = sm_raw + ((1024u - (lp_su32(sm_raw) & 1023u)) & 1023u) / 8;
  double* xs = sm;                                   // NS x SLOT
  double* qs = xs + (size_t)NS * SLOT;               // NQ x QSTAGE
  double* scr = qs + (size_t)NQ * Cf::QSTAGE;        // [rp][slot 0..1][ACC][32]
  double* nrm = scr + Cf::SCR;                       // [tile parity][rp][cw][16] row-norm partials
  uint64_t* xfull = reinterpret_cast<uint64_t*>(nrm + 2 * NRP * NCW * 16);
  uint64_t* xempty = xfull + NS;
  uint64_t* qfull = xempty + NS;
  uint64_t* qempty = qfull + NQ;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t ntiles = (n + R - 1) / R;
  const int T = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      lp_init(&xfull[s], 1);
      lp_init(&xempty[s], NCONS);
    }
    for (int s = 0; s < NQ; ++s) {
      lp_init(&qfull[s], 1);
      lp_init(&qempty[s], NCONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto row0_of = [&](int p) { return ((int64_t)blockIdx.x + (int64_t)p * gridDim.x) * R; };
  const int npass = resid ? 2 : 1;   // residual form: L-hat pass, then update pass per tile
  const int steps = T * nc * npass;

  if (T == 0) {
  } else if (w == NCONS) {
    // X producer.  Residual form: the L-hat pass loads a tile with an L2 evict_last
    // policy, the update pass (same addresses, shortly after) with evict_first, so the
    // second read is served by L2 and HBM sees one read of X_res.
    // lazy X_res copy: block 1 reads the input X (xmap0); the update pass writes X_res
    const CUtensorMap* mp = (lazy && st->t == 1) ? &xmap0 : &xmap;
    if (lane == 0) {
      uint64_t pol_keep, pol_drop;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_keep));
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_drop));
      LpRing xr;
      for (int s = 0; s < steps; ++s) {
        if (s >= NS) lp_wait(&xempty[xr.i], xr.ph ^ 1);
        lp_expect(&xfull[xr.i], SLOT * 8);   // out-of-bounds rows / columns are zero-filled
        double* dst = xs + (size_t)xr.i * SLOT;
        const int y = (int)row0_of(s / (nc * npass)), c = s % nc;
        const bool second = resid && ((s / nc) & 1);
        const uint64_t pol = resid ? (second ? pol_drop : pol_keep) : pol_drop;
#pragma unroll
        for (int b = 0; b < 4; ++b)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
              "[%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(lp_su32(dst + b * BOX)),
              "l"(mp), "r"(c * KC + 16 * b), "r"(y), "r"(lp_su32(&xfull[xr.i])), "l"(pol)
              : "memory");
        xr.next(NS);
      }
    }
    __syncwarp();
  } else if (w == NCONS + 1) {
    // Q producer (the packed Q_b chunk c is the same for every tile)
    if (lane == 0) {
      LpRing qr;
      for (int s = 0; s < steps; ++s) {
        if (s >= NQ) lp_wait(&qempty[qr.i], qr.ph ^ 1);
        lp_expect(&qfull[qr.i], (uint32_t)(Cf::QSTAGE * 8));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                lp_su32(qs + (size_t)qr.i * Cf::QSTAGE)),
            "l"(Qp + (size_t)(s % nc) * PACK_ROWS * KC), "r"((uint32_t)(Cf::QSTAGE * 8)),
            "r"(lp_su32(&qfull[qr.i]))
            : "memory");
        qr.next(NQ);
      }
    }
    __syncwarp();
  } else {
    // consumers: warp = (row pair rp, column group cw)
    const int rp = w >> 2, cw = w & 3;
    const int g = lane >> 2, q = lane & 3;
    const int pg = (g >> 1) + 4 * (g & 1);   // tile row of MMA row g (bank-conflict-free)
    int xo[2][2];                            // [row group][8-column half]
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int h = 0; h < 2; ++h) xo[r][h] = lp_xoff(16 * rp + 8 * r + pg, 16 * cw + 8 * h + 2 * q);
    double2 acc[2][NT];
    LpRing qr, xr;
    for (int p = 0; p < T; ++p) {
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[r][t] = make_double2(0.0, 0.0);
      for (int c = 0; c < nc; ++c) {
        lp_wait(&qfull[qr.i], qr.ph);
        lp_wait(&xfull[xr.i], xr.ph);
        const double* xsl = xs + (size_t)xr.i * SLOT;
        const double* Qs = qs + (size_t)qr.i * Cf::QSTAGE;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double2 a0 = lp_lds2(xsl + xo[0][h]);
          const double2 a1 = lp_lds2(xsl + xo[1][h]);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const int j = 8 * t + g;
            const double2 b = lp_lds2(Qs + j * KC + lp_qswz(j, 16 * cw + 8 * h + 2 * q));
            lp_dmma(acc[0][t], a0.x, b.x);
            lp_dmma(acc[1][t], a1.x, b.x);
            lp_dmma(acc[0][t], a0.y, b.y);
            lp_dmma(acc[1][t], a1.y, b.y);
          }
        }
        __syncwarp();
        if (lane == 0) {   // operands consumed (they fed the MMAs): release both buffers
          lp_arrive(&xempty[xr.i]);
          lp_arrive(&qempty[qr.i]);
        }
        xr.next(NS);
        qr.next(NQ);
      }
      // tile end: P = (c0 + c2) + (c1 + c3) per row pair, in registers of the cw = 0 warp
      double* sl = scr + (size_t)rp * 2 * Cf::ACC * 32;
#define LP_S(slot, r, t, hh) sl[((slot) * Cf::ACC + ((r) * NT + (t)) * 2 + (hh)) * 32 + lane]
      if (cw >= 2) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            LP_S(cw - 2, r, t, 0) = acc[r][t].x;
            LP_S(cw - 2, r, t, 1) = acc[r][t].y;
          }
      }
      lp_bar();
      if (cw < 2) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            acc[r][t].x += LP_S(cw, r, t, 0);
            acc[r][t].y += LP_S(cw, r, t, 1);
          }
      }
      if (cw == 1) {   // c1 + c3 back into slot 1 (read above by this warp only)
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            LP_S(1, r, t, 0) = acc[r][t].x;
            LP_S(1, r, t, 1) = acc[r][t].y;
          }
      }
      lp_bar();
      if (cw == 0) {
        const int64_t r0 = row0_of(p) + 16 * rp;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          double ss = 0.0;
          const int64_t row = r0 + 8 * r + pg;
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const double vx = acc[r][t].x + LP_S(1, r, t, 0);
            const double vy = acc[r][t].y + LP_S(1, r, t, 1);
            const int j = 8 * t + 2 * q;
            if (row < n) {
              if (j < bp) L[row * ldl + k0 + j] = vx;
              if (j + 1 < bp) L[row * ldl + k0 + j + 1] = vy;
            }
            ss += vx * vx + vy * vy;
            if (resid) {   // -P for the update pass, in scratch slot 0 (read only by this warp)
              LP_S(0, r, t, 0) = -vx;
              LP_S(0, r, t, 1) = -vy;
            }
          }
          if (!resid) {
            // l.16 downdate (paper form): sum over the row's columns (q lanes)
            ss += __shfl_xor_sync(0xffffffffu, ss, 1);
            ss += __shfl_xor_sync(0xffffffffu, ss, 2);
            if (q == 0 && row < n) dvec[row] = fmax(dvec[row] - ss, 0.0);
          }
        }
      }
      if (resid) {
        // ----- update pass (residual form, l.16): X(tile) -= L-hat Q_b, chunk by chunk;
        // the chunks come back through L2 (read from HBM by the L-hat pass just before)
        lp_bar();
        double2 pf[2][NT];   // -P rows of this row pair, accumulator layout (A fragments)
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int t = 0; t < NT; ++t) pf[r][t] = make_double2(LP_S(0, r, t, 0), LP_S(0, r, t, 1));
        const int64_t r0 = row0_of(p) + 16 * rp;
        double nr[2] = {0.0, 0.0};
        for (int c = 0; c < nc; ++c) {
          lp_wait(&qfull[qr.i], qr.ph);
          lp_wait(&xfull[xr.i], xr.ph);
          const double* xsl = xs + (size_t)xr.i * SLOT;
          const double* Qs = qs + (size_t)qr.i * Cf::QSTAGE;
          double2 xv[2][2];
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int h = 0; h < 2; ++h) xv[r][h] = lp_lds2(xsl + xo[r][h]);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              const int j0 = 8 * t + 2 * q, col = 16 * cw + 8 * h + g;
              const double b0 = Qs[j0 * KC + lp_qswz(j0, col)];
              const double b1 = Qs[(j0 + 1) * KC + lp_qswz(j0 + 1, col)];
              lp_dmma(xv[0][h], pf[0][t].x, b0);
              lp_dmma(xv[1][h], pf[1][t].x, b0);
              lp_dmma(xv[0][h], pf[0][t].y, b1);
              lp_dmma(xv[1][h], pf[1][t].y, b1);
            }
          }
          __syncwarp();
          if (lane == 0) {
            lp_arrive(&xempty[xr.i]);
            lp_arrive(&qempty[qr.i]);
          }
          xr.next(NS);
          qr.next(NQ);
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int64_t row = r0 + 8 * r + pg;
            if (row >= n) continue;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int col = c * KC + 16 * cw + 8 * h + 2 * q;
              if (col < d) {
                __stcs(reinterpret_cast<double2*>(Xr + row * ldx + col), xv[r][h]);
                nr[r] += xv[r][h].x * xv[r][h].x + xv[r][h].y * xv[r][h].y;
              }
            }
          }
        }
        // d(i) = ||x_res,i||^2: q lanes, then the 4 column groups in order
        double* nb = nrm + (size_t)((p & 1) * NRP + rp) * NCW * 16;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          double v = nr[r];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          if (q == 0) nb[cw * 16 + 8 * r + pg] = v;
        }
        lp_bar();
        if (cw == 0 && lane < 16) {
          const double v = (nb[lane] + nb[16 + lane]) + (nb[32 + lane] + nb[48 + lane]);
          const int64_t row = r0 + lane;
          if (row < n) dvec[row] = v;
        }
      }
#undef LP_S
      // scratch is rewritten at the next tile's fold, nc chunk steps later; the NQ-stage Q
      // ring keeps every warp within NQ steps of the others, so this barrier is only
      // needed when a tile has no more than NQ chunks
      if (nc <= NQ + 1) lp_bar();
    }
  }
  proj_end_stamp(st);
}

static PFN_cuTensorMapEncodeTiled_v12000 lp_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

static int lp_sms() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

int lhat_paper_max_bucket(const void* X, int64_t ldx, int64_t d) {
  if (d % 2 || d < 16 || ldx % 2 || ((uintptr_t)X % 16)) return 0;
  int ns, nq, best = 0;
  if (LpCfg<16>::rings(ns, nq)) best = 16;
  if (LpCfg<32>::rings(ns, nq)) best = 32;
  return best;
}

template <int BPB>
static cudaError_t go_lp(const CUtensorMap& map, const CUtensorMap& map0, int lazy, const double* Qp, double* L,
                         int64_t ldl, int64_t n, int64_t d, double* dvec, DevState* st, double* Xr, int64_t ldx,
                         int resid, cudaStream_t s) {
  using Cf = LpCfg<BPB>;
  int ns, nq;
  if (!Cf::rings(ns, nq)) return cudaErrorInvalidValue;
  const size_t smem = Cf::smem(ns, nq);
  cudaFuncSetAttribute(k_lhat_paper<BPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int nc = (int)((d + lp::KC - 1) / lp::KC);
  k_lhat_paper<BPB><<<lp_sms(), lp::NTH, smem, s>>>(map, map0, lazy, Qp, L, ldl, n, (int)d, nc, ns, nq, dvec, st,
                                                     Xr, ldx, resid);
  return cudaGetLastError();
}

cudaError_t launch_lhat_paper(const double* X, int64_t ldx, const double* Qp, double* L, int64_t ldl,
                              int64_t n, int64_t d, double* dvec, DevState* st, int bucket, bool resid,
                              cudaStream_t s, const double* X0, int64_t ldx0) {
  if (n <= 0) return cudaSuccess;
  auto enc = lp_encode();
  if (!enc) return cudaErrorNotSupported;
  auto make_map = [&](const double* P, int64_t ld, CUtensorMap* map) {
    const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    const cuuint32_t box[2] = {16, (cuuint32_t)lp::R};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)P, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  CUtensorMap map, map0;
  if (!make_map(X, ldx, &map)) return cudaErrorInvalidValue;
  const int lazy = X0 != nullptr ? 1 : 0;
  if (!make_map(lazy ? X0 : X, lazy ? ldx0 : ldx, &map0)) return cudaErrorInvalidValue;
  switch (bucket) {
    case 16: return go_lp<16>(map, map0, lazy, Qp, L, ldl, n, d, dvec, st, (double*)X, ldx, resid ? 1 : 0, s);
    case 32: return go_lp<32>(map, map0, lazy, Qp, L, ldl, n, d, dvec, st, (double*)X, ldx, resid ? 1 : 0, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rbrp
