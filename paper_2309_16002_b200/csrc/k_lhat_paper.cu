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
#include <string.h>

#include "launch.cuh"

#ifndef LP_TRACE
#define LP_TRACE 0   // cycle trace of CTA 0 (build with -DLP_TRACE=1; scripts/lp_trace.py)
#endif

namespace rbrp {

namespace lp {
constexpr int R = 64;            // rows per tile
constexpr int KC = 64;           // columns per chunk
constexpr int NCW = 4;           // column groups (16 columns each)
constexpr int NRP = 4;           // row pairs (16 rows each)
constexpr int NCONS = NCW * NRP; // consumer warps
constexpr int NTH = (NCONS + 2) * 32;   // consumers + X and Q producer warps
constexpr int SLOT = R * KC;     // elements per X slot
constexpr int PACK_ROWS = 64;    // rows of the packed Q_b buffer (k_pack_q)
constexpr int SMEM_MAX = 232448;
}  // namespace lp

__device__ __forceinline__ void lp_dmma(double2& d, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d.x), "+d"(d.y)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void lp_dmma_v(double2& d, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
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
__device__ __forceinline__ double2 lp_lds2s(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void lp_waits(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n"
      "}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void lp_arrives(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(b) : "memory");
}
__device__ __forceinline__ double2 lp_lds2(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(lp_su32(p)));
  return v;
}
__device__ __forceinline__ void lp_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(lp::NCONS * 32) : "memory"); }
// Q chunk layout of k_pack_q: row j, column c at j * 64 + (c ^ f(j))
__device__ __forceinline__ int lp_qswz(int j, int col) { return col ^ (8 * (j & 1)) ^ (4 * ((j >> 1) & 3)); }

// element type of X / X_res / L (storage); the arithmetic is fp64 DMMA either way.  A
// 128-byte TMA box row holds CPB elements; MMA row g of an 8-row group is tile row pg(g),
// chosen so that the 8-byte fragment loads of a half-warp hit 32 distinct banks under the
// 128-byte swizzle (fp64: rows {0,4,1,5}/{2,6,3,7}; fp32: rows {0,2,4,6}/{1,3,5,7}).
template <typename E>
struct LpE;
template <>
struct LpE<double> {
  static constexpr int CPB = 16;
  __device__ static int pg(int g) { return (g >> 1) + 4 * (g & 1); }
  __device__ static double2 ld2(uint32_t a) { return lp_lds2s(a); }
  __device__ static double2 rnd(double2 v) { return v; }   // the value as stored
  __device__ static void st2(double* p, double2 v) { __stcs(reinterpret_cast<double2*>(p), v); }
};
template <>
struct LpE<float> {
  static constexpr int CPB = 32;
  __device__ static int pg(int g) { return 2 * (g & 3) + (g >> 2); }
  __device__ static double2 ld2(uint32_t a) {
    float x, y;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(x), "=f"(y) : "r"(a));
    return make_double2(x, y);
  }
  __device__ static double2 rnd(double2 v) { return make_double2((double)(float)v.x, (double)(float)v.y); }
  __device__ static void st2(float* p, double2 v) {
    __stcs(reinterpret_cast<float2*>(p), make_float2((float)v.x, (float)v.y));
  }
};
// X slot: KC / CPB boxes of 64 rows x CPB elements, 128-byte swizzle of 16-byte chunks by row
template <typename E>
__device__ __forceinline__ int lp_xoff_e(int row, int col) {
  constexpr int CPB = LpE<E>::CPB, EPC = 16 / (int)sizeof(E);   // elements per 16-byte chunk
  const int c = col % CPB;
  return (col / CPB) * (lp::R * CPB) + row * CPB + (((c / EPC) ^ (row & 7)) * EPC) + (c % EPC);
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

template <int BPB, typename E = double>
struct LpCfg {
  static constexpr int NT = BPB / 8;
  static constexpr int ACC = 2 * NT * 2;          // doubles per lane of a row pair's partial
  static constexpr int QSTAGE = BPB * lp::KC;
  static constexpr int SCR = lp::NRP * 2 * ACC * 32;   // two partial slots per row pair
  static constexpr int SLOTB = lp::SLOT * (int)sizeof(E);   // bytes per X slot
  static size_t smem(int ns, int nq) {
    return (size_t)ns * SLOTB + (size_t)nq * QSTAGE * 8 + (size_t)(SCR + 2 * lp::NRP * lp::NCW * 16) * 8 +
           (2 * ns + 2 * nq) * 8 + 1024;
  }
  static bool rings(int& ns, int& nq) {
    ns = BPB <= 16 ? 5 : 4;   // the small-b' pass is HBM-bound: one X slot more in flight
    nq = 4;
    if (const char* e = getenv("RBRP_LP_NS")) ns = atoi(e);   // experiments only
    if (const char* e = getenv("RBRP_LP_NQ")) nq = atoi(e);
    while (smem(ns, nq) > (size_t)lp::SMEM_MAX && nq > 2) --nq;
    while (smem(ns, nq) > (size_t)lp::SMEM_MAX && ns > 2) --ns;
    return smem(ns, nq) <= (size_t)lp::SMEM_MAX;
  }
};

template <int BPB, typename E>
__global__ void __launch_bounds__(lp::NTH, 1)
    k_lhat_paper(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap xmap0,
                 int lazy, const double* __restrict__ Qp,
                 E* __restrict__ L, int64_t ldl, int64_t n, int d, int nc, int NS, int NQ,
                 double* __restrict__ dvec, DevState* st, E* __restrict__ Xr, int64_t ldx, int resid,
                 long long* __restrict__ tr, int part, int pw) {
  using Cf = LpCfg<BPB, E>;
  using LE = LpE<E>;
  constexpr int CPB = LE::CPB, NBOX = lp::KC / CPB, BOXE = lp::R * CPB;
  constexpr int NT = Cf::NT;
  using namespace lp;
  if (st->stop) return;
  // part < 0: the block's b' columns if b' falls in this bucket.  part >= 0 (b' > 32): the
  // balanced part [r0, r0 + cnt) of Q_b's rows (part_range, <= 32); the parts run in order, each
  // on the residual the previous one left (Q_b's rows are orthonormal, so the sequence
  // equals one projection up to rounding; the paper form downdates per part).
  int bp;
  int64_t k0;
  if (part < 0) {
    bp = st->b_prime;
    if (bp <= 0 || bucket_of(bp) != BPB) return;
    k0 = st->k;
  } else {
    int r0;
    if (!part_range(st->b_prime, part, &r0, &bp, pw) || bucket_of(bp) != BPB) return;
    k0 = st->k + r0;
  }
  // DMMA work only for the 8-column groups that hold a column of Q_b (warp-uniform)
  const int ntr = (bp + 7) >> 3;
  if (blockIdx.x == 0 && threadIdx.x == 0 && part <= 0) st->ts0 = gtimer();

  extern __shared__ __align__(1024) double sm_raw[];
  double* sm = sm_raw + ((1024u - (lp_su32(sm_raw) & 1023u)) & 1023u) / 8;
  E* xs = reinterpret_cast<E*>(sm);                  // NS x SLOT elements of E
  double* qs = reinterpret_cast<double*>(xs + (size_t)NS * SLOT);   // NQ x QSTAGE
  double* scr = qs + (size_t)NQ * Cf::QSTAGE;        // [rp][slot 0..1][ACC][32]
  double* nrm = scr + Cf::SCR;                       // [tile parity][rp][cw][16] row-norm partials
  uint64_t* xfull = reinterpret_cast<uint64_t*>(nrm + 2 * NRP * NCW * 16);
  uint64_t* xempty = xfull + NS;
  uint64_t* qfull = xempty + NS;
  uint64_t* qempty = qfull + NQ;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t ntiles = (n + R - 1) / R;
  const int T = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  if (T == 0) {
    proj_end_stamp(st);
    return;
  }
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

  if (w >= NCONS) {
    if (w == NCONS && lane == 0) {
      // X producer.  Residual form: the L-hat pass loads a tile with an L2 evict_last
      // policy, the update pass (same addresses, shortly after) with evict_first, so the
      // second read is served by L2 and HBM sees one read of X_res.
      // Lazy X_res copy: block 1 reads the input X (xmap0); the update pass writes X_res.
      const CUtensorMap* mp = (lazy && st->t == 1 && part <= 0) ? &xmap0 : &xmap;
      uint64_t pol_keep, pol_drop;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_keep));
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_drop));
      LpRing xr;
      for (int s = 0; s < steps; ++s) {
        if (s >= NS) lp_wait(&xempty[xr.i], xr.ph ^ 1);
        const int y = (int)row0_of(s / (nc * npass)), c = s % nc;
        const bool second = resid && ((s / nc) & 1);
        lp_expect(&xfull[xr.i], Cf::SLOTB);   // out-of-bounds rows / columns are zero-filled
        E* dst = xs + (size_t)xr.i * SLOT;
        const uint64_t pol = resid ? (second ? pol_drop : pol_keep) : pol_drop;
#pragma unroll
        for (int b = 0; b < NBOX; ++b)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
              "[%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(lp_su32(dst + b * BOXE)),
              "l"(mp), "r"(c * KC + CPB * b), "r"(y), "r"(lp_su32(&xfull[xr.i])), "l"(pol)
              : "memory");
        xr.next(NS);
      }
    } else if (w == NCONS + 1 && lane == 0) {
      // Q producer: packed Q_b chunk c (image 2, row pairs, for the update pass)
      LpRing qr;
      for (int s = 0; s < steps; ++s) {
        if (s >= NQ) lp_wait(&qempty[qr.i], qr.ph ^ 1);
        lp_expect(&qfull[qr.i], (uint32_t)(Cf::QSTAGE * 8));
        const int in = s % (nc * npass);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                lp_su32(qs + (size_t)qr.i * Cf::QSTAGE)),
            "l"(Qp + (in >= nc ? (size_t)nc * PACK_ROWS * KC : 0) + (size_t)(in % nc) * PACK_ROWS * KC),
            "r"((uint32_t)(Cf::QSTAGE * 8)), "r"(lp_su32(&qfull[qr.i]))
            : "memory");
        qr.next(NQ);
      }
    }
    __syncwarp();
  } else {
    // operands of the step consumed (they fed issued MMAs): release both buffers
    // 32-bit shared addresses, computed once
    const uint32_t xs_s = lp_su32(xs), qs_s = lp_su32(qs);
    const uint32_t xf_s = lp_su32(xfull), xe_s = lp_su32(xempty), qf_s = lp_su32(qfull), qe_s = lp_su32(qempty);
    auto release = [&](int xi, int qi) {
      __syncwarp();
      if (lane == 0) {
        lp_arrives(xe_s + 8 * xi);
        lp_arrives(qe_s + 8 * qi);
      }
    };
    // consumers: warp = (row pair rp, column group cw)
    const int rp = w >> 2, cw = w & 3;
    const int g = lane >> 2, q = lane & 3;
    // optional cycle trace of CTA 0 (RBRP_LP_TRACE=1; profiling only): per warp and tile
    // 8 events, then per warp and chunk step the time its operands were ready
#if LP_TRACE
    int sidx = 0;
    long long* trw = (tr && blockIdx.x == 0 && lane == 0) ? tr + w * 64 : nullptr;
    long long* trs = (tr && blockIdx.x == 0 && lane == 0) ? tr + 1024 + w * 256 : nullptr;
#define LP_T(e)                                                   \
  do {                                                            \
    if (trw && p < 8) trw[p * 8 + (e)] = clock64();               \
  } while (0)
#define LP_TS()                                                   \
  do {                                                            \
    if (trs && sidx < 256) trs[sidx++] = clock64();               \
  } while (0)
#else
#define LP_T(e)
#define LP_TS()
#endif
    const int pg = LE::pg(g);                // tile row of MMA row g (bank-conflict-free)
    int xo[2][2];                            // [row group][8-column half]
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int h = 0; h < 2; ++h) xo[r][h] = lp_xoff_e<E>(16 * rp + 8 * r + pg, 16 * cw + 8 * h + 2 * q);
    double2 acc[2][NT];
    LpRing qr, xr;
    for (int p = 0; p < T; ++p) {
      LP_T(0);
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[r][t] = make_double2(0.0, 0.0);
      for (int c = 0; c < nc; ++c) {
        lp_waits(qf_s + 8 * qr.i, qr.ph);
        lp_waits(xf_s + 8 * xr.i, xr.ph);
        LP_TS();
        const uint32_t xsl = xs_s + xr.i * Cf::SLOTB;
        const uint32_t Qs = qs_s + qr.i * (Cf::QSTAGE * 8);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double2 a0 = LE::ld2(xsl + (int)sizeof(E) * xo[0][h]);
          const double2 a1 = LE::ld2(xsl + (int)sizeof(E) * xo[1][h]);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (t < ntr) {
              const int j = 8 * t + g;
              const double2 b = lp_lds2s(Qs + 8 * (j * KC + lp_qswz(j, 16 * cw + 8 * h + 2 * q)));
              lp_dmma(acc[0][t], a0.x, b.x);
              lp_dmma(acc[1][t], a1.x, b.x);
              lp_dmma(acc[0][t], a0.y, b.y);
              lp_dmma(acc[1][t], a1.y, b.y);
            }
          }
        }
        release(xr.i, qr.i);
        xr.next(NS);
        qr.next(NQ);
      }
      // tile end: P = (c0 + c2) + (c1 + c3) per row pair, in registers of the cw = 0 warp
      LP_T(1);
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
      LP_T(2);
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
      LP_T(3);
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
              if (j < bp) L[row * ldl + k0 + j] = (E)vx;
              if (j + 1 < bp) L[row * ldl + k0 + j + 1] = (E)vy;
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
            if (q == 0 && row < n && dvec) dvec[row] = fmax(dvec[row] - ss, 0.0);   // none: plain GEMM
          }
        }
      }
      if (resid) {
        // ----- update pass (residual form, l.16): X(tile) -= L-hat Q_b, chunk by chunk;
        // the chunks come back through L2 (read from HBM by the L-hat pass just before)
        lp_bar();
        LP_T(4);
        double2 pf[2][NT];   // -P rows of this row pair, accumulator layout (A fragments)
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int t = 0; t < NT; ++t) pf[r][t] = make_double2(LP_S(0, r, t, 0), LP_S(0, r, t, 1));
        const int64_t r0 = row0_of(p) + 16 * rp;
        double nr[2] = {0.0, 0.0};
        // this lane's two rows (MMA rows g of the two 8-row groups) and columns 2q, 2q+1 of
        // its two 8-column halves; padding rows / columns were zero-filled by TMA, so they
        // add nothing to the norms
        const bool v0 = r0 + pg < n, v1 = r0 + 8 + pg < n;
        E* xp = Xr + (r0 + pg) * ldx + 16 * cw + 2 * q;
        const int64_t l8 = 8 * ldx;
        for (int c = 0; c < nc; ++c) {
          lp_waits(qf_s + 8 * qr.i, qr.ph);
          lp_waits(xf_s + 8 * xr.i, xr.ph);
          LP_TS();
          const uint32_t xsl = xs_s + xr.i * Cf::SLOTB;
          const uint32_t Qs = qs_s + qr.i * (Cf::QSTAGE * 8);
          double2 xv[2][2];
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int h = 0; h < 2; ++h) xv[r][h] = LE::ld2(xsl + (int)sizeof(E) * xo[r][h]);
          // B fragments from the pair image: (Q(j0, col), Q(j0 + 1, col)), j0 = 8t + 2q, in
          // one 16-byte load, one t ahead; the four accumulator chains interleaved in issue
          // order (volatile: ptxas would otherwise run them two at a time)
          const uint32_t qb = Qs + 16 * (q * KC + ((16 * cw + g) ^ (2 * q)));
          double2 bb[2], bn[2];
          bb[0] = lp_lds2s(qb);
          bb[1] = lp_lds2s(qb + 128);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (t >= ntr) break;
            if (t + 1 < NT) {
              bn[0] = lp_lds2s(qb + 16 * 4 * KC * (t + 1));
              bn[1] = lp_lds2s(qb + 16 * 4 * KC * (t + 1) + 128);
            }
            lp_dmma_v(xv[0][0], pf[0][t].x, bb[0].x);
            lp_dmma_v(xv[1][0], pf[1][t].x, bb[0].x);
            lp_dmma_v(xv[0][1], pf[0][t].x, bb[1].x);
            lp_dmma_v(xv[1][1], pf[1][t].x, bb[1].x);
            lp_dmma_v(xv[0][0], pf[0][t].y, bb[0].y);
            lp_dmma_v(xv[1][0], pf[1][t].y, bb[0].y);
            lp_dmma_v(xv[0][1], pf[0][t].y, bb[1].y);
            lp_dmma_v(xv[1][1], pf[1][t].y, bb[1].y);
            if (t + 1 < NT) {
              bb[0] = bn[0];
              bb[1] = bn[1];
            }
          }
          release(xr.i, qr.i);
          xr.next(NS);
          qr.next(NQ);
          E* xc = xp + c * KC;
          if (c * KC + KC <= d) {
            if (v0) {
              LE::st2(xc, xv[0][0]);
              LE::st2(xc + 8, xv[0][1]);
            }
            if (v1) {
              LE::st2(xc + l8, xv[1][0]);
              LE::st2(xc + l8 + 8, xv[1][1]);
            }
          } else {   // ragged last chunk (d even: a column pair is in or out as a whole)
            const int col = c * KC + 16 * cw + 2 * q;
            if (v0 && col < d) LE::st2(xc, xv[0][0]);
            if (v0 && col + 8 < d) LE::st2(xc + 8, xv[0][1]);
            if (v1 && col < d) LE::st2(xc + l8, xv[1][0]);
            if (v1 && col + 8 < d) LE::st2(xc + l8 + 8, xv[1][1]);
          }
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int h = 0; h < 2; ++h) {   // norms of the stored (rounded) residual
              const double2 u = LE::rnd(xv[r][h]);
              nr[r] += u.x * u.x + u.y * u.y;
            }
        }
        LP_T(5);
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
        LP_T(6);
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
      LP_T(7);
    }
#undef LP_T
#undef LP_TS
  }
  proj_end_stamp(st);
}

// ------------------------------------------------------------------------------------
// k_lhat64: the same two passes for 32 < b' <= 64 columns of Q_b in ONE pass over X
// (fp64).  k_lhat_paper's K-split warps would hold 2 x 64 accumulator columns per row pair
// (and the update pass the whole -P row block) in registers; here the warps split N:
// warp (rp, cw) computes L-hat(16 rows of rp, Q_b rows 16 cw .. 16 cw + 15) over every
// column of each chunk, so a lane holds 8 accumulator doubles and no K fold is needed.
// At the tile end each warp writes its block of -L-hat into a shared 64 x 64 tile P_s
// (16-byte units XOR-swizzled by row); the update pass reads its A fragments (-P of its
// 16 rows, all b' columns) from P_s and its B fragments from the pair image, as
// k_lhat_paper's update pass does.  Rings: 3 X slots, 2 Q stages of 32 KB (227 KB).
// The summation order of every output (L-hat: chunk by chunk, 8-column groups in order,
// x then y halves; update: t in order) is fixed: bitwise reproducible.
namespace lp64 {
constexpr int BPB = 64, NT = 2;              // Q_b rows per warp column group: 2 x 8
constexpr int QSTAGE = BPB * lp::KC;         // doubles per Q stage
constexpr int PS = lp::R * BPB;              // doubles of the -P tile
constexpr int NRM = 2 * lp::NRP * lp::NCW * 16;
__host__ __device__ constexpr size_t smem(int ns, int nq) {
  return (size_t)ns * lp::SLOT * 8 + (size_t)nq * QSTAGE * 8 + (size_t)(PS + NRM) * 8 + (2 * ns + 2 * nq) * 8 +
         1024;
}
}  // namespace lp64

__global__ void __launch_bounds__(lp::NTH, 1)
    k_lhat64(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap xmap0, int lazy,
             const double* __restrict__ Qp, double* __restrict__ L, int64_t ldl, int64_t n, int d, int nc,
             int NS, int NQ, double* __restrict__ dvec, DevState* st, double* __restrict__ Xr, int64_t ldx,
             int resid, int part, int pw, int bkt) {
  using LE = LpE<double>;
  constexpr int CPB = LE::CPB, NBOX = lp::KC / CPB, BOXE = lp::R * CPB;
  using namespace lp;
  using lp64::NT;
  if (st->stop) return;
  int bp;
  int64_t k0;
  if (part < 0) {
    bp = st->b_prime;
    if (bp <= 0 || bucket_of(bp) != bkt) return;
    k0 = st->k;
  } else {
    int r0;
    if (!part_range(st->b_prime, part, &r0, &bp, pw) || bucket_of(bp) != bkt) return;
    k0 = st->k + r0;
  }
  const int ntr = (bp + 7) >> 3;   // 8-row groups of Q_b that hold a row (<= 8)
  if (blockIdx.x == 0 && threadIdx.x == 0 && part <= 0) st->ts0 = gtimer();

  extern __shared__ __align__(1024) double sm_raw[];
  double* sm = sm_raw + ((1024u - (lp_su32(sm_raw) & 1023u)) & 1023u) / 8;
  double* xs = sm;                                    // NS x SLOT
  double* qs = xs + (size_t)NS * SLOT;                // NQ x QSTAGE
  double* ps = qs + (size_t)NQ * lp64::QSTAGE;        // -P: [64 rows][32 units of 2], swizzled
  double* nrm = ps + lp64::PS;                        // [tile parity][rp][cw][16]
  uint64_t* xfull = reinterpret_cast<uint64_t*>(nrm + lp64::NRM);
  uint64_t* xempty = xfull + NS;
  uint64_t* qfull = xempty + NS;
  uint64_t* qempty = qfull + NQ;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t ntiles = (n + R - 1) / R;
  const int T = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  if (T == 0) {
    proj_end_stamp(st);
    return;
  }
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
  const int npass = resid ? 2 : 1;
  const int steps = T * nc * npass;

  if (w >= NCONS) {
    if (w == NCONS && lane == 0) {   // X producer (as k_lhat_paper)
      const CUtensorMap* mp = (lazy && st->t == 1 && part <= 0) ? &xmap0 : &xmap;
      uint64_t pol_keep, pol_drop;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_keep));
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_drop));
      LpRing xr;
      for (int s = 0; s < steps; ++s) {
        if (s >= NS) lp_wait(&xempty[xr.i], xr.ph ^ 1);
        const int y = (int)row0_of(s / (nc * npass)), c = s % nc;
        const bool second = resid && ((s / nc) & 1);
        lp_expect(&xfull[xr.i], SLOT * 8);
        double* dst = xs + (size_t)xr.i * SLOT;
        const uint64_t pol = resid ? (second ? pol_drop : pol_keep) : pol_drop;
#pragma unroll
        for (int b = 0; b < NBOX; ++b)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
              "[%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(lp_su32(dst + b * BOXE)),
              "l"(mp), "r"(c * KC + CPB * b), "r"(y), "r"(lp_su32(&xfull[xr.i])), "l"(pol)
              : "memory");
        xr.next(NS);
      }
    } else if (w == NCONS + 1 && lane == 0) {   // Q producer: image 1 (L-hat pass), image 2 (update)
      LpRing qr;
      for (int s = 0; s < steps; ++s) {
        if (s >= NQ) lp_wait(&qempty[qr.i], qr.ph ^ 1);
        lp_expect(&qfull[qr.i], (uint32_t)(lp64::QSTAGE * 8));
        const int in = s % (nc * npass);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                lp_su32(qs + (size_t)qr.i * lp64::QSTAGE)),
            "l"(Qp + (in >= nc ? (size_t)nc * PACK_ROWS * KC : 0) + (size_t)(in % nc) * PACK_ROWS * KC),
            "r"((uint32_t)(lp64::QSTAGE * 8)), "r"(lp_su32(&qfull[qr.i]))
            : "memory");
        qr.next(NQ);
      }
    }
    __syncwarp();
  } else {
    const uint32_t xs_s = lp_su32(xs), qs_s = lp_su32(qs), ps_s = lp_su32(ps);
    const uint32_t xf_s = lp_su32(xfull), xe_s = lp_su32(xempty), qf_s = lp_su32(qfull), qe_s = lp_su32(qempty);
    auto release = [&](int xi, int qi) {
      __syncwarp();
      if (lane == 0) {
        lp_arrives(xe_s + 8 * xi);
        lp_arrives(qe_s + 8 * qi);
      }
    };
    const int rp = w >> 2, cw = w & 3;
    const int g = lane >> 2, q = lane & 3;
    const int pg = LE::pg(g);
    // this lane's tile rows (MMA row g of the two 8-row groups) and their swizzle keys
    const int ra = 16 * rp + pg, rb = ra + 8;
    const int sw = ra & 7;   // = rb & 7
    // L-hat pass, X fragments: row ra / rb, columns 8h + 2q of the chunk (h = 0..7):
    // lp_xoff_e(row, 8h + 2q) = (h >> 1) * 1024 + row * 16 + (((4 (h & 1) + q) ^ (row & 7)) * 2)
    const int xa = ra * 16, xb = rb * 16;
    // update pass, X fragments: columns 16 cw + 8 hh + 2q (k_lhat_paper's layout)
    int xo[2][2];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) xo[r][hh] = lp_xoff_e<double>(r ? rb : ra, 16 * cw + 8 * hh + 2 * q);
    // Q image 1 rows of this warp: j = 16 cw + 8 t + g
    int qj[NT], qf[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      qj[t] = 16 * cw + 8 * t + g;
      qf[t] = (8 * (qj[t] & 1)) ^ (4 * ((qj[t] >> 1) & 3));
    }
    const bool on0 = 2 * cw < ntr, on1 = 2 * cw + 1 < ntr;   // warp-uniform
    // L-hat pass work split.  v1 (ntr >= 7): warp (rp, cw) = 2 row groups x the 2 column
    // tiles 2 cw, 2 cw + 1.  v2 (ntr <= 6, where v1 would idle the cw = 3 warps): warp
    // (rg, cg) = 1 row group (8 rows) x column tiles [tb, tb + tn) of a 2-way split of the ntr
    // tiles (at most 3 per warp instead of 4)
    const bool v2 = ntr <= 6;
    const int rg = w >> 1, cg = w & 1, T0 = (ntr + 1) >> 1;
    const int tb = cg ? T0 : 0, tn = cg ? ntr - T0 : T0;   // warp-uniform, tn <= 3
    const int rr = 8 * rg + pg;                          // v2: this lane's tile row
    int qj2[3], qf2[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      qj2[t] = 8 * (tb + t) + g;
      qf2[t] = (8 * (qj2[t] & 1)) ^ (4 * ((qj2[t] >> 1) & 3));
    }
    LpRing qr, xr;
    for (int p = 0; p < T; ++p) {
      double2 acc[2][NT], acc2[3];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[r][t] = make_double2(0.0, 0.0);
#pragma unroll
      for (int t = 0; t < 3; ++t) acc2[t] = make_double2(0.0, 0.0);
      for (int c = 0; c < nc; ++c) {
        lp_waits(qf_s + 8 * qr.i, qr.ph);
        lp_waits(xf_s + 8 * xr.i, xr.ph);
        const uint32_t xsl = xs_s + xr.i * (SLOT * 8);
        const uint32_t Qs = qs_s + qr.i * (lp64::QSTAGE * 8);
        if (v2) {
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            const int cu = 4 * (h & 1) + q, bo = (h >> 1) * 1024;
            const double2 a = lp_lds2s(xsl + 8 * (bo + 16 * rr + ((cu ^ pg) * 2)));
#pragma unroll
            for (int t = 0; t < 3; ++t) {
              if (t < tn) {
                const double2 b = lp_lds2s(Qs + 8 * (qj2[t] * KC + ((8 * h + 2 * q) ^ qf2[t])));
                lp_dmma(acc2[t], a.x, b.x);
                lp_dmma(acc2[t], a.y, b.y);
              }
            }
          }
        } else if (on0) {
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            const int cu = 4 * (h & 1) + q, bo = (h >> 1) * 1024;
            const double2 a0 = lp_lds2s(xsl + 8 * (bo + xa + ((cu ^ sw) * 2)));
            const double2 a1 = lp_lds2s(xsl + 8 * (bo + xb + ((cu ^ sw) * 2)));
            const double2 b0 = lp_lds2s(Qs + 8 * (qj[0] * KC + ((8 * h + 2 * q) ^ qf[0])));
            lp_dmma(acc[0][0], a0.x, b0.x);
            lp_dmma(acc[1][0], a1.x, b0.x);
            lp_dmma(acc[0][0], a0.y, b0.y);
            lp_dmma(acc[1][0], a1.y, b0.y);
            if (on1) {
              const double2 b1 = lp_lds2s(Qs + 8 * (qj[1] * KC + ((8 * h + 2 * q) ^ qf[1])));
              lp_dmma(acc[0][1], a0.x, b1.x);
              lp_dmma(acc[1][1], a1.x, b1.x);
              lp_dmma(acc[0][1], a0.y, b1.y);
              lp_dmma(acc[1][1], a1.y, b1.y);
            }
          }
        }
        release(xr.i, qr.i);
        xr.next(NS);
        qr.next(NQ);
      }
      // tile end: L-hat to L; -L-hat into P_s (residual form) or the l.16 downdate (paper)
      const int64_t r0 = row0_of(p);
      auto put = [&](int trow, int j, double vx, double vy) {   // columns j, j + 1 of row trow
        const int64_t row = r0 + trow;
        if (row < n) {
          if (j < bp) L[row * ldl + k0 + j] = vx;
          if (j + 1 < bp) L[row * ldl + k0 + j + 1] = vy;
        }
        if (resid) {
          const int u = j >> 1;   // 16-byte unit (columns 2u, 2u + 1)
          double* dst = ps + trow * lp64::BPB + 2 * (u ^ (trow & 7));
          dst[0] = -vx;
          dst[1] = -vy;
        }
      };
      double ss[2] = {0.0, 0.0};
      if (v2) {
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          if (t < tn) {
            const double vx = acc2[t].x, vy = acc2[t].y;
            put(rr, 8 * (tb + t) + 2 * q, vx, vy);
            ss[0] += vx * vx + vy * vy;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (!(t ? on1 : on0)) continue;
            const double vx = acc[r][t].x, vy = acc[r][t].y;
            put(r ? rb : ra, 16 * cw + 8 * t + 2 * q, vx, vy);
            ss[r] += vx * vx + vy * vy;
          }
        }
      }
      double* nb = nrm + (size_t)((p & 1) * NRP + rp) * NCW * 16;
      if (!resid) {
        // l.16 downdate (paper form): sum over the row's columns, q lanes then the column
        // groups in order
        if (v2) {
          double* nb2 = nrm + (size_t)(p & 1) * NRP * NCW * 16 + rg * 16;   // [rg][cg][8]
          double v = ss[0];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          if (q == 0) nb2[cg * 8 + pg] = v;
          lp_bar();
          if (cg == 0 && lane < 8 && dvec) {
            const double vv = nb2[lane] + nb2[8 + lane];
            const int64_t row = r0 + 8 * rg + lane;
            if (row < n) dvec[row] = fmax(dvec[row] - vv, 0.0);
          }
        } else {
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            double v = ss[r];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            if (q == 0) nb[cw * 16 + 8 * r + pg] = v;
          }
          lp_bar();
          if (cw == 0 && lane < 16 && dvec) {
            const double v = (nb[lane] + nb[16 + lane]) + (nb[32 + lane] + nb[48 + lane]);
            const int64_t row = r0 + 16 * rp + lane;
            if (row < n) dvec[row] = fmax(dvec[row] - v, 0.0);
          }
        }
      } else {
        lp_bar();   // P_s complete
        // ----- update pass (l.16): X(tile) -= L-hat Q_b, chunk by chunk through L2
        double nr[2] = {0.0, 0.0};
        const bool v0 = r0 + ra < n, v1 = r0 + rb < n;
        double* xp = Xr + (r0 + ra) * ldx + 16 * cw + 2 * q;
        const int64_t l8 = 8 * ldx;
        const uint32_t pa = ps_s + 8 * (ra * lp64::BPB), pb = ps_s + 8 * (rb * lp64::BPB);
        for (int c = 0; c < nc; ++c) {
          lp_waits(qf_s + 8 * qr.i, qr.ph);
          lp_waits(xf_s + 8 * xr.i, xr.ph);
          const uint32_t xsl = xs_s + xr.i * (SLOT * 8);
          const uint32_t Qs = qs_s + qr.i * (lp64::QSTAGE * 8);
          double2 xv[2][2];
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) xv[r][hh] = lp_lds2s(xsl + 8 * xo[r][hh]);
          const uint32_t qb = Qs + 16 * (q * KC + ((16 * cw + g) ^ (2 * q)));
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            if (t >= ntr) break;
            const double2 b0 = lp_lds2s(qb + 16 * 4 * KC * t);
            const double2 b1 = lp_lds2s(qb + 16 * 4 * KC * t + 128);
            const int u = (4 * t + q) ^ sw;
            const double2 fa = lp_lds2s(pa + 16 * u), fb = lp_lds2s(pb + 16 * u);
            lp_dmma_v(xv[0][0], fa.x, b0.x);
            lp_dmma_v(xv[1][0], fb.x, b0.x);
            lp_dmma_v(xv[0][1], fa.x, b1.x);
            lp_dmma_v(xv[1][1], fb.x, b1.x);
            lp_dmma_v(xv[0][0], fa.y, b0.y);
            lp_dmma_v(xv[1][0], fb.y, b0.y);
            lp_dmma_v(xv[0][1], fa.y, b1.y);
            lp_dmma_v(xv[1][1], fb.y, b1.y);
          }
          release(xr.i, qr.i);
          xr.next(NS);
          qr.next(NQ);
          double* xc = xp + c * KC;
          if (c * KC + KC <= d) {
            if (v0) {
              LE::st2(xc, xv[0][0]);
              LE::st2(xc + 8, xv[0][1]);
            }
            if (v1) {
              LE::st2(xc + l8, xv[1][0]);
              LE::st2(xc + l8 + 8, xv[1][1]);
            }
          } else {
            const int col = c * KC + 16 * cw + 2 * q;
            if (v0 && col < d) LE::st2(xc, xv[0][0]);
            if (v0 && col + 8 < d) LE::st2(xc + 8, xv[0][1]);
            if (v1 && col < d) LE::st2(xc + l8, xv[1][0]);
            if (v1 && col + 8 < d) LE::st2(xc + l8 + 8, xv[1][1]);
          }
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) nr[r] += xv[r][hh].x * xv[r][hh].x + xv[r][hh].y * xv[r][hh].y;
        }
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
          const int64_t row = r0 + 16 * rp + lane;
          if (row < n) dvec[row] = v;
        }
      }
      // P_s and nrm are rewritten one tile later (nc chunk steps); the rings keep every warp
      // within max(NS, NQ) steps of the others, so a barrier is only needed for short tiles
      if (nc <= (NS > NQ ? NS : NQ) + 1) lp_bar();
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

static long long* g_lp_trace = nullptr;
static long long* lp_trace_buf() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("RBRP_LP_TRACE");
    on = e && e[0] == '1';
    if (on && cudaMalloc(&g_lp_trace, 5120 * sizeof(long long)) != cudaSuccess) g_lp_trace = nullptr;
    if (g_lp_trace) cudaMemset(g_lp_trace, 0, 5120 * sizeof(long long));
  }
  return g_lp_trace;
}
extern "C" int rbrp_debug_lp_trace(long long* host, int count) {
  if (!g_lp_trace) return -1;
  if (count > 5120) count = 5120;
  return cudaMemcpy(host, g_lp_trace, count * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? count : -1;
}

static int lp_sms() { return device_sms(); }

// TMA: 16-byte aligned base and row stride; fragments read column pairs (d even)
template <typename E>
int lhat_paper_max_bucket_t(const void* X, int64_t ldx, int64_t d) {
  if (d % 2 || d < 16 || (ldx * (int64_t)sizeof(E)) % 16 || ((uintptr_t)X % 16)) return 0;
  int ns, nq, best = 0;
  if (LpCfg<16, E>::rings(ns, nq)) best = 16;
  if (LpCfg<32, E>::rings(ns, nq)) best = 32;
  if (sizeof(E) == 8 && best == 32 && lp64::smem(3, 2) <= (size_t)lp::SMEM_MAX && !getenv("RBRP_NO_LP64")) best = 64;
  return best;
}
int lhat_paper_max_bucket(const void* X, int64_t ldx, int64_t d) { return lhat_paper_max_bucket_t<double>(X, ldx, d); }
int lhat_paper_max_bucket_f32(const void* X, int64_t ldx, int64_t d) {
  return lhat_paper_max_bucket_t<float>(X, ldx, d);
}

template <int BPB, typename E>
static cudaError_t go_lp(const CUtensorMap& map, const CUtensorMap& map0, int lazy, const double* Qp, E* L,
                         int64_t ldl, int64_t n, int64_t d, double* dvec, DevState* st, E* Xr, int64_t ldx,
                         int resid, cudaStream_t s, int part, int pw) {
  using Cf = LpCfg<BPB, E>;
  int ns, nq;
  if (!Cf::rings(ns, nq)) return cudaErrorInvalidValue;
  const size_t smem = Cf::smem(ns, nq);
  cudaFuncSetAttribute(k_lhat_paper<BPB, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int nc = (int)((d + lp::KC - 1) / lp::KC);
  long long* tr = nullptr;
  static int traced = 0;
  if (BPB == 32 && sizeof(E) == 8 && lp_trace_buf() && !traced) {   // first fp64 bucket-32 launch only
    tr = lp_trace_buf();
    traced = 1;
  }
  k_lhat_paper<BPB, E><<<lp_sms(), lp::NTH, smem, s>>>(map, map0, lazy, Qp, L, ldl, n, (int)d, nc, ns, nq, dvec,
                                                        st, Xr, ldx, resid, tr, part, pw);
  return cudaGetLastError();
}

// RBRP_LP64_ALL=1 (experiment): b' <= 32 on k_lhat64 as well.  Measured slower on c2
// (b' = 31: 0.36 vs 0.32 ms per block): the K-split warps of k_lhat_paper<32> stay the default.
static bool lp64_all() {
  const char* e = getenv("RBRP_LP64_ALL");
  return e && e[0] == '1';
}

static cudaError_t go_lp64(const CUtensorMap& map, const CUtensorMap& map0, int lazy, const double* Qp, double* L,
                           int64_t ldl, int64_t n, int64_t d, double* dvec, DevState* st, double* Xr, int64_t ldx,
                           int resid, cudaStream_t s, int part, int pw, int bkt) {
  const int ns = 3, nq = 2;
  const size_t smem = lp64::smem(ns, nq);
  static PerDevice attr;
  const cudaError_t ae = attr.once([smem] {
    return cudaFuncSetAttribute(k_lhat64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (ae != cudaSuccess) return ae;
  const int nc = (int)((d + lp::KC - 1) / lp::KC);
  k_lhat64<<<lp_sms(), lp::NTH, smem, s>>>(map, map0, lazy, Qp, L, ldl, n, (int)d, nc, ns, nq, dvec, st, Xr, ldx,
                                            resid, part, pw, bkt);
  return cudaGetLastError();
}

template <typename E>
static cudaError_t launch_lhat_paper_t(const E* X, int64_t ldx, const double* Qp, E* L, int64_t ldl, int64_t n,
                                       int64_t d, double* dvec, DevState* st, int bucket, bool resid,
                                       cudaStream_t s, const E* X0, int64_t ldx0, int part, int pw) {
  if (n <= 0) return cudaSuccess;
  if (pw <= 0) pw = bucket;
  auto enc = lp_encode();
  if (!enc) return cudaErrorNotSupported;
  auto make_map = [&](const E* P, int64_t ld, CUtensorMap* map) {
    const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(E)};
    const cuuint32_t box[2] = {(cuuint32_t)LpE<E>::CPB, (cuuint32_t)lp::R};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, sizeof(E) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
               (void*)P, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  CUtensorMap map, map0;
  if (!make_map(X, ldx, &map)) return cudaErrorInvalidValue;
  const int lazy = X0 != nullptr ? 1 : 0;
  if (!make_map(lazy ? X0 : X, lazy ? ldx0 : ldx, &map0)) return cudaErrorInvalidValue;
  switch (bucket) {
    case 16:
    case 32:
      // fp64 with RBRP_LP64_ALL=1 (experiment): k_lhat64's split L-hat pass for ntr <= 4 too
      if (sizeof(E) == 8 && lp64_all())
        return go_lp64(map, map0, lazy, Qp, (double*)L, ldl, n, d, dvec, st, (double*)X, ldx, resid ? 1 : 0, s,
                       part, pw, bucket);
      if (bucket == 16)
        return go_lp<16, E>(map, map0, lazy, Qp, L, ldl, n, d, dvec, st, (E*)X, ldx, resid ? 1 : 0, s, part, pw);
      return go_lp<32, E>(map, map0, lazy, Qp, L, ldl, n, d, dvec, st, (E*)X, ldx, resid ? 1 : 0, s, part, pw);
    case 64:
      if (sizeof(E) != 8) return cudaErrorInvalidValue;
      return go_lp64(map, map0, lazy, Qp, (double*)L, ldl, n, d, dvec, st, (double*)X, ldx, resid ? 1 : 0, s, part,
                     pw, 64);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_lhat_paper(const double* X, int64_t ldx, const double* Qp, double* L, int64_t ldl,
                              int64_t n, int64_t d, double* dvec, DevState* st, int bucket, bool resid,
                              cudaStream_t s, const double* X0, int64_t ldx0, int part, int pw) {
  return launch_lhat_paper_t<double>(X, ldx, Qp, L, ldl, n, d, dvec, st, bucket, resid, s, X0, ldx0, part, pw);
}
cudaError_t launch_lhat_paper(const float* X, int64_t ldx, const double* Qp, float* L, int64_t ldl,
                              int64_t n, int64_t d, double* dvec, DevState* st, int bucket, bool resid,
                              cudaStream_t s, const float* X0, int64_t ldx0, int part, int pw) {
  return launch_lhat_paper_t<float>(X, ldx, Qp, L, ldl, n, d, dvec, st, bucket, resid, s, X0, ldx0, part, pw);
}

// ------------------------------------------------------------------------------------
// C = A B^T as a sequence of read-only L-hat passes (the paper-form kernel without a
// downdate), 32 columns of C per launch: every launch streams A once through TMA and
// runs the 64-row-tile DMMA loop that reaches 97% of the DMMA rate (profiles/README).
// Used for W = L L_1^{-1} (Alg. 3) and the SkLUPP-OSID GEMMs.  Each column group gets
// its own DevState (b_prime = group width, k = first column) in the scratch.
// ------------------------------------------------------------------------------------
__global__ void k_gemm_groups(DevState* st, int64_t N, int gw) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g * gw >= N) return;
  DevState z;
  memset(&z, 0, sizeof(z));
  z.k = g * gw;
  z.k_cap = N;
  z.b_prime = (int)(N - g * gw < gw ? N - g * gw : gw);
  z.t = 2;
  st[g] = z;
}

size_t gemm_lp_scratch_bytes(int64_t N, int64_t K) {
  const int64_t G = (N + 31) / 32;
  return ((fused_pack_bytes(K) + 255) & ~(size_t)255) + (size_t)G * sizeof(DevState);
}

// min_k: k_lhat_paper's per-tile fold of the 4-way K split needed K >= 512 to beat
// k_nt_mma; the 64-column groups on k_lhat64 (no fold) win from K = 128 (scripts/w_bench.py)
template <typename E>
static int lp_max_bucket_e(const E* A, int64_t lda, int64_t K) {
  return sizeof(E) == 8 ? lhat_paper_max_bucket(A, lda, K) : lhat_paper_max_bucket_f32(A, lda, K);
}

template <typename E>
static bool gemm_lp_supported_t(const E* A, int64_t lda, const E* B, int64_t ldb, int64_t K, int64_t min_k) {
  return K >= min_k && lp_max_bucket_e(A, lda, K) >= 32 && ldb == K && ((uintptr_t)B % 16) == 0;
}
bool gemm_lp_supported(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t K, int64_t min_k) {
  return gemm_lp_supported_t(A, lda, B, ldb, K, min_k);
}
bool gemm_lp_supported(const float* A, int64_t lda, const float* B, int64_t ldb, int64_t K, int64_t min_k) {
  return gemm_lp_supported_t(A, lda, B, ldb, K, min_k);
}

// fp32 storage: k_lhat_paper<32, float> groups (fp64 DMMA arithmetic on the fp32 values,
// the result rounded once to fp32)
template <typename E>
static cudaError_t gemm_nt_lp_t(const E* A, int64_t lda, const E* B, int64_t ldb, E* C, int64_t ldc, int64_t M,
                                int64_t N, int64_t K, void* scratch, cudaStream_t s, bool lower_b, int64_t min_k,
                                int* nlaunch) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (!gemm_lp_supported_t(A, lda, B, ldb, K, min_k)) return cudaErrorNotSupported;
  double* Qp = (double*)scratch;
  DevState* st = (DevState*)((char*)scratch + ((fused_pack_bytes(K) + 255) & ~(size_t)255));
  // groups of 64 columns of C on k_lhat64 (one read of A per 64 columns), else 32
  const int gw = (lp_max_bucket_e(A, lda, K) >= 64 && !getenv("RBRP_GEMM_GW32")) ? 64 : 32;
  const int64_t G = (N + gw - 1) / gw;
  k_gemm_groups<<<(unsigned)((G + 127) / 128), 128, 0, s>>>(st, N, gw);
  if (nlaunch) *nlaunch += 1 + 2 * (int)G;
  cudaError_t e = cudaGetLastError();
  for (int64_t g = 0; g < G && e == cudaSuccess; ++g) {
    const int bg = (int)(N - gw * g < gw ? N - gw * g : gw);
    const int64_t k0 = lower_b ? (gw * g / lp::KC) * lp::KC : 0;   // B(rows of g, m < k0) = 0
    e = launch_pack_q(B + gw * g * ldb + k0, K - k0, Qp, st + g, s, -1, ldb);
    if (e == cudaSuccess)
      e = launch_lhat_paper(A + k0, lda, Qp, C, ldc, M, K - k0, nullptr, st + g, bucket_of(bg), false, s);
  }
  return e;
}
cudaError_t gemm_nt_lp(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                       int64_t M, int64_t N, int64_t K, void* scratch, cudaStream_t s, bool lower_b, int64_t min_k,
                       int* nlaunch) {
  return gemm_nt_lp_t(A, lda, B, ldb, C, ldc, M, N, K, scratch, s, lower_b, min_k, nlaunch);
}
cudaError_t gemm_nt_lp(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                       int64_t M, int64_t N, int64_t K, void* scratch, cudaStream_t s, bool lower_b, int64_t min_k,
                       int* nlaunch) {
  return gemm_nt_lp_t(A, lda, B, ldb, C, ldc, M, N, K, scratch, s, lower_b, min_k, nlaunch);
}

}  // namespace rbrp
