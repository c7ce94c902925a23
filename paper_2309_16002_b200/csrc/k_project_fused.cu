// k_project_fused.cu — a4 projection as ONE pass over the residual (north_star step 4;
// Alg. 2 l.13 + l.16; the right-looking form of P:523):
//
//     L-hat = X_res Q_b^T        (n x b', written to L[:, k : k+b'])
//     X_res <- X_res - L-hat Q_b ,   d(i) = ||x_res,i||^2 (fp64)
//
// Every residual element is read from HBM once and written once per block; the two
// products run on the FP64 tensor path (DMMA, mma.sync.m8n8k4.f64 — tcgen05 has no f64
// kind on sm_100a).
//
// Schedule (persistent, one CTA per SM, tiles of R = 16 rows x the full width d):
//   The tile's rows stay in shared memory between the two products.  The width is cut
//   into KC = 64-column chunks; pass p walks the chunks c = 0..nc-1 once and, at every
//   chunk, does
//     phase 2 (tile p-1):  X(p-1)[:, c] -= P(p-1) Q_b[:, c]^T, write it out, norms
//     phase 1 (tile p):    P(p) += X(p)[:, c] Q_b[:, c]^T
//   so each Q_b chunk is fetched from L2 once per tile and serves both products.
//   P(p) is complete at the end of pass p and drives phase 2 of pass p+1.
//
// Shared memory: a ring of NS = nc + E chunk slots (16 rows x 64 doubles, TMA 128-byte
// swizzle) holds the current tile plus E chunks of look-ahead; an NQ-stage ring holds
// Q_b chunks (pre-packed in global by k_pack_q in their shared-memory image, one 1-D
// bulk copy each).  A producer warp fills both on mbarrier full/empty pairs; 8 consumer
// warps own 8 columns of every chunk each.  Phase 1 splits K over the warps; the 8
// partial P tiles are reduced in a fixed order (bitwise reproducible) once per pass.
//
// Bank-conflict-free fragment loads without padding:
//   X: MMA row g of an 8-row group is tile row pi(g) = (g >> 1) + 4 (g & 1), so the two
//      rows of every 8-lane 16-byte phase land in opposite halves of the 128-byte swizzle.
//   Q: column c of row j is stored at c ^ f(j), f(j) = 8 (j & 1) ^ 4 ((j >> 1) & 3),
//      conflict-free for the phase-1 (16-byte, row = n index) and phase-2 (8-byte,
//      row = k index) B-fragment patterns.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "launch.cuh"

namespace rbrp {

namespace fz {
constexpr int R = 16;      // rows per tile (two 8-row MMA groups)
constexpr int KC = 64;     // columns per chunk
constexpr int NW = 8;      // consumer warps (warp w owns columns [8w, 8w+8) of a chunk)
constexpr int NTH = (2 * NW + 3) * 32;   // 8 phase-1 + 8 phase-2 + X-load, Q-load, X-store warps
constexpr int PACK_ROWS = 64;   // rows of the packed Q_b buffer (largest fused bucket)
constexpr int SLOT = R * KC;    // doubles per X slot (4 TMA boxes of 16 x 16)
constexpr int SMEM_MAX = 232448;
#ifndef FZ_XPF
#define FZ_XPF 0
#endif
constexpr int XPF = FZ_XPF;          // L2 prefetch distance of X chunks (steps)
}  // namespace fz

// not volatile: the compiler may schedule the MMAs (they have register outputs)
__device__ __forceinline__ void dmma_f(double2& d, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d.x), "+d"(d.y)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
// consumer release: relaxed (does not wait for this thread's earlier global stores to
// drain).  Callers place it after the instructions that consume the shared-memory
// operands, so the reads are complete before the producer can refill the buffer.
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* b) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(su32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map),
               "r"(x), "r"(y), "r"(su32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(map), "r"(x), "r"(y)
               : "memory");
}
// explicit 16-byte shared-memory accesses (the compiler may otherwise split them)
__device__ __forceinline__ double2 lds2(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(su32(p)));
  return v;
}
__device__ __forceinline__ void sts2(double* p, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(su32(p)), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void bar_p1() { asm volatile("bar.sync 1, %0;\n" ::"n"(fz::NW * 32) : "memory"); }
__device__ __forceinline__ void bar_p1x() { asm volatile("bar.sync 3, %0;\n" ::"n"(2 * fz::NW * 32) : "memory"); }
__device__ __forceinline__ void bar_p2() { asm volatile("bar.sync 2, %0;\n" ::"n"(fz::NW * 32) : "memory"); }

// Q_b chunk layout (shared-memory image): row j, column c at j * 64 + (c ^ f(j))
__host__ __device__ __forceinline__ int qswz(int j, int col) {
  return col ^ (8 * (j & 1)) ^ (4 * ((j >> 1) & 3));
}
// X slot (TMA SWIZZLE_128B, boxes of 16 rows x 16 doubles): row, column (even) -> offset
__device__ __forceinline__ int xoff(int row, int col) {
  return (col >> 4) * 256 + row * 16 + ((((col & 15) >> 1) ^ (row & 7)) << 1);
}
__device__ __forceinline__ int pi_row(int g) { return (g >> 1) + 4 * (g & 1); }

// part < 0: rows [0, b'), b' <= 64.  part >= 0 (b' > 32 split into 32-row parts, see
// launch_lhat_paper): rows [32 part, min(b', 32 part + 32)).
template <typename QT>
__global__ void k_pack_q(const QT* __restrict__ Qt, int64_t d, double* __restrict__ Qp,
                         const DevState* st, int part, int64_t ldq) {
  if (st->stop) return;
  const int bpa = st->b_prime;
  int bp, r0 = 0;
  if (part < 0) {
    bp = bpa;
    if (bp <= 0 || bp > fz::PACK_ROWS) return;
  } else {
    r0 = 32 * part;
    bp = bpa - r0 < 32 ? bpa - r0 : 32;
    if (bpa <= 32 || bp <= 0) return;
  }
  const int c = blockIdx.x, j = blockIdx.y, col = threadIdx.x;   // blockDim = KC
  const int64_t gc = (int64_t)c * fz::KC + col;
  const double v = (j < bp && gc < d) ? (double)Qt[(int64_t)(r0 + j) * ldq + gc] : 0.0;
  Qp[((int64_t)c * fz::PACK_ROWS + j) * fz::KC + qswz(j, col)] = v;
  // second image (update pass of k_lhat_paper): rows in pairs, (Q(2p, col), Q(2p+1, col))
  // adjacent, 16-byte unit of pair p and column col at p * KC + (col ^ 2 (p & 3))
  const int pr = j >> 1;
  double* Q2 = Qp + (int64_t)gridDim.x * fz::PACK_ROWS * fz::KC + (int64_t)c * fz::PACK_ROWS * fz::KC;
  Q2[(pr * fz::KC + (col ^ (2 * (pr & 3)))) * 2 + (j & 1)] = v;
}

template <int BPB>
struct FzCfg {
  static constexpr int NT = BPB / 8;            // 8-column output tiles of P
  static constexpr int ACC = 2 * NT * 2;        // doubles of one warp-lane's P partial
  static constexpr int QSTAGE = BPB * fz::KC;   // doubles per Q stage
  static constexpr int FIXED = (6 * 32 * ACC + 2 * fz::NW * fz::R) * 8 + 2048 + 64;   // scratch, P, norms, align
  static size_t smem(int ns, int nq) {
    return (size_t)FIXED + (size_t)ns * fz::SLOT * 8 + (size_t)nq * QSTAGE * 8 + (3 * ns + 2 * nq) * 8;
  }
  // ring sizes: X slots NS = nc + E and Q stages NQ.  Look-ahead is split between the two
  // rings (E >= 2, NQ >= 2), then grown alternately while shared memory lasts.  Returns
  // false if not even E = NQ = 2 fits.
  static bool rings(int nc, int& ns, int& nq, bool paper = false) {
    if (paper) {   // streaming X ring (no tile residency): fixed look-ahead
      ns = 12;
      nq = 5;
      while (smem(ns, nq) > (size_t)fz::SMEM_MAX && ns > 4) --ns;
      return smem(ns, nq) <= (size_t)fz::SMEM_MAX;
    }
    const char* ee = getenv("RBRP_FZ_E");
    const char* eq = getenv("RBRP_FZ_NQ");
    int e = 2;
    nq = 2;
    if (smem(nc + e, nq) > (size_t)fz::SMEM_MAX) return false;
    for (int it = 0; it < 16; ++it) {
      const bool grow_q = (nq <= e - 1);
      int e2 = e + (grow_q ? 0 : 1), q2 = nq + (grow_q ? 1 : 0);
      if (q2 > 6) { q2 = nq; e2 = e + 1; }
      if (e2 > 8) break;
      if (smem(nc + e2, q2) > (size_t)fz::SMEM_MAX) break;
      e = e2;
      nq = q2;
    }
    if (ee) e = atoi(ee);
    if (eq) nq = atoi(eq);
    ns = nc + e;
    return smem(ns, nq) <= (size_t)fz::SMEM_MAX && e >= 1 && nq >= 2;
  }
};

// ring position with its mbarrier phase parity
struct Ring {
  int i = 0, ph = 0;
  __device__ __forceinline__ void next(int n) {
    if (++i == n) {
      i = 0;
      ph ^= 1;
    }
  }
};

// Warp roles (NW = 8 per group): warps [0, 8) phase 1 (P += X Q^T, K split over the
// warps), warps [8, 16) phase 2 (X -= P Q, norms, L-hat rows), warp 16 the producer.
// Four consumer warps per SM sub-partition hide each other's per-chunk overhead.
template <int BPB>
__global__ void __launch_bounds__(fz::NTH, 1)
    k_proj_fused(const __grid_constant__ CUtensorMap xmap, double* __restrict__ X, int64_t ldx,
                 const double* __restrict__ Qp, double* __restrict__ L, int64_t ldl, int64_t n, int d,
                 int nc, int NS, int NQ, double* __restrict__ dvec, DevState* st, long long* trace, int xmode,
                 int paper) {
  using Cf = FzCfg<BPB>;
  constexpr int NT = Cf::NT;
  using namespace fz;
  if (st->stop) return;
  const int bp = st->b_prime;
  if (bp <= 0 || bucket_of(bp) != BPB) return;
  const int64_t k0 = st->k;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->ts0 = gtimer();

  extern __shared__ __align__(1024) double sm_raw[];
  // the 128-byte swizzle pattern repeats every 1 KB: align the X ring to 1 KB (pointer
  // arithmetic on sm_raw keeps the shared address space: LDS, not generic loads)
  double* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u) / 8;
  double* xs = sm;                                   // NS x SLOT
  double* qs = xs + (size_t)NS * SLOT;               // NQ x QSTAGE
  double* scr = qs + NQ * Cf::QSTAGE;                // 4 x ACC x 32
  double* pbuf = scr + 4 * 32 * Cf::ACC;             // 2 x ACC x 32: -P per pass parity
  double* nrm = pbuf + 2 * 32 * Cf::ACC;             // 2 x NW x R (pass parity)
  uint64_t* xfull = reinterpret_cast<uint64_t*>(nrm + 2 * NW * R);
  uint64_t* xempty = xfull + NS;
  uint64_t* qfull = xempty + NS;
  uint64_t* qempty = qfull + NQ;
  uint64_t* xdone = qempty + NQ;                     // [NS]: phase 2 has updated the slot
  uint64_t* pready = xdone + NS;                     // [2]: -P(p) in pbuf[p & 1]
  uint64_t* pfree = pready + 2;                      // [2]: phase-2 warps have read it

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t ntiles = (n + R - 1) / R;
  const int T = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], paper ? NW : 1);   // store warp once written back (paper: phase 1)
      mbar_init(&xdone[s], NW);          // phase-2 warps: updated chunk is in the slot
    }
    for (int s = 0; s < NQ; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], paper ? NW : 2 * NW);   // released by every consumer warp
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&pready[s], NW);
      mbar_init(&pfree[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  auto row0_of = [&](int p) { return ((int64_t)blockIdx.x + (int64_t)p * gridDim.x) * R; };
  const int g = lane >> 2, q = lane & 3;
  const int pg = pi_row(g);            // tile row of MMA row g (within an 8-row group)
  // optional cycle trace of CTA 0 (RBRP_FZ_TRACE=1; profiling only)
  long long* tr = (trace && blockIdx.x == 0) ? trace : nullptr;
  constexpr int TRN = 512;
#define FZ_S(slot, r, t, h) scr[((slot) * Cf::ACC + ((r) * NT + (t)) * 2 + (h)) * 32 + lane]

  if (T == 0) {
  } else if (w == 2 * NW) {
    // ---------------------------- X producer warp ----------------------------
    // X(sx) reuses the slot the phase-2 warps free at step sx - E
    if (lane == 0) {
      const int xsteps = T * nc;
      int xp = 0, xc = 0;
      Ring xr;
      for (int s2 = 0; s2 < XPF && s2 < xsteps; ++s2) {
        const int y2 = (int)row0_of(s2 / nc);
#pragma unroll
        for (int b = 0; b < 4; ++b) tma_prefetch_2d(&xmap, (s2 % nc) * KC + 16 * b, y2);
      }
      for (int sx = 0; sx < xsteps; ++sx) {
        if (sx >= NS) mbar_wait(&xempty[xr.i], xr.ph ^ 1);
        if (tr && sx < TRN) tr[sx] = clock64();
        mbar_expect_tx(&xfull[xr.i], SLOT * 8);   // out-of-bounds elements are zero-filled
        double* dst = xs + (size_t)xr.i * SLOT;
        const int y = (int)row0_of(xp);
#pragma unroll
        for (int b = 0; b < 4; ++b) tma_2d(dst + b * 256, &xmap, xc * KC + 16 * b, y, &xfull[xr.i]);
        if (sx + XPF < xsteps) {   // the chunk XPF steps ahead into L2
          const int s2 = sx + XPF;
          const int y2 = (int)row0_of(s2 / nc);
#pragma unroll
          for (int b = 0; b < 4; ++b) tma_prefetch_2d(&xmap, (s2 % nc) * KC + 16 * b, y2);
        }
        xr.next(NS);
        if (++xc == nc) {
          xc = 0;
          ++xp;
        }
      }
    }
    __syncwarp();
  } else if (w == 2 * NW + 1) {
    // ---------------------------- Q producer warp ----------------------------
    // Q(sq) reuses the stage every consumer warp frees at step sq - NQ
    if (lane == 0) {
      const int qsteps = (T + (paper ? 0 : 1)) * nc;
      Ring qr;
      for (int sq = 0; sq < qsteps; ++sq) {
        if (sq >= NQ) mbar_wait(&qempty[qr.i], qr.ph ^ 1);
        if (tr && sq < TRN) tr[TRN + sq] = clock64();
        mbar_expect_tx(&qfull[qr.i], (uint32_t)(Cf::QSTAGE * 8));
        bulk_g2s(qs + qr.i * Cf::QSTAGE, Qp + (size_t)(sq % nc) * PACK_ROWS * KC, (uint32_t)(Cf::QSTAGE * 8),
                 &qfull[qr.i]);
        qr.next(NQ);
      }
    }
    __syncwarp();
  } else if (w == 2 * NW + 2) {
    // ---------------------------- X store warp -----------------------------
    // writes each updated chunk back with TMA (full 128-byte lines, no per-thread
    // stores on the phase-2 warps), then hands the slot to the X producer
    if (lane == 0 && !paper) {
      const int xsteps = T * nc;
      int xp = 0, xc = 0;
      Ring xr;
      for (int s2 = 0; s2 < xsteps; ++s2) {
        mbar_wait(&xdone[xr.i], xr.ph);
        const double* src = xs + (size_t)xr.i * SLOT;
        const int y = (int)row0_of(xp);
        if (!(xmode & 1)) {
#pragma unroll
          for (int b = 0; b < 4; ++b) tma_store_2d(&xmap, src + b * 256, xc * KC + 16 * b, y);
        }
        bulk_commit();
        bulk_wait_read0();   // the slot has been read: it may be refilled
        mbar_arrive(&xempty[xr.i]);
        xr.next(NS);
        if (++xc == nc) {
          xc = 0;
          ++xp;
        }
      }
      bulk_wait0();   // writes complete before the kernel's end stamp
    }
    __syncwarp();
  } else if (w < NW || (paper && w < 2 * NW)) {
    // ------------------------- phase 1: P(p) += X(p) Q^T -------------------------
    // paper form: the phase-2 warps are free, so 16 warps run phase 1 as two sets that
    // take alternate chunks (set = w >> 3); the 16 K-partials are folded in fixed order
    const int set = w >> 3, cw = w & 7, nset = paper ? 2 : 1;
    const int xo0 = xoff(pg, 8 * cw + 2 * q), xo1 = xoff(8 + pg, 8 * cw + 2 * q);
    double2 acc[2][NT];   // acc[r][t] = P[8r+pi(g)][8t+2q+{0,1}] (K-partial of this warp)
    Ring qr, xr;
    const int passes = paper ? T : T + 1;
    for (int p = 0; p < passes; ++p) {
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[r][t] = make_double2(0.0, 0.0);
      const bool ph1 = p < T;
      for (int c = 0; c < nc; ++c) {
        const int stp = p * nc + c;
        const bool trw = tr && w == 0 && lane == 0 && stp < TRN;
        if (nset == 2 && (c & 1) != set) {   // the other set's chunk
          qr.next(NQ);
          xr.next(NS);
          continue;
        }
        mbar_wait(&qfull[qr.i], qr.ph);
        if (trw) tr[2 * TRN + stp] = clock64();
        if (ph1) {
          const double* Qs = qs + qr.i * Cf::QSTAGE;
          mbar_wait(&xfull[xr.i], xr.ph);
          if (trw) tr[3 * TRN + stp] = clock64();
          const double* xsl = xs + (size_t)xr.i * SLOT;
          const double2 a0 = lds2(xsl + xo0);
          const double2 a1 = lds2(xsl + xo1);
          double2 b[NT];
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const int j = 8 * t + g;
            b[t] = lds2(Qs + j * KC + qswz(j, 8 * cw + 2 * q));
          }
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (xmode & 2) {
              acc[0][t].x += a0.x * b[t].x; acc[1][t].y += a1.y * b[t].y;
            } else {
              dmma_f(acc[0][t], a0.x, b[t].x);
              dmma_f(acc[1][t], a1.x, b[t].x);
              dmma_f(acc[0][t], a0.y, b[t].y);
              dmma_f(acc[1][t], a1.y, b[t].y);
            }
          }
          if (trw) tr[11 * TRN + stp] = clock64();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive_relaxed(&qempty[qr.i]);
            if (paper) mbar_arrive_relaxed(&xempty[xr.i]);   // no phase 2: slot done
          }
          if (trw) tr[12 * TRN + stp] = clock64() + (long long)(acc[0][0].x == 1.2345e300);
          xr.next(NS);
        } else {
          __syncwarp();
          if (lane == 0) mbar_arrive_relaxed(&qempty[qr.i]);
        }
        if (trw) tr[4 * TRN + stp] = clock64();
        qr.next(NQ);
      }
      // pass end (phase-1 warps only): fixed-order reduction of the 8 K-partials,
      // -P(p) into pbuf[p & 1] for the phase-2 warps, L-hat rows of tile p (l.13)
      if (ph1) {
        // fold the K-partials into slots 0..3: slot s = acc(s) + acc(s+4) [+ acc(s+8) +
        // acc(s+12)], added from the highest warp down (fixed order)
        const int nw1 = NW * nset;
        for (int top = nw1 - 4; top >= 4; top -= 4) {
          if (w >= top && w < top + 4) {
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
              for (int t = 0; t < NT; ++t) {
                if (top == nw1 - 4) {
                  FZ_S(w - top, r, t, 0) = acc[r][t].x;
                  FZ_S(w - top, r, t, 1) = acc[r][t].y;
                } else {
                  FZ_S(w - top, r, t, 0) = acc[r][t].x + FZ_S(w - top, r, t, 0);
                  FZ_S(w - top, r, t, 1) = acc[r][t].y + FZ_S(w - top, r, t, 1);
                }
              }
          }
          if (nset == 2) bar_p1x(); else bar_p1();
        }
        if (w < 4) {
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              FZ_S(w, r, t, 0) = acc[r][t].x + FZ_S(w, r, t, 0);
              FZ_S(w, r, t, 1) = acc[r][t].y + FZ_S(w, r, t, 1);
            }
        }
        if (nset == 2) bar_p1x(); else bar_p1();
        const int pb = p & 1;
        if (p >= 2 && !paper) mbar_wait(&pfree[pb], ((p >> 1) - 1) & 1);
        double* P = pbuf + pb * Cf::ACC * 32;
        const int64_t r0p = row0_of(p);
#pragma unroll
        for (int cb = 0; cb < Cf::ACC; cb += NW) {   // (r, t, h) combos w, w + 8, ...
          const int combo = cb + w;
          if (w < NW && combo < Cf::ACC) {
            const int i = combo * 32 + lane;
            const double v = (scr[(0 * Cf::ACC) * 32 + i] + scr[(1 * Cf::ACC) * 32 + i]) +
                             (scr[(2 * Cf::ACC) * 32 + i] + scr[(3 * Cf::ACC) * 32 + i]);
            P[i] = paper ? v : -v;
            const int r = combo / (2 * NT), t = (combo >> 1) % NT, h = combo & 1;
            const int j = 8 * t + 2 * q + h;
            const int64_t row = r0p + 8 * r + pg;
            if (j < bp && row < n) L[row * ldl + k0 + j] = v;
          }
        }
        if (paper) {
          // l.16 (paper form): d(i) <- max(0, d(i) - ||L-hat(i,:)||^2), fixed order (t, h, q)
          bar_p1x();
          if (w == 0 && lane < R) {
            const int rr = lane, r = rr >> 3, x = rr & 7;
            const int gg = 2 * (x & 3) + (x >> 2);   // pi^-1
            double ss = 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t)
#pragma unroll
              for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                  const double v = P[((r * NT + t) * 2 + h) * 32 + 4 * gg + qq];
                  ss += v * v;
                }
            const int64_t row = r0p + rr;
            if (row < n) dvec[row] = fmax(dvec[row] - ss, 0.0);
          }
        } else {
          __syncwarp();
          if (lane == 0) mbar_arrive(&pready[pb]);   // release: P stores ordered before
        }
        if (nset == 2) bar_p1x(); else bar_p1();   // scratch is rewritten at the next pass end
      }
    }
  } else {
    // -------------------- phase 2: X(p-1) -= P(p-1) Q, norms --------------------
    if (paper) goto done;   // left-looking form: X is read only
    {
    const int w2 = w - NW;
    const int xo0 = xoff(pg, 8 * w2 + 2 * q), xo1 = xoff(8 + pg, 8 * w2 + 2 * q);
    double2 pf[2][NT];    // -P(p-1) in the accumulator layout (A fragments)
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int t = 0; t < NT; ++t) pf[r][t] = make_double2(0.0, 0.0);
    Ring qr, xr;
    double nr0 = 0.0, nr1 = 0.0;
    for (int p = 0; p <= T; ++p) {
      nr0 = 0.0;
      nr1 = 0.0;
      const int64_t r0m = row0_of(p - 1);
      const bool ph2 = p >= 1;
      for (int c = 0; c < nc; ++c) {
        const int stp = p * nc + c;
        const bool trw = tr && w2 == 0 && lane == 0 && stp < TRN;
        mbar_wait(&qfull[qr.i], qr.ph);
        if (trw) tr[5 * TRN + stp] = clock64();
        if (ph2) {
          const double* Qs = qs + qr.i * Cf::QSTAGE;
          mbar_wait(&xfull[xr.i], xr.ph);   // completed a pass ago (acquire for this warp)
          if (trw) tr[7 * TRN + stp] = clock64();
          double* xsl = xs + (size_t)xr.i * SLOT;
          double2 x0 = lds2(xsl + xo0);
          double2 x1 = lds2(xsl + xo1);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const int j0 = 8 * t + 2 * q;
            const double b0 = Qs[j0 * KC + qswz(j0, 8 * w2 + g)];
            const double b1 = Qs[(j0 + 1) * KC + qswz(j0 + 1, 8 * w2 + g)];
            if (xmode & 4) {
              x0.x += pf[0][t].x * b0; x1.y += pf[1][t].y * b1;
            } else {
              dmma_f(x0, pf[0][t].x, b0);
              dmma_f(x1, pf[1][t].x, b0);
              dmma_f(x0, pf[0][t].y, b1);
              dmma_f(x1, pf[1][t].y, b1);
            }
          }
          if (trw) tr[8 * TRN + stp] = clock64();
          __syncwarp();
          if (lane == 0) mbar_arrive_relaxed(&qempty[qr.i]);   // Q operands consumed
          if (trw) tr[9 * TRN + stp] = clock64();
          // updated residual back into the slot (same conflict-free offsets), made
          // visible to the TMA engine, then handed to the store warp
          sts2(xsl + xo0, x0);
          sts2(xsl + xo1, x1);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&xdone[xr.i]);
          xr.next(NS);
          const int col = c * KC + 8 * w2 + 2 * q;
          if (col < d) {
            if (r0m + pg < n) nr0 += x0.x * x0.x + x0.y * x0.y;
            if (r0m + 8 + pg < n) nr1 += x1.x * x1.x + x1.y * x1.y;
          }
          if (trw) tr[10 * TRN + stp] = clock64();
        } else {
          __syncwarp();
          if (lane == 0) mbar_arrive_relaxed(&qempty[qr.i]);
        }
        if (trw) tr[6 * TRN + stp] = clock64();
        qr.next(NQ);
      }
      // pass end
      double* nb = nrm + (p & 1) * NW * R;
      if (ph2) {   // row norms of tile p-1 over this warp's columns: lanes q = 0
        nr0 += __shfl_xor_sync(0xffffffffu, nr0, 1);
        nr0 += __shfl_xor_sync(0xffffffffu, nr0, 2);
        nr1 += __shfl_xor_sync(0xffffffffu, nr1, 1);
        nr1 += __shfl_xor_sync(0xffffffffu, nr1, 2);
        if (q == 0) {
          nb[w2 * R + pg] = nr0;
          nb[w2 * R + 8 + pg] = nr1;
        }
      }
      bar_p2();
      if (ph2 && w2 == 0 && lane < R) {
        double v = 0.0;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) v += nb[ww * R + lane];
        const int64_t row = r0m + lane;
        if (row < n) dvec[row] = v;
      }
      if (p < T) {   // -P(p) for phase 2 of the next pass
        const int pb = p & 1;
        mbar_wait(&pready[pb], (p >> 1) & 1);
        const double* P = pbuf + pb * Cf::ACC * 32;
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            pf[r][t].x = P[(((r * NT + t) * 2) + 0) * 32 + lane];
            pf[r][t].y = P[(((r * NT + t) * 2) + 1) * 32 + lane];
          }
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfree[pb]);
      }
    }
    }
  }
done:
#undef FZ_S
  proj_end_stamp(st);
}

static int fz_num_sms() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

static long long* g_fz_trace = nullptr;
static long long* fz_trace_buf() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("RBRP_FZ_TRACE");
    on = e && e[0] == '1';
    if (on && cudaMalloc(&g_fz_trace, 16 * 512 * sizeof(long long)) != cudaSuccess) g_fz_trace = nullptr;
  }
  return g_fz_trace;
}
extern "C" int rbrp_debug_fz_trace(long long* host, int count) {
  if (!g_fz_trace) return -1;
  if (count > 16 * 512) count = 16 * 512;
  return cudaMemcpy(host, g_fz_trace, count * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? count : -1;
}

static int fz_nc(int64_t d) { return (int)((d + fz::KC - 1) / fz::KC); }

size_t fused_pack_bytes(int64_t d) { return 2 * (size_t)fz_nc(d) * fz::PACK_ROWS * fz::KC * 8; }   // two images

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// Largest fused bucket for this width (0: not supported -> two-kernel path).
int fused_max_bucket(const void* X, int64_t ldx, int64_t d) {
  if (d % 2 || d < 16 || ldx % 2 || ((uintptr_t)X % 16)) return 0;
  const int nc = fz_nc(d);
  int best = 0, ns, nq;
  if (FzCfg<16>::rings(nc, ns, nq)) best = 16;
  if (FzCfg<32>::rings(nc, ns, nq)) best = 32;
  // bucket 64 spills under the 96-register cap of 18 warps: two-kernel path for now
  return best;
}

template <int BPB>
static cudaError_t go_fused(const CUtensorMap& map, double* X, int64_t ldx, const double* Qp, double* L,
                            int64_t ldl, int64_t n, int64_t d, double* dvec, DevState* st, bool paper,
                            cudaStream_t s) {
  using Cf = FzCfg<BPB>;
  const int nc = fz_nc(d);
  int ns = 0, nq = 0;
  if (!Cf::rings(nc, ns, nq, paper)) return cudaErrorInvalidValue;
  const size_t smem = Cf::smem(ns, nq);
  auto kern = k_proj_fused<BPB>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long* tr = nullptr;
  static int traced = 0;
  if (BPB == 32 && fz_trace_buf() && !traced) {   // first bucket-32 launch only
    tr = fz_trace_buf();
    traced = 1;
  }
#ifndef FZ_XMODE
#define FZ_XMODE 0   // timing ablations of profiles/r01b_fused_ablation.jsonl (wrong results);
#endif               // a profiling build sets it with RBRP_EXTRA_NVCC=-DFZ_XMODE=n
  const int xmode = FZ_XMODE;
  kern<<<fz_num_sms(), fz::NTH, smem, s>>>(map, X, ldx, Qp, L, ldl, n, (int)d, nc, ns, nq, dvec, st, tr, xmode,
                                           paper ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_pack_q(const float* Qt, int64_t d, double* Qp, DevState* st, cudaStream_t s, int part,
                          int64_t ldq) {
  dim3 grid((unsigned)fz_nc(d), fz::PACK_ROWS);
  k_pack_q<float><<<grid, fz::KC, 0, s>>>(Qt, d, Qp, st, part, ldq > 0 ? ldq : d);
  return cudaGetLastError();
}

cudaError_t launch_pack_q(const double* Qt, int64_t d, double* Qp, DevState* st, cudaStream_t s, int part,
                          int64_t ldq) {
  dim3 grid((unsigned)fz_nc(d), fz::PACK_ROWS);
  k_pack_q<double><<<grid, fz::KC, 0, s>>>(Qt, d, Qp, st, part, ldq > 0 ? ldq : d);
  return cudaGetLastError();
}

cudaError_t launch_proj_fused(double* Xres, int64_t ldx, const double* Qp, double* L, int64_t ldl,
                              int64_t n, int64_t d, double* dvec, DevState* st, int bucket, bool paper,
                              cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  auto enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)ldx * 8};
  const cuuint32_t box[2] = {16, (cuuint32_t)fz::R};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)Xres, dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  switch (bucket) {
    case 16: return go_fused<16>(map, Xres, ldx, Qp, L, ldl, n, d, dvec, st, paper, s);
    case 32: return go_fused<32>(map, Xres, ldx, Qp, L, ldl, n, d, dvec, st, paper, s);
    case 64: return go_fused<64>(map, Xres, ldx, Qp, L, ldl, n, d, dvec, st, paper, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rbrp
