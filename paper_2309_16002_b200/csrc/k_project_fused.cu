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

#include "launch.cuh"

namespace rbrp {

namespace fz {
constexpr int R = 16;      // rows per tile (two 8-row MMA groups)
constexpr int KC = 64;     // columns per chunk
constexpr int NW = 8;      // consumer warps (warp w owns columns [8w, 8w+8) of a chunk)
constexpr int NTH = (2 * NW + 1) * 32;   // 8 phase-1 + 8 phase-2 + 1 producer warp
constexpr int PACK_ROWS = 64;   // rows of the packed Q_b buffer (largest fused bucket)
constexpr int SLOT = R * KC;    // doubles per X slot (4 TMA boxes of 16 x 16)
constexpr int SMEM_MAX = 232448;
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
__device__ __forceinline__ void bar_consumers() { asm volatile("bar.sync 1, %0;\n" ::"n"(2 * fz::NW * 32) : "memory"); }

// Q_b chunk layout (shared-memory image): row j, column c at j * 64 + (c ^ f(j))
__host__ __device__ __forceinline__ int qswz(int j, int col) {
  return col ^ (8 * (j & 1)) ^ (4 * ((j >> 1) & 3));
}
// X slot (TMA SWIZZLE_128B, boxes of 16 rows x 16 doubles): row, column (even) -> offset
__device__ __forceinline__ int xoff(int row, int col) {
  return (col >> 4) * 256 + row * 16 + ((((col & 15) >> 1) ^ (row & 7)) << 1);
}
__device__ __forceinline__ int pi_row(int g) { return (g >> 1) + 4 * (g & 1); }

__global__ void k_pack_q(const double* __restrict__ Qt, int64_t d, double* __restrict__ Qp,
                         const DevState* st) {
  if (st->stop) return;
  const int bp = st->b_prime;
  if (bp <= 0 || bp > fz::PACK_ROWS) return;
  const int c = blockIdx.x, j = blockIdx.y, col = threadIdx.x;   // blockDim = KC
  const int64_t gc = (int64_t)c * fz::KC + col;
  const double v = (j < bp && gc < d) ? Qt[(int64_t)j * d + gc] : 0.0;
  Qp[((int64_t)c * fz::PACK_ROWS + j) * fz::KC + qswz(j, col)] = v;
}

template <int BPB>
struct FzCfg {
  static constexpr int NT = BPB / 8;            // 8-column output tiles of P
  static constexpr int ACC = 2 * NT * 2;        // doubles of one warp-lane's P partial
  static constexpr int QSTAGE = BPB * fz::KC;   // doubles per Q stage
  static constexpr int NQ = BPB == 16 ? 4 : 3;  // Q stages
  static constexpr int FIXED = (NQ * QSTAGE + 4 * 32 * ACC + 2 * fz::NW * fz::R) * 8;
  static int ns_for(int nc) {   // X slots that fit; >= nc + 2 required
    int ns = (fz::SMEM_MAX - FIXED - 2048) / (fz::SLOT * 8);
    return ns > nc + 8 ? nc + 8 : ns;
  }
  static size_t smem(int ns) {
    return (size_t)FIXED + (size_t)ns * fz::SLOT * 8 + (2 * ns + 2 * NQ) * 8 + 1024;   // +1 KB: alignment
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
                 int nc, int NS, double* __restrict__ dvec, DevState* st) {
  using Cf = FzCfg<BPB>;
  constexpr int NT = Cf::NT, NQ = Cf::NQ;
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
  double* nrm = scr + 4 * 32 * Cf::ACC;              // 2 x NW x R (pass parity)
  uint64_t* xfull = reinterpret_cast<uint64_t*>(nrm + 2 * NW * R);
  uint64_t* xempty = xfull + NS;
  uint64_t* qfull = xempty + NS;
  uint64_t* qempty = qfull + NQ;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t ntiles = (n + R - 1) / R;
  const int T = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], NW);         // released by the phase-2 warps
    }
    for (int s = 0; s < NQ; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], 2 * NW);     // released by every consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  auto row0_of = [&](int p) { return ((int64_t)blockIdx.x + (int64_t)p * gridDim.x) * R; };
  const int g = lane >> 2, q = lane & 3;
  const int pg = pi_row(g);            // tile row of MMA row g (within an 8-row group)
#define FZ_S(slot, r, t, h) scr[((slot) * Cf::ACC + ((r) * NT + (t)) * 2 + (h)) * 32 + lane]

  if (T == 0) {
  } else if (w == 2 * NW) {
    // ------------------------------- producer warp -------------------------------
    if (lane == 0) {
      const int xsteps = T * nc, qsteps = (T + 1) * nc;
      const int E = NS - nc;
      int sx = 0, sq = 0, xp = 0, xc = 0;
      Ring xr, qr;
      while (sx < xsteps || sq < qsteps) {
        // issue in the order the consumers release the buffers: X(sx) reuses the slot
        // freed at consumer step sx - E, Q(sq) the stage freed at step sq - NQ
        const bool do_x = sx < xsteps && (sq >= qsteps || sx - E <= sq - NQ);
        if (do_x) {
          if (sx >= NS) mbar_wait(&xempty[xr.i], xr.ph ^ 1);
          mbar_expect_tx(&xfull[xr.i], SLOT * 8);   // out-of-bounds elements are zero-filled
          double* dst = xs + (size_t)xr.i * SLOT;
          const int y = (int)row0_of(xp);
#pragma unroll
          for (int b = 0; b < 4; ++b) tma_2d(dst + b * 256, &xmap, xc * KC + 16 * b, y, &xfull[xr.i]);
          xr.next(NS);
          if (++xc == nc) {
            xc = 0;
            ++xp;
          }
          ++sx;
        } else {
          if (sq >= NQ) mbar_wait(&qempty[qr.i], qr.ph ^ 1);
          mbar_expect_tx(&qfull[qr.i], (uint32_t)(Cf::QSTAGE * 8));
          bulk_g2s(qs + qr.i * Cf::QSTAGE, Qp + (size_t)(sq % nc) * PACK_ROWS * KC,
                   (uint32_t)(Cf::QSTAGE * 8), &qfull[qr.i]);
          qr.next(NQ);
          ++sq;
        }
      }
    }
    __syncwarp();
  } else if (w < NW) {
    // ------------------------- phase 1: P(p) += X(p) Q^T -------------------------
    const int xo0 = xoff(pg, 8 * w + 2 * q), xo1 = xoff(8 + pg, 8 * w + 2 * q);
    double2 acc[2][NT];   // acc[r][t] = P[8r+pi(g)][8t+2q+{0,1}] (K-partial of this warp)
    Ring qr, xr;
    for (int p = 0; p <= T; ++p) {
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[r][t] = make_double2(0.0, 0.0);
      const bool ph1 = p < T;
      for (int c = 0; c < nc; ++c) {
        mbar_wait(&qfull[qr.i], qr.ph);
        if (ph1) {
          const double* Qs = qs + qr.i * Cf::QSTAGE;
          mbar_wait(&xfull[xr.i], xr.ph);
          const double* xsl = xs + (size_t)xr.i * SLOT;
          const double2 a0 = *reinterpret_cast<const double2*>(xsl + xo0);
          const double2 a1 = *reinterpret_cast<const double2*>(xsl + xo1);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const int j = 8 * t + g;
            const double2 b = *reinterpret_cast<const double2*>(Qs + j * KC + qswz(j, 8 * w + 2 * q));
            dmma_f(acc[0][t], a0.x, b.x);
            dmma_f(acc[1][t], a1.x, b.x);
            dmma_f(acc[0][t], a0.y, b.y);
            dmma_f(acc[1][t], a1.y, b.y);
          }
          xr.next(NS);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&qempty[qr.i]);
        qr.next(NQ);
      }
      // pass end: fixed-order reduction of the 8 K-partials into scratch slots 0..3
      if (ph1 && w >= 4) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            FZ_S(w - 4, r, t, 0) = acc[r][t].x;
            FZ_S(w - 4, r, t, 1) = acc[r][t].y;
          }
      }
      bar_consumers();   // A
      if (ph1 && w < 4) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            FZ_S(w, r, t, 0) = acc[r][t].x + FZ_S(w, r, t, 0);
            FZ_S(w, r, t, 1) = acc[r][t].y + FZ_S(w, r, t, 1);
          }
      }
      bar_consumers();   // B
      // the phase-1 warps may run at most NQ - 1 chunks ahead of the phase-2 warps; with
      // nc <= NQ they could reach the next pass end (scratch writes) before the phase-2
      // warps have read this pass's scratch
      if (nc <= NQ) bar_consumers();   // C
    }
  } else {
    // -------------------- phase 2: X(p-1) -= P(p-1) Q, norms --------------------
    const int w2 = w - NW;
    const int xo0 = xoff(pg, 8 * w2 + 2 * q), xo1 = xoff(8 + pg, 8 * w2 + 2 * q);
    double2 pf[2][NT];    // -P(p-1) in the accumulator layout (A fragments)
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int t = 0; t < NT; ++t) pf[r][t] = make_double2(0.0, 0.0);
    Ring qr, xr;
    for (int p = 0; p <= T; ++p) {
      double nr0 = 0.0, nr1 = 0.0;
      const int64_t r0m = row0_of(p - 1);
      const bool ph2 = p >= 1;
      for (int c = 0; c < nc; ++c) {
        mbar_wait(&qfull[qr.i], qr.ph);
        if (ph2) {
          const double* Qs = qs + qr.i * Cf::QSTAGE;
          mbar_wait(&xfull[xr.i], xr.ph);   // completed a pass ago (acquire for this warp)
          const double* xsl = xs + (size_t)xr.i * SLOT;
          double2 x0 = *reinterpret_cast<const double2*>(xsl + xo0);
          double2 x1 = *reinterpret_cast<const double2*>(xsl + xo1);
          double2 z0 = make_double2(0.0, 0.0), z1 = make_double2(0.0, 0.0);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const int j0 = 8 * t + 2 * q;
            const double b0 = Qs[j0 * KC + qswz(j0, 8 * w2 + g)];
            const double b1 = Qs[(j0 + 1) * KC + qswz(j0 + 1, 8 * w2 + g)];
            dmma_f(x0, pf[0][t].x, b0);
            dmma_f(x1, pf[1][t].x, b0);
            dmma_f(z0, pf[0][t].y, b1);
            dmma_f(z1, pf[1][t].y, b1);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&xempty[xr.i]);
          xr.next(NS);
          const int col = c * KC + 8 * w2 + 2 * q;
          if (col < d) {
            const double2 v0 = make_double2(x0.x + z0.x, x0.y + z0.y);
            const double2 v1 = make_double2(x1.x + z1.x, x1.y + z1.y);
            const int64_t row0 = r0m + pg, row1 = r0m + 8 + pg;
            if (row0 < n) {
              __stcs(reinterpret_cast<double2*>(X + row0 * ldx + col), v0);
              nr0 += v0.x * v0.x + v0.y * v0.y;
            }
            if (row1 < n) {
              __stcs(reinterpret_cast<double2*>(X + row1 * ldx + col), v1);
              nr1 += v1.x * v1.x + v1.y * v1.y;
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&qempty[qr.i]);
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
      bar_consumers();   // A
      if (ph2 && w2 == 0 && lane < R) {
        double v = 0.0;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) v += nb[ww * R + lane];
        const int64_t row = r0m + lane;
        if (row < n) dvec[row] = v;
      }
      bar_consumers();   // B
      if (p < T) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            pf[r][t].x = -((FZ_S(0, r, t, 0) + FZ_S(1, r, t, 0)) + (FZ_S(2, r, t, 0) + FZ_S(3, r, t, 0)));
            pf[r][t].y = -((FZ_S(0, r, t, 1) + FZ_S(1, r, t, 1)) + (FZ_S(2, r, t, 1) + FZ_S(3, r, t, 1)));
          }
        // L-hat rows of tile p (l.13): warp w2 writes tile rows 2w2, 2w2+1, lane = column
        // j, read back from the four scratch slots in the same summation order
        const int64_t r0p = row0_of(p);
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int rr = 2 * w2 + h2, r = rr >> 3, x = rr & 7;
          const int gg = 2 * (x & 3) + (x >> 2);   // pi^-1
          const int64_t row = r0p + rr;
#pragma unroll
          for (int jb = 0; jb < BPB; jb += 32) {
            const int j = jb + lane;
            if (j < BPB && j < bp && row < n) {
              const int t = j >> 3, qq = (j & 7) >> 1, h = j & 1;
              const int base = ((r * NT + t) * 2 + h) * 32 + 4 * gg + qq;
              const double v = (scr[(0 * Cf::ACC) * 32 + base] + scr[(1 * Cf::ACC) * 32 + base]) +
                               (scr[(2 * Cf::ACC) * 32 + base] + scr[(3 * Cf::ACC) * 32 + base]);
              L[row * ldl + k0 + j] = v;
            }
          }
        }
      }
      if (nc <= NQ) bar_consumers();   // C
    }
  }
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

static int fz_nc(int64_t d) { return (int)((d + fz::KC - 1) / fz::KC); }

size_t fused_pack_bytes(int64_t d) { return (size_t)fz_nc(d) * fz::PACK_ROWS * fz::KC * 8; }

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
  int best = 0;
  if (FzCfg<16>::ns_for(nc) >= nc + 2) best = 16;
  if (FzCfg<32>::ns_for(nc) >= nc + 2) best = 32;
  if (FzCfg<64>::ns_for(nc) >= nc + 2) best = 64;
  return best;
}

template <int BPB>
static cudaError_t go_fused(const CUtensorMap& map, double* X, int64_t ldx, const double* Qp, double* L,
                            int64_t ldl, int64_t n, int64_t d, double* dvec, DevState* st, cudaStream_t s) {
  using Cf = FzCfg<BPB>;
  const int nc = fz_nc(d);
  const int ns = Cf::ns_for(nc);
  const size_t smem = Cf::smem(ns);
  auto kern = k_proj_fused<BPB>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<fz_num_sms(), fz::NTH, smem, s>>>(map, X, ldx, Qp, L, ldl, n, (int)d, nc, ns, dvec, st);
  return cudaGetLastError();
}

cudaError_t launch_pack_q(const double* Qt, int64_t d, double* Qp, DevState* st, cudaStream_t s) {
  dim3 grid((unsigned)fz_nc(d), fz::PACK_ROWS);
  k_pack_q<<<grid, fz::KC, 0, s>>>(Qt, d, Qp, st);
  return cudaGetLastError();
}

cudaError_t launch_proj_fused(double* Xres, int64_t ldx, const double* Qp, double* L, int64_t ldl,
                              int64_t n, int64_t d, double* dvec, DevState* st, int bucket,
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
    case 16: return go_fused<16>(map, Xres, ldx, Qp, L, ldl, n, d, dvec, st, s);
    case 32: return go_fused<32>(map, Xres, ldx, Qp, L, ldl, n, d, dvec, st, s);
    case 64: return go_fused<64>(map, Xres, ldx, Qp, L, ldl, n, d, dvec, st, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rbrp
