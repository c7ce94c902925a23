// k_proj_tc32.cu — the a4 projection for fp32 data on the 5th-generation tensor cores
// (north_star step 4; Alg. 2 l.13 + l.16, in the right-looking form of P:523):
//
//     L-hat = X_res Q_b^T                 (n x b', written to L[:, k : k+b'])
//     X_res <- X_res - L-hat Q_b ,  d(i) = ||x_res,i||^2  (fp64)
//
// fp32 accuracy from TF32 tensor cores by the 3xTF32 split (reading R19): every operand
// v = v_hi + v_lo with v_hi = v truncated to TF32 (low 13 mantissa bits cleared, exact in
// TF32) and v_lo = v - v_hi (exact in fp32); a product is a_hi b_hi + a_hi b_lo + a_lo b_hi
// (the dropped a_lo b_lo and the TF32 rounding of the lo parts are ~2^-21 relative), with
// fp32 accumulation in TMEM.
//
// Tiles of M = 128 rows (one TMEM lane per row), persistent CTAs (one per SM), chunks of
// KC = 32 columns (one 128-byte swizzle row of fp32).  Per tile:
//   pass 1 (l.13): per chunk c the X chunk arrives by TMA (128-byte swizzle); 8 row warps
//     split it into hi / lo and store both into TMEM (tcgen05.st, two A stages); one thread
//     issues, per 8-column k-step,
//         D1[0:2N1)  += X_hi . [Q_hi ; Q_lo]^T      (N = 2 N1: both products, one A read)
//         D1[0:N1)   += X_lo . Q_hi^T
//     (tcgen05.mma kind::tf32, A from TMEM, B = the packed Q_b chunk in shared memory,
//     K-major, 128-byte swizzle).  L-hat = D1[0:N1) + D1[N1:2N1).
//   epilogue 1: the row warps read L-hat (tcgen05.ld), write L, and store its hi / lo split
//     back into TMEM as the A operand of pass 2.
//   pass 2 (l.16): per chunk c the same X chunk comes back through L2 (pass 1 loaded it
//     with an evict_last policy, pass 2 with evict_first); per 8-row k-step of Q_b
//         D2 += L_hi . Q_hi  +  L_hi . Q_lo  +  L_lo . Q_hi   (N = 32, B = the same packed
//     chunk read MN-major); the row warps form x - D2 in fp32, store it (the residual is
//     read once from HBM and written once), and accumulate ||x_res,i||^2 in fp64.
// N1 = b' rounded up to 16 (<= 64; b' > 64 runs as 64-column parts in sequence, as the
// DMMA kernel does with 32-column parts: Q_b's rows are orthonormal).
//
// Warp roles (352 threads): warp 0 X producer (TMA), warp 1 MMA issuer (one thread; the
// warp allocates TMEM), warp 2 Q producer (1-D bulk copies of the pre-packed chunk
// images), warps 3..10 row warps: warp w serves TMEM lanes 32 (w % 4) .. +32 (the
// tcgen05.ld/st lane-quarter rule) and columns 16 h .. +16 of a chunk, h = (w - 3) / 4.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>
#include <string.h>

#include "launch.cuh"

namespace rbrp {

#ifndef TC_KEEP_FRAC
#define TC_KEEP_FRAC 0.75
#endif
namespace tc {
constexpr int M = 128;                    // rows per tile (TMEM lanes)
constexpr int KC = 32;                    // columns per chunk (128-byte swizzle row)
constexpr int NMAX = 64;                  // Q_b rows per part
constexpr int XSLOT = M * KC * 4;         // 16 KB X chunk
constexpr int QSLOT = 2 * NMAX * KC * 4;  // 16 KB shared-memory Q stage (one image)
constexpr int QIMG = 2 * QSLOT;           // global: image 1 (pass 1) + image 2 (pass 2) per chunk
constexpr int NSX = 7;                    // X ring depth (default; RBRP_TC_NSX, <= NSXMAX)
constexpr int NSXMAX = 12;
constexpr int QRING = 96 * 1024;          // Q ring bytes (default; RBRP_TC_QRING_KB): slots of the launch's image size (<= QSLOT)
constexpr int NSQMAX = 24;
constexpr int NROWW = 8;                  // row warps
constexpr int W_XP = 0, W_MMA = 1, W_QP = 2, W_ROW0 = 3;
constexpr int W_ST = W_ROW0 + NROWW;      // pass-2 TMA store issuer
constexpr int NTH = (W_ST + 1) * 32;
constexpr int NACC2 = 4;
// TMEM columns (512 allocated)
constexpr uint32_t T_ACC1 = 0;     // D1: 2 N1 <= 128 columns
constexpr uint32_t T_XA = 128;     // pass-1 A: 2 stages x (hi 32 | lo 32)
constexpr uint32_t T_LA = 256;     // pass-2 A: L-hat hi (64) | lo (64)
constexpr uint32_t T_ACC2 = 384;   // D2: NACC2 stages x 32
constexpr size_t smem_bytes(int nsx, int qring) { return 1024 + (size_t)nsx * XSLOT + qring + 2 * 2 * M * 8 + 1024; }
constexpr size_t SMEM = smem_bytes(NSX, QRING);
constexpr size_t SMEM_MAX = 232448;
}  // namespace tc

__device__ __forceinline__ uint32_t tc_su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tc_bar_init(uint32_t b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(count) : "memory");
}
__device__ __forceinline__ void tc_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(b) : "memory");
}
__device__ __forceinline__ void tc_expect(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tc_wait(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n"
      "}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// tcgen05.mma kind::tf32, A from TMEM, B from a shared-memory descriptor, D in TMEM.  Called
// by the whole (converged) MMA warp with warp-uniform operands; elect.sync picks the one
// lane that issues (no per-instruction divergence loop around the uniform-datapath op).
__device__ __forceinline__ void tc_mma(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p, e;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " setp.ne.b32 p, %4, 0;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// arrive on the mbarrier once every tcgen05 operation issued so far by the elected lane
// (always lane 0 of the converged warp) is done
__device__ __forceinline__ void tc_commit(uint32_t b) {
  asm volatile(
      "{\n .reg .pred e;\n"
      " elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(b)
      : "memory");
}
// shared-memory matrix descriptor: 128-byte swizzle, version 1 (sm_100)
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor: D f32, A/B tf32, A K-major, B K-major (b_mn = 0) or MN-major,
// M = 128, N
__device__ __forceinline__ uint32_t tc_idesc(int N, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(tc::M >> 4) << 24);
}
__device__ __forceinline__ void tc_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tc_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tc_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ float4 tc_lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
// TF32 split: hi = v with the low 13 mantissa bits cleared, lo = v - hi (exact)
__device__ __forceinline__ void tc_split(float v, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(v) & 0xFFFFE000u;
  lo = __float_as_uint(v - __uint_as_float(hi));
}
__device__ __forceinline__ void tc_arrive_n(uint32_t b, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(n) : "memory");
}
__device__ __forceinline__ void tc_sts4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void tc_rowbar() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(tc::NROWW * 32) : "memory");
}

// dst[0 .. cnt) = v[0 .. cnt), cnt <= 32: PRE scalars up to 16-byte alignment, then float4s
template <int PRE>
__device__ __forceinline__ void tc_store_row(float* dst, const float (&v)[32], int cnt) {
#pragma unroll
  for (int j = 0; j < PRE; ++j)
    if (j < cnt) __stcs(dst + j, v[j]);
#pragma unroll
  for (int j = PRE; j + 4 <= 32; j += 4) {
    if (j + 4 <= cnt) {
      __stcs(reinterpret_cast<float4*>(dst + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j + u < cnt) __stcs(dst + j + u, v[j + u]);
    }
  }
#pragma unroll
  for (int j = PRE + ((32 - PRE) / 4) * 4; j < 32; ++j)
    if (j < cnt) __stcs(dst + j, v[j]);
}

struct TcRing {
  int i = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next(int n) {
    if (++i == n) {
      i = 0;
      ph ^= 1u;
    }
  }
};

__global__ void __launch_bounds__(tc::NTH, 1)
    k_proj_tc32(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap xmap0, int lazy,
                const float* __restrict__ Qimg, float* __restrict__ L, int64_t ldl, int64_t n, int d, int nc,
                DevState* st, float* __restrict__ Xr, int64_t ldx, double* __restrict__ dvec, int part,
                long long* __restrict__ tr, int nsx, int qring, int keep_from) {
  using namespace tc;
  // optional cycle trace of CTA 0, tiles 0-1 (RBRP_TC_TRACE=1; profiling only):
  // tr[(event * 2 + tile) * 128 + step]
  if (blockIdx.x != 0) tr = nullptr;
#define TC_T(ev, pp, ss)                                                             \
  do {                                                                               \
    if (tr && (pp) < 2 && (ss) < 128) tr[((ev) * 2 + (pp)) * 128 + (ss)] = clock64(); \
  } while (0)
  if (st->stop) return;
  int bp;
  int64_t k0;
  if (part < 0) {
    bp = st->b_prime;
    if (bp <= 0 || bp > NMAX) return;
    k0 = st->k;
  } else {
    const int bpa = st->b_prime;
    bp = bpa - NMAX * part < NMAX ? bpa - NMAX * part : NMAX;
    if (bpa <= NMAX || bp <= 0) return;
    k0 = st->k + NMAX * part;
  }
  const int N1 = (bp + 15) & ~15;
  // Q ring slots sized for this launch's images (1 KB multiples: 1024-byte-aligned images)
  const int nkb_ = (N1 + 31) / 32;
  const int qslot = max(2 * N1 * KC * 4, 2 * nkb_ * KC * 128);
  const int NSQ = min(NSQMAX, qring / qslot);
  if (blockIdx.x == 0 && threadIdx.x == 0 && part <= 0) st->ts0 = gtimer();

  extern __shared__ __align__(1024) uint8_t tc_smem[];
  uint8_t* sm = tc_smem + ((1024u - (tc_su32(tc_smem) & 1023u)) & 1023u);
  uint8_t* xs = sm;
  uint8_t* qs = xs + (size_t)nsx * XSLOT;
  double* nrm = reinterpret_cast<double*>(qs + qring);   // [tile parity][h][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(nrm + 2 * 2 * M);
  uint64_t* xfull = bars;
  uint64_t* xempty = xfull + nsx;
  uint64_t* qfull = xempty + nsx;
  uint64_t* qempty = qfull + NSQMAX;
  uint64_t* afull = qempty + NSQMAX;
  uint64_t* aempty = afull + 2;
  uint64_t* a2full = aempty + 2;
  uint64_t* a2empty = a2full + NACC2;
  uint64_t* a1full = a2empty + NACC2;
  uint64_t* lafull = a1full + 1;
  uint64_t* xdone = lafull + 1;   // [NSXMAX] pass 2: the row warps have written the slot
  uint32_t* tslot = reinterpret_cast<uint32_t*>(xdone + NSXMAX);

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t ntiles = (n + M - 1) / M;
  const int T = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  if (T == 0) {
    proj_end_stamp(st);
    return;
  }
  if (tid == 0) {
    for (int s = 0; s < nsx; ++s) {
      tc_bar_init(tc_su32(&xfull[s]), 1);
      tc_bar_init(tc_su32(&xempty[s]), NROWW);
    }
    for (int s = 0; s < NSQMAX; ++s) {
      tc_bar_init(tc_su32(&qfull[s]), 1);
      tc_bar_init(tc_su32(&qempty[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc_bar_init(tc_su32(&afull[s]), NROWW);
      tc_bar_init(tc_su32(&aempty[s]), 1);
    }
    for (int s = 0; s < NACC2; ++s) {
      tc_bar_init(tc_su32(&a2full[s]), 1);
      tc_bar_init(tc_su32(&a2empty[s]), NROWW);
    }
    tc_bar_init(tc_su32(a1full), 1);
    tc_bar_init(tc_su32(lafull), NROWW);
    for (int s = 0; s < nsx; ++s) tc_bar_init(tc_su32(&xdone[s]), NROWW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (w == W_MMA) {   // the whole warp allocates all 512 TMEM columns (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(tc_su32(tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  auto row0_of = [&](int p) { return ((int64_t)blockIdx.x + (int64_t)p * gridDim.x) * M; };
  const int steps = T * 2 * nc;

  if (w == W_XP) {
    if (lane == 0) {
      // X chunks, pass 1 then pass 2 of every tile.  Lazy X_res copy: block 1 reads X itself
      const CUtensorMap* mp = (lazy && st->t == 1 && part <= 0) ? &xmap0 : &xmap;
      uint64_t pol_keep, pol_drop;
      // pass-1 chunks below keep_from (the oldest, re-read last in the reversed pass 2) are
      // not marked evict_last: with 148 x 1 MB tiles in flight the L2 cannot hold them all,
      // so it keeps the newer ones (keep_from: host, launch_proj_tc32)
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_keep));
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_drop));
      TcRing xr;
      for (int s = 0; s < steps; ++s) {
        tc_wait(tc_su32(&xempty[xr.i]), xr.ph ^ 1u);
        TC_T(8, s / (2 * nc), s % (2 * nc));
        const bool second = (s / nc) & 1;
        // pass 2 walks the chunks in reverse: the most recently loaded ones are re-read first,
        // while they are still in L2
        const int y = (int)row0_of(s / (2 * nc)), c = second ? nc - 1 - s % nc : s % nc;
        const uint32_t fb = tc_su32(&xfull[xr.i]);
        tc_expect(fb, XSLOT);   // out-of-bounds rows / columns are zero-filled
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
            "[%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(tc_su32(xs + (size_t)xr.i * XSLOT)),
            "l"(mp), "r"(c * KC), "r"(y), "r"(fb), "l"((second || c < keep_from) ? pol_drop : pol_keep)
            : "memory");
        xr.next(nsx);
      }
    }
  } else if (w == W_QP) {
    if (lane == 0) {
      // packed Q_b chunk images: pass 1 image 1 (hi rows [0, N1), lo rows [N1, 2 N1), K-major
      // B of N = 2 N1), pass 2 image 2 (Q_b^T blocks of 32 columns x 32 K: hi blocks, then
      // lo blocks, K-major B of N = 32)
      const int nkb = (N1 + 31) / 32;
      const uint32_t bytes1 = (uint32_t)(2 * N1 * KC * 4), bytes2 = (uint32_t)(2 * nkb * KC * 128);
      TcRing qr;
      for (int s = 0; s < steps; ++s) {
        tc_wait(tc_su32(&qempty[qr.i]), qr.ph ^ 1u);
        const uint32_t fb = tc_su32(&qfull[qr.i]);
        const bool second = (s / nc) & 1;
        const uint32_t bytes = second ? bytes2 : bytes1;
        tc_expect(fb, bytes);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                tc_su32(qs + (size_t)qr.i * qslot)),
            "l"(Qimg + (size_t)(second ? nc - 1 - s % nc : s % nc) * (QIMG / 4) + (second ? QSLOT / 4 : 0)), "r"(bytes),
            "r"(fb)
            : "memory");
        qr.next(NSQ);
      }
    }
  } else if (w == W_ST) {
    if (lane == 0) {
      // pass-2 stores: once the 8 row warps have written chunk c's residual into its X slot
      // (xdone), one TMA bulk tensor store per chunk; the slot is released to the X producer
      // when the store has read it.  The row warps never wait for a store.
      uint64_t pol_st;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_st));
      TcRing xr;
      uint32_t dph = 0;   // per-slot parity of xdone
      int pend = -1;
      for (int s = 0; s < steps; ++s) {
        const int p = s / (2 * nc), in = s % (2 * nc);
        if (in >= nc) {
          const int c = in - nc;
          tc_wait(tc_su32(&xdone[xr.i]), (dph >> xr.i) & 1u);
          dph ^= 1u << xr.i;
          const int col = (nc - 1 - c) * KC;   // reverse chunk order (see the X producer)
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;\n" ::"l"(
                  &xmap),
              "r"(col), "r"((int)row0_of(p)), "r"(tc_su32(xs + (size_t)xr.i * XSLOT)), "l"(pol_st)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
          if (pend >= 0) {
            asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            tc_arrive_n(tc_su32(&xempty[pend]), NROWW);
          }
          pend = xr.i;
          TC_T(7, p, c);
          if (c == nc - 1) {   // tile end: release the last slot now (the producer reuses it
            // for the next tile's pass 1, before any further pass-2 store of this warp)
            asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            tc_arrive_n(tc_su32(&xempty[pend]), NROWW);
            pend = -1;
          }
        }
        xr.next(nsx);
      }
      asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");   // stores complete
    }
  } else if (w == W_MMA) {
    {   // the whole warp runs the issue loop (uniform control flow); one elected lane issues
      const uint32_t id1a = tc_idesc(2 * N1, 0), id1b = tc_idesc(N1, 0), id2 = tc_idesc(KC, 0);
      const int nkb = (N1 + 31) / 32;
      const uint32_t qs0 = tc_su32(qs);
      TcRing qr, ar, cr;
      for (int p = 0; p < T; ++p) {
        // pass 1: D1 = X_hi [Q_hi; Q_lo]^T + X_lo [Q_hi]^T
        for (int c = 0; c < nc; ++c) {
          tc_wait(tc_su32(&afull[ar.i]), ar.ph);
          tc_wait(tc_su32(&qfull[qr.i]), qr.ph);
          tc_fence_after();
          if (lane == 0) TC_T(0, p, c);
          const uint32_t qa = qs0 + qr.i * qslot;
          const uint32_t xa = tbase + T_XA + 64u * ar.i;
#pragma unroll
          for (int ks = 0; ks < KC / 8; ++ks) {
            const uint64_t bd = tc_desc(qa + 32 * ks, 16, 1024);   // K-major: advance 8 fp32 along K
            tc_mma(tbase + T_ACC1, xa + 8 * ks, bd, id1a, (c | ks) != 0);
            tc_mma(tbase + T_ACC1, xa + 32 + 8 * ks, bd, id1b, 1u);
          }
          tc_commit(tc_su32(&aempty[ar.i]));
          tc_commit(tc_su32(&qempty[qr.i]));
          if (lane == 0) TC_T(1, p, c);
          ar.next(2);
          qr.next(NSQ);
        }
        tc_commit(tc_su32(a1full));
        // pass 2: D2(chunk) = L_hi Q_hi + L_hi Q_lo + L_lo Q_hi  (B = image 2, K-major)
        tc_wait(tc_su32(lafull), (uint32_t)(p & 1));
        tc_fence_after();
        for (int c = 0; c < nc; ++c) {
          tc_wait(tc_su32(&qfull[qr.i]), qr.ph);
          tc_wait(tc_su32(&a2empty[cr.i]), cr.ph ^ 1u);
          tc_fence_after();
          if (lane == 0) TC_T(0, p, nc + c);
          const uint32_t qa = qs0 + qr.i * qslot;
          const uint32_t da = tbase + T_ACC2 + KC * cr.i;
          for (int ks = 0; ks < N1 / 8; ++ks) {
            const uint32_t kb = (uint32_t)(ks >> 2), koff = 32u * (ks & 3);   // 32-K block, 8-K step in it
            const uint64_t bh = tc_desc(qa + 4096u * kb + koff, 16, 1024);
            const uint64_t bl = tc_desc(qa + 4096u * (nkb + kb) + koff, 16, 1024);
            tc_mma(da, tbase + T_LA + 8 * ks, bh, id2, ks != 0);
            tc_mma(da, tbase + T_LA + 8 * ks, bl, id2, 1u);
            tc_mma(da, tbase + T_LA + 64 + 8 * ks, bh, id2, 1u);
          }
          tc_commit(tc_su32(&qempty[qr.i]));
          tc_commit(tc_su32(&a2full[cr.i]));
          if (lane == 0) TC_T(1, p, nc + c);
          qr.next(NSQ);
          cr.next(NACC2);
        }
      }
    }
  } else {
    // row warps
    const int e = w - W_ROW0;
    const int qq = w & 3;                 // TMEM lane quarter of this warp
    const int h = e >> 2;                 // column half of a chunk
    const int r = 32 * qq + lane;         // tile row
    const uint32_t tl = tbase + ((uint32_t)(32 * qq) << 16);
    const uint32_t xs0 = tc_su32(xs);
    const int half = N1 / 2;
    TcRing xr, ar, cr;
    for (int p = 0; p < T; ++p) {
      const int64_t row = row0_of(p) + r;
      const bool vr = row < n;
      // ---- pass 1: split the X chunk into TMEM (A operand)
      for (int c = 0; c < nc; ++c) {
        tc_wait(tc_su32(&xfull[xr.i]), xr.ph);
        if (w == W_ROW0 && lane == 0) TC_T(2, p, c);
        const uint32_t xa = xs0 + xr.i * XSLOT + r * 128;
        float v[16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 f = tc_lds4(xa + ((((4 * h + i) ^ (r & 7))) << 4));
          v[4 * i] = f.x;
          v[4 * i + 1] = f.y;
          v[4 * i + 2] = f.z;
          v[4 * i + 3] = f.w;
        }
        __syncwarp();
        if (lane == 0) tc_arrive(tc_su32(&xempty[xr.i]));
        xr.next(nsx);
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) tc_split(v[i], hi[i], lo[i]);
        tc_wait(tc_su32(&aempty[ar.i]), ar.ph ^ 1u);
        tc_fence_after();
        if (w == W_ROW0 && lane == 0) TC_T(3, p, c);
        tc_st16(tl + T_XA + 64u * ar.i + 16 * h, hi);
        tc_st16(tl + T_XA + 64u * ar.i + 32 + 16 * h, lo);
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) tc_arrive(tc_su32(&afull[ar.i]));
        if (w == W_ROW0 && lane == 0) TC_T(4, p, c);
        ar.next(2);
      }
      // ---- epilogue 1: L-hat = D1[0:N1) + D1[N1:2N1) -> L, and its split -> TMEM (pass-2 A)
      tc_wait(tc_su32(a1full), (uint32_t)(p & 1));
      tc_fence_after();
      float P[32];   // L-hat(row, h half .. + half), kept for the L stores below
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        if (8 * g < half) {
          const int j0 = h * half + 8 * g;
          float a[8], b[8];
          tc_ld8(tl + T_ACC1 + j0, a);
          tc_ld8(tl + T_ACC1 + N1 + j0, b);
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            P[8 * g + j] = a[j] + b[j];
            tc_split(P[8 * g + j], hi[j], lo[j]);
          }
          tc_st8(tl + T_LA + j0, hi);
          tc_st8(tl + T_LA + 64 + j0, lo);
        }
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) tc_arrive(tc_su32(lafull));   // pass 2 may start; L is written meanwhile
      if (vr) {
        const int cnt = min(half, bp - h * half);
        float* dst = L + row * ldl + k0 + h * half;
        switch ((4 - (int)(((uintptr_t)dst >> 2) & 3)) & 3) {   // warp-uniform (ldl % 4 == 0)
          case 0: tc_store_row<0>(dst, P, cnt); break;
          case 1: tc_store_row<1>(dst, P, cnt); break;
          case 2: tc_store_row<2>(dst, P, cnt); break;
          default: tc_store_row<3>(dst, P, cnt); break;
        }
      }
      // ---- pass 2: x_res = x - D2, written back into the X slot and stored by the store warp
      // (one TMA bulk tensor store per chunk, full 128-byte lines); fp64 norms of the stored
      // values in four independent accumulators
      double nq[4] = {0.0, 0.0, 0.0, 0.0};
      for (int c = 0; c < nc; ++c) {
        tc_wait(tc_su32(&a2full[cr.i]), cr.ph);
        tc_fence_after();
        if (w == W_ROW0 && lane == 0) TC_T(5, p, c);
        float a[16];
        tc_ld16(tl + T_ACC2 + KC * cr.i + 16 * h, a);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) tc_arrive(tc_su32(&a2empty[cr.i]));
        cr.next(NACC2);
        tc_wait(tc_su32(&xfull[xr.i]), xr.ph);
        if (w == W_ROW0 && lane == 0) TC_T(6, p, c);
        const uint32_t xsl = xs0 + xr.i * XSLOT;
        const uint32_t xa = xsl + r * 128;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t ad = xa + ((((4 * h + i) ^ (r & 7))) << 4);
          const float4 xv = tc_lds4(ad);
          float4 o;
          o.x = xv.x - a[4 * i];
          o.y = xv.y - a[4 * i + 1];
          o.z = xv.z - a[4 * i + 2];
          o.w = xv.w - a[4 * i + 3];
          nq[i] = fma((double)o.x, (double)o.x, nq[i]);
          nq[i] = fma((double)o.y, (double)o.y, nq[i]);
          nq[i] = fma((double)o.z, (double)o.z, nq[i]);
          nq[i] = fma((double)o.w, (double)o.w, nq[i]);
          tc_sts4(ad, o);
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // visible to the TMA store
        __syncwarp();
        if (lane == 0) tc_arrive(tc_su32(&xdone[xr.i]));
        xr.next(nsx);
      }
      const double nr = (nq[0] + nq[1]) + (nq[2] + nq[3]);
      // d(i) = ||x_res,i||^2: the two column halves summed in a fixed order
      double* nb = nrm + (size_t)(p & 1) * 2 * M;
      nb[h * M + r] = nr;
      tc_rowbar();
      if (h == 0 && vr) dvec[row] = nb[r] + nb[M + r];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == W_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase) : "memory");
  }
  proj_end_stamp(st);
#undef TC_T
}

// Packed Q_b chunk images for k_proj_tc32 (128-byte swizzle of a 1024-byte-aligned shared-
// memory image: row r is 128 bytes, its 16-byte unit u stored at u ^ (r & 7)), per chunk c
// of 32 columns, QIMG bytes apart:
//   image 1 (pass 1, K-major B, N = 2 N1): rows [0, N1) = hi, [N1, 2 N1) = lo of
//     Q_b(r0 + j, 32 c .. 32 c + 32);
//   image 2 (pass 2, K-major B, N = 32, at +QSLOT): blocks of 32 rows (one per column of the
//     chunk) x 32 K values (Q_b rows 32 kb .. +32): hi blocks kb = 0 .. nkb-1, then lo blocks.
// Rows j >= b' and columns >= d are zero.
__global__ void k_pack_tc32(const float* __restrict__ Qt, int64_t d, float* __restrict__ Qimg, const DevState* st,
                            int part, int64_t ldq) {
  using namespace tc;
  if (st->stop) return;
  const int bpa = st->b_prime;
  int bp, r0 = 0;
  if (part < 0) {
    bp = bpa;
    if (bp <= 0 || bp > NMAX) return;
  } else {
    r0 = NMAX * part;
    bp = bpa - r0 < NMAX ? bpa - r0 : NMAX;
    if (bpa <= NMAX || bp <= 0) return;
  }
  const int N1 = (bp + 15) & ~15;
  const int c = blockIdx.x, y = blockIdx.y, lane = threadIdx.x;   // blockDim = 32
  float* img = Qimg + (size_t)c * (QIMG / 4);
  if (y < 2 * NMAX) {   // image 1: row rr = y, column lane
    const int rr = y;
    if (rr >= 2 * N1) return;
    const int j = rr < N1 ? rr : rr - N1;
    const int64_t gc = (int64_t)c * KC + lane;
    const float v = (j < bp && gc < d) ? Qt[(int64_t)(r0 + j) * ldq + gc] : 0.0f;
    const uint32_t hi = __float_as_uint(v) & 0xFFFFE000u;
    const float out = rr < N1 ? __uint_as_float(hi) : v - __uint_as_float(hi);
    img[rr * KC + ((((lane >> 2) ^ (rr & 7))) << 2) + (lane & 3)] = out;
  } else {              // image 2: block (hl, kb), row n (column of the chunk), K index lane
    const int yy = y - 2 * NMAX, nkb = (N1 + 31) / 32;
    const int hl = yy / (2 * KC), kb = (yy / KC) & 1, nn = yy % KC;
    if (kb >= nkb) return;
    const int j = 32 * kb + lane;
    const int64_t gc = (int64_t)c * KC + nn;
    const float v = (j < bp && gc < d) ? Qt[(int64_t)(r0 + j) * ldq + gc] : 0.0f;
    const uint32_t hi = __float_as_uint(v) & 0xFFFFE000u;
    const float out = hl == 0 ? __uint_as_float(hi) : v - __uint_as_float(hi);
    img[QSLOT / 4 + (hl * nkb + kb) * (KC * KC) + nn * KC + ((((lane >> 2) ^ (nn & 7))) << 2) + (lane & 3)] = out;
  }
}

static long long* g_tc_trace = nullptr;
extern "C" int rbrp_debug_tc_trace(long long* host, int count) {
  if (!g_tc_trace) return -1;
  if (count > 9 * 2 * 128) count = 9 * 2 * 128;
  return cudaMemcpy(host, g_tc_trace, count * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? count : -1;
}

static PFN_cuTensorMapEncodeTiled_v12000 tc_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

bool proj_tc32_supported(const void* X, int64_t ldx, int64_t d) {
  return d >= 8 && d % 4 == 0 && ldx % 4 == 0 && ((uintptr_t)X % 16) == 0 && tc_encode() != nullptr;
}

size_t tc32_pack_bytes(int64_t d) { return (size_t)((d + tc::KC - 1) / tc::KC) * tc::QIMG; }

cudaError_t launch_pack_tc32(const float* Qt, int64_t d, float* Qimg, DevState* st, cudaStream_t s, int part) {
  dim3 grid((unsigned)((d + tc::KC - 1) / tc::KC), 2 * tc::NMAX + 4 * tc::KC);
  k_pack_tc32<<<grid, tc::KC, 0, s>>>(Qt, d, Qimg, st, part, d);
  return cudaGetLastError();
}

static bool tc_map(CUtensorMap* map, const float* X, int64_t ldx, int64_t n, int64_t d) {
  auto enc = tc_encode();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)(n > 0 ? n : 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)ldx * 4};
  const cuuint32_t box[2] = {(cuuint32_t)tc::KC, (cuuint32_t)tc::M};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)X, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_proj_tc32(float* X, int64_t ldx, const float* Qimg, float* L, int64_t ldl, int64_t n, int64_t d,
                             double* dvec, DevState* st, cudaStream_t s, const float* X0, int64_t ldx0, int part) {
  if (n <= 0) return cudaSuccess;
  CUtensorMap map, map0;
  if (!tc_map(&map, X, ldx, n, d)) return cudaErrorInvalidValue;
  if (X0) {
    if (!tc_map(&map0, X0, ldx0, n, d)) return cudaErrorInvalidValue;
  } else {
    map0 = map;
  }
  // ring sizes (experiments: RBRP_TC_NSX X slots, RBRP_TC_QRING_KB of Q ring)
  int nsx = tc::NSX, qring = tc::QRING;
  if (const char* e1 = getenv("RBRP_TC_NSX")) nsx = std::max(2, std::min(tc::NSXMAX, atoi(e1)));
  if (const char* e2 = getenv("RBRP_TC_QRING_KB")) qring = std::max(16, atoi(e2)) * 1024;
  if (tc::smem_bytes(nsx, qring) > tc::SMEM_MAX) return cudaErrorInvalidValue;
  static PerDevice attr;
  cudaError_t e = attr.once(
      [] { return cudaFuncSetAttribute(k_proj_tc32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc::SMEM_MAX); });
  long long* tr = nullptr;
  {   // RBRP_TC_TRACE=k (profiling only): cycle trace of the k-th launch of the process
    static long long* buf = nullptr;
    static int nlaunch = 0;
    const char* ev = getenv("RBRP_TC_TRACE");
    if (ev && atoi(ev) == ++nlaunch) {
      if (!buf && cudaMalloc(&buf, 9 * 2 * 128 * sizeof(long long)) == cudaSuccess)
        cudaMemset(buf, 0, 9 * 2 * 128 * sizeof(long long));
      tr = buf;
      g_tc_trace = buf;
    }
  }
  if (e != cudaSuccess) return e;
  const int nc = (int)((d + tc::KC - 1) / tc::KC);
  // pass-1 chunks [0, keep_from) are loaded evict_first: when the 148 tiles in flight
  // (128 x d x 4 bytes each) exceed about half the L2, the oldest quarter is let go
  // (RBRP_TC_KEEP = fraction kept, experiments)
  double keep = (double)device_sms() * tc::M * d * 4 > 64e6 ? TC_KEEP_FRAC : 1.0;
  if (const char* e3 = getenv("RBRP_TC_KEEP")) keep = atof(e3);
  const int keep_from = (int)(nc * (1.0 - keep));
  int grid = device_sms();
  if (const char* g = getenv("RBRP_TC_GRID")) grid = atoi(g);   // experiments only (L2 working set)
  k_proj_tc32<<<grid, tc::NTH, tc::smem_bytes(nsx, qring), s>>>(map, map0, X0 ? 1 : 0, Qimg, L, ldl, n, (int)d, nc,
                                                                 st, X, ldx, dvec, part, tr, nsx, qring, keep_from);
  return cudaGetLastError();
}

}  // namespace rbrp

// Development probe (not in the ABI header): one projection of X (n x d, device, ld d) by
// the b rows of Q (device, b x d): X <- X - (X Q^T) Q in place, L (n x b) and d(i) out.
extern "C" int rbrp_debug_tc32(float* X, int64_t n, int64_t d, const float* Q, int b, float* L, double* dvec) {
  using namespace rbrp;
  DevState h;
  memset(&h, 0, sizeof(h));
  h.b_prime = b;
  h.k = 0;
  h.t = 2;
  DevState* st = nullptr;
  float* img = nullptr;
  if (cudaMalloc(&st, sizeof(DevState)) != cudaSuccess) return -5;
  if (cudaMalloc(&img, tc32_pack_bytes(d)) != cudaSuccess) return -5;
  cudaMemcpy(st, &h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemset(img, 0xff, tc32_pack_bytes(d));
  cudaError_t e = launch_pack_tc32(Q, d, img, st, 0, -1);
  if (e == cudaSuccess) e = launch_proj_tc32(X, d, img, L, b, n, d, dvec, st, 0, nullptr, 0, -1);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(st);
  cudaFree(img);
  return e == cudaSuccess ? 0 : -(int)e;
}
