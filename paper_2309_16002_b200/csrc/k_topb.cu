// k_topb.cu — RBGP candidate block (Remark 4.2): the b_t
// largest residual norms, ties to the lower row, positive entries only (the oracle's
// top_block).  Replaces the draw of l.5; everything else of Alg. 2 is unchanged.
//
// A tournament of CTA-local bitonic sorts: level 0 sorts 4096-row slices of d and keeps
// the first B = b entries of each (key = (~bits(d), row): for d > 0 the IEEE bit pattern
// is monotone, so ascending keys = descending d, ties by row); every further level sorts
// 4096 candidates at a time, until one CTA holds the final top B.  Deterministic.
#include "launch.cuh"

namespace rbrp {

constexpr int kTopN = 4096;      // keys per CTA sort
constexpr int kTopThreads = 512;

struct TopKey {
  unsigned long long k;   // ~bits(d) for d > 0, all ones otherwise
  long long i;            // global row id
};

__device__ __forceinline__ bool key_less(const TopKey& a, const TopKey& b) {
  return a.k < b.k || (a.k == b.k && a.i < b.i);
}

__device__ __forceinline__ TopKey make_key(double v, long long row) {
  TopKey t;
  t.k = v > 0.0 ? ~(unsigned long long)__double_as_longlong(v) : ~0ull;
  t.i = row;
  return t;
}

// level 0 (dvec != nullptr): keys from d(r), r in [blk*4096, ...), ids r + row_offset;
// level >= 1: keys from the previous level's candidate list (m entries).
__global__ void __launch_bounds__(kTopThreads) k_topb(const double* __restrict__ dvec, int64_t n,
                                                      int64_t row_offset, const TopKey* __restrict__ cin,
                                                      int64_t m, TopKey* __restrict__ cout, int B,
                                                      int64_t* __restrict__ S_top, int* __restrict__ top_cnt,
                                                      const DevState* st) {
  if (st->stop) return;
  extern __shared__ TopKey ks[];   // [kTopN]
  const int64_t base = (int64_t)blockIdx.x * kTopN;
  const int64_t cnt = dvec ? n : m;
  for (int e = threadIdx.x; e < kTopN; e += kTopThreads) {
    const int64_t g = base + e;
    if (g < cnt) ks[e] = dvec ? make_key(dvec[g], g + row_offset) : cin[g];
    else ks[e] = TopKey{~0ull, 0x7fffffffffffffffll};
  }
  __syncthreads();
  for (int k = 2; k <= kTopN; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int e = threadIdx.x; e < kTopN; e += kTopThreads) {
        const int ixj = e ^ j;
        if (ixj > e) {
          const bool up = (e & k) == 0;
          const TopKey a = ks[e], b = ks[ixj];
          if (up ? key_less(b, a) : key_less(a, b)) {
            ks[e] = b;
            ks[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  if (S_top) {   // final level: one CTA
    for (int e = threadIdx.x; e < B; e += kTopThreads) S_top[e] = ks[e].i;
    if (threadIdx.x == 0) {
      int c = 0;
      while (c < B && ks[c].k != ~0ull) ++c;
      *top_cnt = c;
    }
  } else {
    for (int e = threadIdx.x; e < B; e += kTopThreads) cout[(int64_t)blockIdx.x * B + e] = ks[e];
  }
}

size_t topb_scratch_bytes(int64_t n, int B) {
  const int64_t g0 = (n + kTopN - 1) / kTopN;
  return (size_t)2 * (size_t)(g0 > 0 ? g0 : 1) * B * sizeof(TopKey);
}

// S_top[0..B): the top-B rows of d in order; *top_cnt = how many of them have d > 0.
cudaError_t launch_topb(const double* dvec, int64_t n, int64_t row_offset, int B, void* scratch, int64_t* S_top,
                        int* top_cnt, const DevState* st, cudaStream_t s) {
  constexpr size_t kSm = kTopN * sizeof(TopKey);
  static PerDevice attr;
  const cudaError_t ae =
      attr.once([] { return cudaFuncSetAttribute(k_topb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSm); });
  if (ae != cudaSuccess) return ae;
  TopKey* buf[2] = {(TopKey*)scratch, (TopKey*)scratch + ((n + kTopN - 1) / kTopN) * B};
  int64_t g = (n + kTopN - 1) / kTopN;
  if (g <= 1) {
    k_topb<<<1, kTopThreads, kSm, s>>>(dvec, n, row_offset, nullptr, 0, nullptr, B, S_top, top_cnt, st);
    return cudaGetLastError();
  }
  k_topb<<<(unsigned)g, kTopThreads, kSm, s>>>(dvec, n, row_offset, nullptr, 0, buf[0], B, nullptr, nullptr, st);
  int cur = 0;
  int64_t m = g * B;
  while (true) {
    const int64_t g2 = (m + kTopN - 1) / kTopN;
    if (g2 <= 1) {
      k_topb<<<1, kTopThreads, kSm, s>>>(nullptr, 0, 0, buf[cur], m, nullptr, B, S_top, top_cnt, st);
      break;
    }
    k_topb<<<(unsigned)g2, kTopThreads, kSm, s>>>(nullptr, 0, 0, buf[cur], m, buf[cur ^ 1], B, nullptr, nullptr, st);
    cur ^= 1;
    m = g2 * B;
  }
  return cudaGetLastError();
}

}  // namespace rbrp
