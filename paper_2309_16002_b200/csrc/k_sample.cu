// k_sample.cu — a2 sample + a5 stop test (Alg. 2 l.3-5).
//
// One CTA.  (1) Inclusive prefix over the per-chunk totals in a fixed order (warp 0),
// giving ||d||_1 bit-identically on every rank; (2) the stop test of l.3 (reading R1:
// continue while ||d||_1 > tau ||d^(0)||_1, or |S| < k in fixed-rank mode) and l.4's
// b_t = min(b, k - |S|) (reading R15); (3) S_t ~ d/||d||_1 without replacement
// (Eq. 2.2; reading R6): rounds of 256 Philox draws (counter (j, t, 0, 0)),
// each resolved by binary search over the chunk prefix and then over the chunk-local
// prefix of d (reading R8), repeats rejected in draw order.  Small support (reading
// R7): all positive rows in row order.
#include "launch.cuh"
#include "philox.cuh"

namespace rbrp {

constexpr int kSampleThreads = 256;
constexpr int kSmemChunks = 2048;   // chunk prefixes searched in shared memory up to 8.4M rows

constexpr int kHashBits = 10;       // repeat-rejection hash set (<= kMaxB + 256 live keys)
constexpr int kHashSize = 1 << kHashBits;
static_assert(kMaxB + kSampleThreads <= kHashSize / 2 && kMaxB + kSampleRound <= kHashSize / 2,
              "hash set load factor");

constexpr int kSkipRows = 64;       // rows per entry of the shared skip table
constexpr int kSkipMax = 2048;      // skip table in shared memory up to 131072 local rows
static_assert(kMaxB <= kSampleThreads, "one block-log entry per thread");
static_assert(kChunk % kSampleThreads == 0 && kChunk / 2 <= kSkipMax, "fused one-chunk scan");

// smallest local row r of global chunk q with cpre[r] > tq; falls back to the last
// positive row of the chunk when tq is past the chunk's end (rounding).  skip (optional):
// cpre at the last row of every 64-row sub-block of the local rows, so the search runs
// over the chunk's sub-blocks in shared memory first (cpre is non-decreasing inside a
// chunk: the first row above tq lies in the first sub-block whose last value is above
// tq), then over 64 rows -- the same row, 6 global loads on the dependent path, not 12.
__device__ int64_t resolve_in_chunk(int q, double tq, const double* __restrict__ cpre,
                                    const double* __restrict__ dvec, int64_t n_local,
                                    int64_t row_offset, const double* skip = nullptr, int sg = kSkipRows) {
  int64_t lo = (int64_t)q * kChunk - row_offset;
  int64_t hi = lo + kChunk;
  if (hi > n_local) hi = n_local;
  if (lo < 0 || lo >= n_local) return -1;   // chunk owned by another rank
  int64_t a = lo, b = hi;                    // search in [a, b)
  if (skip && lo % sg == 0) {
    int64_t sa = lo / sg, sb = (hi + sg - 1) / sg;
    while (sa < sb) {
      const int64_t m = (sa + sb) >> 1;
      if (skip[m] > tq) sb = m; else sa = m + 1;
    }
    a = sa * sg;
    if (a > hi) a = hi;
    b = a + sg < hi ? a + sg : hi;
    if (sg == 1) b = a;   // the skip table is cpre itself
  }
  while (a < b) {
    int64_t m = (a + b) >> 1;
    if (cpre[m] > tq) b = m; else a = m + 1;
  }
  if (a >= hi) {
    a = hi - 1;
    while (a > lo && !(dvec[a] > 0.0)) --a;
  }
  return a + row_offset;
}

// slot of row in the open-addressing set hkey (inserted if absent); rows are distinct keys
__device__ __forceinline__ int hash_slot(unsigned long long* hkey, int64_t row) {
  const unsigned long long key = (unsigned long long)row;
  int h = (int)((uint32_t)((key ^ (key >> 29)) * 2654435761u) >> (32 - kHashBits));
  while (true) {
    const unsigned long long old = atomicCAS(&hkey[h], ~0ull, key);
    if (old == ~0ull || old == key) return h;
    h = (h + 1) & (kHashSize - 1);
  }
}

__device__ __forceinline__ void sstamp(long long* dbg, int k) {
  if (dbg && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    dbg[k] = (long long)t;
  }
}

__global__ void __launch_bounds__(kSampleThreads) k_sample(SampleArgs A) {
  sstamp(A.dbg, 0);
  DevState* st = A.st;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  __shared__ int s_stop, s_bt, s_c, s_new;
  __shared__ double s_total;
  __shared__ int64_t s_np;
  __shared__ int64_t chosen[kMaxB];
  __shared__ unsigned long long hkey[kHashSize];
  __shared__ int hidx[kHashSize];
  __shared__ int wcount[kSampleThreads / 32];
  __shared__ int s_tcur;
  __shared__ double s_cpref[kSmemChunks];
  __shared__ double s_skip[kSkipMax];

  // one round of global loads for the whole prologue: warp 1 snapshots DevState into shared
  // memory while warp 0 loads the chunk totals (the stop test below reads only the snapshot);
  // every thread also loads its entries of the skip table and of the block log
  // skip granularity: the smallest power of two that fits the table in shared memory (one
  // row: the whole cpre, no global load on the draw's path), at most 64 rows
  int sg = 1;
  while (sg < kSkipRows && (A.n_local + sg - 1) / sg > kSkipMax) sg *= 2;
  const int64_t nskip = (A.n_local + sg - 1) / sg;
  const bool use_skip = nskip <= kSkipMax && A.replay_len < 0 && !A.greedy && !A.dist;
  constexpr int kSkipU = kSkipMax / kSampleThreads;
  double skv[kSkipU];
  if (use_skip && !A.fuse_scan) {
#pragma unroll
    for (int u = 0; u < kSkipU; ++u) {
      const int64_t j = tid + (int64_t)u * kSampleThreads, r = j * sg + sg - 1;
      skv[u] = j < nskip ? A.cpre[r < A.n_local ? r : A.n_local - 1] : 0.0;
    }
  }
  // fused scan (one chunk): thread t owns rows [16 t, 16 t + 16) of d
  constexpr int kScanR = kChunk / kSampleThreads;
  double dv[kScanR];
  if (A.fuse_scan) {
#pragma unroll
    for (int u = 0; u < kScanR; ++u) {
      const int64_t r = (int64_t)kScanR * tid + u;
      dv[u] = r < A.n_local ? A.dvec[r] : 0.0;
    }
  }
  const bool may_log = !A.first && A.log.bt != nullptr && tid < A.log.b;
  const int64_t lg_st = may_log ? A.S_t[tid] : -1;
  const int32_t lg_pv = may_log ? A.piv[tid] : -1;
  __shared__ DevState s_st;
  static_assert(sizeof(DevState) % 8 == 0, "DevState snapshot by 8-byte words");
  constexpr int kStWords = (int)(sizeof(DevState) / 8);
  static_assert(kStWords <= 32, "one warp snapshots DevState");
  if (w == 1 && lane < kStWords)
    reinterpret_cast<unsigned long long*>(&s_st)[lane] = reinterpret_cast<const unsigned long long*>(st)[lane];
  // (1) chunk prefix, fixed order: lane l sums a contiguous range of chunks
  if (A.fuse_scan) {
    // the chunk-local prefix cpre of k_chunk_scan, computed here (fixed order: rows within a
    // thread, then a warp scan, then the warp totals): cpre to global memory and, as the skip
    // table, to shared memory; the chunk's total and positive count
    __shared__ double s_wsum[kSampleThreads / 32];
    __shared__ int s_wcnt[kSampleThreads / 32];
    double sacc = 0.0;
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < kScanR; ++u) {
      sacc += dv[u];
      cnt += dv[u] > 0.0;
    }
    double incl = sacc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int wc = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 31) s_wsum[w] = incl;
    if (lane == 0) s_wcnt[w] = wc;
    __syncthreads();
    double base = 0.0;
    long long np = 0;
    for (int q = 0; q < kSampleThreads / 32; ++q) {
      if (q < w) base += s_wsum[q];
      np += s_wcnt[q];
    }
    double pfx = base + incl - sacc;   // exclusive prefix of this thread's rows
#pragma unroll
    for (int u = 0; u < kScanR; ++u) {
      const int64_t r = (int64_t)kScanR * tid + u;
      pfx += dv[u];
      if (r < A.n_local) {
        A.cpre[r] = pfx;
        if (sg == 1) s_skip[r] = pfx;
        else if ((r & 1) || r == A.n_local - 1) s_skip[r >> 1] = pfx;   // sg = 2
      }
    }
    if (tid == kSampleThreads - 1) {
      s_total = pfx;
      s_np = np;
      A.cprefix[0] = pfx;
      s_cpref[0] = pfx;
      A.ctot[0] = pfx;
      A.cpos[0] = (int32_t)np;
    }
  } else if (w == 0) {
    const int nch = A.nchunks;
    const int per = (nch + 31) / 32;
    const int c0 = lane * per, c1 = min(nch, c0 + per);
    double s = 0.0;
    long long np = 0;
    for (int c = c0; c < c1; ++c) { s += A.ctot[c]; np += A.cpos[c]; }
    double incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    double p = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) p = 0.0;
    for (int c = c0; c < c1; ++c) {
      p += A.ctot[c];
      A.cprefix[c] = p;
      if (nch <= kSmemChunks) s_cpref[c] = p;   // the draws search a shared copy
    }
    if (c0 < nch && c1 == nch) s_total = p;     // = cprefix[nch - 1], no read-back
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) np += __shfl_xor_sync(0xffffffffu, np, o);
    if (lane == 0) s_np = np;
  }
  __syncthreads();
  sstamp(A.dbg, 1);
  // log the block that just finished (device-side, read by the host at the end)
  const int tprev = s_st.t, btprev = s_st.b_t, bpprev = s_st.b_prime;
  const bool do_log = (!A.first && tprev >= 1 && tprev > s_st.nlogged && tprev <= A.log.maxlog &&
                    A.log.bt != nullptr);
  if (do_log) {
    const int slot = tprev - 1;
    if (tid < A.log.b) {   // A.log.b = b <= kMaxB <= kSampleThreads
      A.log.St[(int64_t)slot * A.log.b + tid] = tid < btprev ? lg_st : -1;
      A.log.piv[(int64_t)slot * A.log.b + tid] = tid < bpprev ? lg_pv : -1;
    }
    if (tid == 0) {
      A.log.bt[slot] = btprev;
      A.log.bp[slot] = bpprev;
      A.log.ts[2 * slot] = s_st.ts0;
      A.log.ts[2 * slot + 1] = s_st.ts1;
    }
  }
  sstamp(A.dbg, 2);
  if (tid == 0) {
    const double total = s_total;
    const int64_t k = s_st.k + s_st.b_prime;   // l.14: S <- S u S'_t of the previous block
    const double D0 = A.first ? total : s_st.D0;
    uint32_t flags = s_st.flags;
    st->k = k;
    st->b_prime = 0;
    st->total = total;
    st->npos = s_np;
    if (A.first) st->D0 = total;
    if (do_log) {
      A.log.rho[tprev - 1] = total / D0;
      st->nlogged = tprev;
    }
    const bool fixed = !(s_st.tau > 0.0);
    bool stop = s_st.stop != 0;
    if (!stop && k >= s_st.k_cap) {
      stop = true;
      if (!fixed && total > s_st.tau * D0) flags |= RBRP_F_TOL_UNREACHED;
    }
    if (!stop && !fixed && !(total > s_st.tau * D0)) stop = true;   // l.3
    if (!stop && s_np == 0) {
      stop = true;
      flags |= RBRP_F_SUPPORT_EXHAUSTED;
    }
    if (!stop && A.replay_len == -2) stop = true;   // replay log exhausted
    int bt = 0;
    if (!stop) {
      st->t = s_st.t + 1;                                             // l.4
      const int64_t room = s_st.k_cap - k;
      bt = (int)(s_st.b < room ? s_st.b : room);
    }
    if (flags != s_st.flags) st->flags = flags;
    st->stop = stop ? 1 : 0;
    s_stop = stop;
    s_bt = bt;
    s_c = 0;
    s_tcur = stop ? s_st.t : s_st.t + 1;
    if (A.cond) cudaGraphSetConditional((cudaGraphConditionalHandle)A.cond, stop ? 0u : 1u);
    // row-sharded graph loop: the draw rounds run while this block still needs rows
    if (A.cond2) cudaGraphSetConditional((cudaGraphConditionalHandle)A.cond2, stop ? 0u : 1u);
  }
  __syncthreads();
  sstamp(A.dbg, 3);
  if (s_stop) return;
  if (A.dist && A.replay_len < 0) {   // drawing happens in the resolve / accept rounds
    if (tid == 0) {
      st->jb = 0;
      st->sample_c = 0;
      st->sample_done = 0;
      st->exhausted = s_np <= s_bt ? 1 : 0;
      st->b_t = s_bt;
      st->draws = 0;
    }
    return;
  }
  if (A.replay_len >= 0) {
    for (int i = tid; i < A.replay_len; i += kSampleThreads) A.S_t[i] = A.S_rep[i];
    if (tid == 0) { st->b_t = A.replay_len; st->draws = 0; }
    return;
  }
  if (A.greedy) {   // RBGP (Remark 4.2): the top b_t rows of d, in order (k_topb)
    const int c = min(s_bt, *A.top_cnt);
    for (int i = tid; i < c; i += kSampleThreads) A.S_t[i] = A.S_top[i];
    if (tid == 0) {
      st->b_t = c;
      st->draws = 0;
      if (c < s_bt) st->flags |= RBRP_F_SUPPORT_EXHAUSTED;
    }
    return;
  }
  const int bt = s_bt;
  if (s_np <= bt) {
    // reading R7: every positive-weight row, in row order (local rows; single GPU)
    for (int64_t r0 = 0; r0 < A.n_local; r0 += kSampleThreads) {
      int64_t r = r0 + tid;
      int f = (r < A.n_local && A.dvec[r] > 0.0) ? 1 : 0;
      unsigned m = __ballot_sync(0xffffffffu, f);
      if (lane == 0) wcount[w] = __popc(m);
      __syncthreads();
      int off = s_c;
      for (int q = 0; q < w; ++q) off += wcount[q];
      off += __popc(m & ((1u << lane) - 1u));
      if (f && off < kMaxB) chosen[off] = r + A.row_offset;
      __syncthreads();
      if (tid == 0) {
        int tot = 0;
        for (int q = 0; q < kSampleThreads / 32; ++q) tot += wcount[q];
        s_c += tot;
      }
      __syncthreads();
    }
    const int c = min(s_c, kMaxB);
    for (int i = tid; i < c; i += kSampleThreads) A.S_t[i] = chosen[i];
    if (tid == 0) {
      st->b_t = c;
      st->draws = 0;
      st->flags |= RBRP_F_SUPPORT_EXHAUSTED;
    }
    return;
  }
  // (3) rejection rounds
  if (use_skip && !A.fuse_scan) {
#pragma unroll
    for (int u = 0; u < kSkipU; ++u) {
      const int64_t j = tid + (int64_t)u * kSampleThreads;
      if (j < nskip) s_skip[j] = skv[u];
    }
    __syncthreads();
  }
  for (int h = tid; h < kHashSize; h += kSampleThreads) {
    hkey[h] = ~0ull;
    hidx[h] = kSampleThreads;
  }
  __syncthreads();
  sstamp(A.dbg, 4);
  const double total = s_total;
  const uint2 key = make_uint2((uint32_t)(A.seed & 0xffffffffu), (uint32_t)(A.seed >> 32));
  const uint32_t t = (uint32_t)s_tcur;
  int64_t jb = 0;
  for (; jb < kJMax; jb += kSampleThreads) {
    const int c = s_c;
    if (c >= bt) break;
    const uint32_t j = (uint32_t)(jb + tid);
    const double u = u53(philox4x32_10(make_uint4(j, t, 0u, 0u), key));
    const double target = u * total;
    // first chunk q with cprefix[q] > target
    const double* cpf = A.nchunks <= kSmemChunks ? s_cpref : A.cprefix;
    int a = 0, b = A.nchunks;
    while (a < b) {
      int m = (a + b) >> 1;
      if (cpf[m] > target) b = m; else a = m + 1;
    }
    int64_t row;
    if (a >= A.nchunks) {
      // past the end (rounding): last positive row overall
      int q = A.nchunks - 1;
      while (q > 0 && A.cpos[q] == 0) --q;
      row = resolve_in_chunk(q, 1e308, A.cpre, A.dvec, A.n_local, A.row_offset);
    } else {
      const double tq = target - (a > 0 ? cpf[a - 1] : 0.0);
      row = resolve_in_chunk(a, tq, A.cpre, A.dvec, A.n_local, A.row_offset, use_skip ? s_skip : nullptr, sg);
    }
    // repeats: a shared hash set of the rows seen, hidx = the first draw of this round that
    // hit the row, or -1 once the row is in S_t (reading R6: repeats rejected in draw order)
    int slot = -1;
    if (row >= 0) {
      slot = hash_slot(hkey, row);
      atomicMin(&hidx[slot], tid);
    }
    __syncthreads();
    int isnew = slot >= 0 && hidx[slot] == tid;
    unsigned msk = __ballot_sync(0xffffffffu, isnew);
    if (lane == 0) wcount[w] = __popc(msk);
    __syncthreads();
    int off = 0;
    for (int q = 0; q < w; ++q) off += wcount[q];
    off += __popc(msk & ((1u << lane) - 1u));
    if (isnew && c + off < bt) {
      chosen[c + off] = row;
      hidx[slot] = -1;
    }
    if (isnew && c + off == bt - 1) s_new = (int)(jb + tid + 1);   // draws consumed
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int q = 0; q < kSampleThreads / 32; ++q) tot += wcount[q];
      s_c = min(bt, c + tot);
    }
    __syncthreads();
  }
  sstamp(A.dbg, 5);
  if (A.dbg && tid == 0) A.dbg[6] = jb / kSampleThreads;   // rounds
  const int c = s_c;
  for (int i = tid; i < c; i += kSampleThreads) A.S_t[i] = chosen[i];
  if (tid == 0) {
    st->b_t = c;
    st->draws = (c == bt) ? s_new : (int)jb;
  }
  sstamp(A.dbg, 7);
}

cudaError_t launch_sample(const SampleArgs& a, cudaStream_t s) {
  k_sample<<<1, kSampleThreads, 0, s>>>(a);
  return cudaGetLastError();
}

// Round of kSampleRound draws: cand[j] = the global row of draw jb + j if it lands in one
// of this rank's chunks (else left at -1).  Small support (reading R7): this rank's
// positive rows, in row order, at slots [sum of positive counts of the earlier chunks, ...).
__global__ void __launch_bounds__(kSampleRound) k_draw_resolve(SampleArgs A) {
  const DevState* st = A.st;
  if (st->stop || st->sample_done) return;
  const int tid = threadIdx.x;
  if (st->exhausted) {
    __shared__ long long base;
    __shared__ int wc[kSampleRound / 32];
    const int lane = tid & 31, w = tid >> 5;
    if (tid == 0) {
      long long b = 0;
      const int c0 = (int)(A.row_offset / kChunk);
      for (int c = 0; c < c0; ++c) b += A.cpos[c];
      base = b;
    }
    __syncthreads();
    for (int64_t r0 = 0; r0 < A.n_local; r0 += kSampleRound) {
      const int64_t r = r0 + tid;
      const int f = (r < A.n_local && A.dvec[r] > 0.0) ? 1 : 0;
      const unsigned m = __ballot_sync(0xffffffffu, f);
      if (lane == 0) wc[w] = __popc(m);
      __syncthreads();
      long long off = base;
      for (int q = 0; q < w; ++q) off += wc[q];
      off += __popc(m & ((1u << lane) - 1u));
      if (f && off < kSampleRound) A.cand[off] = r + A.row_offset;
      __syncthreads();
      if (tid == 0) {
        long long t = 0;
        for (int q = 0; q < kSampleRound / 32; ++q) t += wc[q];
        base += t;
      }
      __syncthreads();
    }
    return;
  }
  const double total = st->total;
  const uint2 key = make_uint2((uint32_t)(A.seed & 0xffffffffu), (uint32_t)(A.seed >> 32));
  const uint32_t t = (uint32_t)st->t;
  const uint32_t j = (uint32_t)(st->jb + tid);
  const double u = u53(philox4x32_10(make_uint4(j, t, 0u, 0u), key));
  const double target = u * total;
  int a = 0, b = A.nchunks;
  while (a < b) {
    const int m = (a + b) >> 1;
    if (A.cprefix[m] > target) b = m; else a = m + 1;
  }
  int64_t row;
  if (a >= A.nchunks) {
    int q = A.nchunks - 1;
    while (q > 0 && A.cpos[q] == 0) --q;
    row = resolve_in_chunk(q, 1e308, A.cpre, A.dvec, A.n_local, A.row_offset);
  } else {
    const double tq = target - (a > 0 ? A.cprefix[a - 1] : 0.0);
    row = resolve_in_chunk(a, tq, A.cpre, A.dvec, A.n_local, A.row_offset);
  }
  if (row >= 0) A.cand[tid] = row;
}

// Accept the combined candidates of a round in draw order, rejecting repeats (reading
// R6) — the same rule as k_sample's single-GPU loop, so S_t is identical for any sharding.
__global__ void __launch_bounds__(kSampleRound) k_draw_accept(SampleArgs A) {
  DevState* st = A.st;
  if (st->stop || st->sample_done) {
    if (A.cond2 && threadIdx.x == 0) cudaGraphSetConditional((cudaGraphConditionalHandle)A.cond2, 0u);
    return;
  }
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  __shared__ int64_t chosen[kMaxB];
  __shared__ int64_t cand[kSampleRound];
  __shared__ int wcount[kSampleRound / 32];
  __shared__ unsigned long long hkey[kHashSize];
  __shared__ int hidx[kHashSize];
  const int bt = st->b_t;
  const int c = st->sample_c;
  for (int i = tid; i < c; i += kSampleRound) chosen[i] = A.S_t[i];
  const int64_t row = A.cand[tid];
  cand[tid] = row;
  __syncthreads();
  if (st->exhausted) {
    const int n = (int)min((int64_t)kMaxB, st->npos);
    if (tid < n) A.S_t[tid] = cand[tid];
    if (tid == 0) {
      st->b_t = n;
      st->sample_c = n;
      st->sample_done = 1;
      st->flags |= RBRP_F_SUPPORT_EXHAUSTED;
      if (A.cond2) cudaGraphSetConditional((cudaGraphConditionalHandle)A.cond2, 0u);
    }
    return;
  }
  // repeats (reading R6, draw order): S_t's rows so far enter the hash set with hidx = -1,
  // then every draw's row with atomicMin of its index
  for (int h = tid; h < kHashSize; h += kSampleRound) {
    hkey[h] = ~0ull;
    hidx[h] = kSampleRound;
  }
  __syncthreads();
  for (int i = tid; i < c; i += kSampleRound) hidx[hash_slot(hkey, chosen[i])] = -1;
  __syncthreads();
  int slot = -1;
  if (row >= 0) {
    slot = hash_slot(hkey, row);
    atomicMin(&hidx[slot], tid);
  }
  __syncthreads();
  const int isnew = slot >= 0 && hidx[slot] == tid;
  const unsigned msk = __ballot_sync(0xffffffffu, isnew);
  if (lane == 0) wcount[w] = __popc(msk);
  __syncthreads();
  int off = 0;
  for (int q = 0; q < w; ++q) off += wcount[q];
  off += __popc(msk & ((1u << lane) - 1u));
  if (isnew && c + off < bt) A.S_t[c + off] = row;
  if (tid == 0) {
    int tot = 0;
    for (int q = 0; q < kSampleRound / 32; ++q) tot += wcount[q];
    const int nc = min(bt, c + tot);
    st->sample_c = nc;
    st->jb += kSampleRound;
    const bool done = nc >= bt || st->jb >= kJMax;
    if (done) {
      st->sample_done = 1;
      st->b_t = nc;
    }
    if (A.cond2) cudaGraphSetConditional((cudaGraphConditionalHandle)A.cond2, done ? 0u : 1u);
  }
}

cudaError_t launch_draw_resolve(const SampleArgs& a, cudaStream_t s) {
  k_draw_resolve<<<1, kSampleRound, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_draw_accept(const SampleArgs& a, cudaStream_t s) {
  k_draw_accept<<<1, kSampleRound, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rbrp
