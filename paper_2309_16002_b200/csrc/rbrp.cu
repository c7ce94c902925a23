// rbrp.cu — C ABI of librbrp.so (include/rbrp.h) and the host orchestration of
// Alg. 2 + Alg. 3.
//
// Every decision of the loop (stop test l.3, b_t l.4, sampling l.5, b' l.8, |S| l.14)
// is taken on the device in DevState, so the block loop needs no host round trip: the
// kernels of one block are captured once into the body of a CUDA-graph conditional WHILE
// node whose condition the sampler kernel sets (cudaGraphSetConditional).  The whole
// selection runs as one graph launch; the instantiated graph is cached per (problem,
// buffers).  Replay / profiling / graph-less runs use the same kernels launched eagerly,
// with one host read of DevState per block.  Per-block results go to a device log that
// the host reads once at the end.
#include <cuda_runtime.h>
#include <float.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>   // environ

#include <algorithm>
#include <list>
#include <memory>
#include <mutex>
#include <vector>

#include <chrono>

#include "comm.cuh"
#include "launch.cuh"

using namespace rbrp;

namespace {

#define CK(x)                                   \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) return RBRP_ECUDA;   \
  } while (0)

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t Xres = SIZE_MAX, Qall = SIZE_MAX, Ccgs = SIZE_MAX, Topb = SIZE_MAX, Stop = SIZE_MAX, Tcnt = SIZE_MAX, dvec, cpre, ctot, cpos, cprefix, L, Qt, Qp, Vg, Gpart, G, Tg, Ag, R11, Rtot,
         piv, mass, St, Srep, S, forced, dbg, cand, st, L1 = SIZE_MAX, LinvT = SIZE_MAX, Wsc = SIZE_MAX,
         Pinv = SIZE_MAX, Qtc = SIZE_MAX;
  size_t lbt, lbp, lrho, lSt, lpiv, lts, total;
  int nsplit, maxlog;
  int64_t nchunks, k_cap;
};

int64_t k_cap_of(const rbrp_problem* p) {
  return p->k_max > 0 ? p->k_max : std::min<int64_t>(p->n_global, p->d);
}

int validate(const rbrp_problem* p) {
  if (!p) return RBRP_EINVAL;
  if (p->dtype != RBRP_F32 && p->dtype != RBRP_F64) return RBRP_EINVAL;
  if (p->b < 1 || p->b > RBRP_MAX_B) return RBRP_EINVAL;
  if (p->d < 1 || p->ld < p->d) return RBRP_EINVAL;
  if (p->n_global < 1 || p->n_local < 0 || p->row_offset < 0 ||
      p->row_offset + p->n_local > p->n_global)
    return RBRP_EINVAL;
  if (p->tol != p->tol || p->tol >= 1.0) return RBRP_EINVAL;
  if (!(p->tol > 0.0) && p->k_max < 1) return RBRP_EINVAL;
  if (p->k_max < 0) return RBRP_EINVAL;
  if (p->tau_b != p->tau_b || p->tau_b > 1.0) return RBRP_EINVAL;
  if (p->replay_nblocks < 0 || (p->replay_nblocks > 0 && (!p->replay_blocks || !p->replay_lens)))
    return RBRP_EINVAL;
  return RBRP_OK;
}

Layout make_layout(const rbrp_problem* p) {
  Layout L;
  const size_t w = p->dtype == RBRP_F64 ? 8 : 4;
  const int64_t n = p->n_local, d = p->d;
  L.k_cap = k_cap_of(p);
  L.nchunks = (p->n_global + RBRP_CHUNK - 1) / RBRP_CHUNK;
  L.nsplit = filter_coop_nsplit(d);
  L.maxlog = (int)std::min<int64_t>(L.k_cap + 1, 8192);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + std::max<size_t>(bytes, 1));
    return o;
  };
  const size_t B = RBRP_MAX_B;
  const bool paper = (p->flags & RBRP_FORM_PAPER) != 0;
  if (!(p->flags & RBRP_INPLACE) && !paper) L.Xres = take((size_t)n * d * w);
  if (p->greedy) {   // RBGP candidate tournament (k_topb)
    L.Topb = take(topb_scratch_bytes(n, p->b));
    L.Stop = take((size_t)RBRP_MAX_B * 8);
    L.Tcnt = take(8);
  }
  if (paper) {
    L.Qall = take((size_t)L.k_cap * d * w);   // Q = [Q_1 ... Q_t] rows (l.10)
    L.Ccgs = take((size_t)RBRP_MAX_B * L.k_cap * 8);   // CGS coefficients (l.6)
  }
  L.dvec = take((size_t)n * 8);
  L.cpre = take((size_t)n * 8);
  L.ctot = take((size_t)L.nchunks * 8);
  L.cpos = take((size_t)L.nchunks * 4);
  L.cprefix = take((size_t)L.nchunks * 8);
  L.L = take((size_t)n * L.k_cap * w);
  L.Qt = take(B * d * w);
  L.Qp = take(fused_pack_bytes(d));
  if (p->dtype == RBRP_F32) L.Qtc = take(tc32_pack_bytes(d));   // packed Q_b images of k_proj_tc32
  L.Vg = take(B * d * 8);
  L.Gpart = take((size_t)L.nsplit * B * B * 8);
  L.G = take(B * B * 8);
  L.Tg = take((size_t)L.nsplit * B * B * 8);
  L.Ag = take((size_t)L.nsplit * B * B * 8);
  L.R11 = take(B * B * 8);
  L.Rtot = take(B * B * 8);
  L.piv = take(B * 4);
  L.mass = take(B * 8);
  L.St = take(B * 8);
  L.Srep = take(B * 8);
  L.S = take((size_t)L.k_cap * 8);
  L.forced = take(B * 4);
  L.dbg = take(64 * 8);
  L.cand = take((size_t)kSampleRound * 8);
  L.st = take(sizeof(DevState));
  L.lbt = take((size_t)L.maxlog * 4);
  L.lbp = take((size_t)L.maxlog * 4);
  L.lrho = take((size_t)L.maxlog * 8);
  L.lSt = take((size_t)L.maxlog * p->b * 8);
  L.lpiv = take((size_t)L.maxlog * p->b * 4);
  L.lts = take((size_t)L.maxlog * 16);
  if (!(p->flags & RBRP_NO_W)) {
    L.L1 = take((size_t)L.k_cap * L.k_cap * 8);
    L.LinvT = take((size_t)L.k_cap * ((L.k_cap + 7) / 8 * 8) * w);   // k x round8(k) (K padded for DMMA)
    L.Wsc = take(gemm_lp_scratch_bytes(L.k_cap, (L.k_cap + 7) / 8 * 8));   // packed L_1^{-T} groups
    L.Pinv = take(pinv_scratch_bytes(L.k_cap));   // Remark 5.2 fallback: Jacobi V + counters
  }
  L.total = off;
  return L;
}

// pinned host staging (per host thread), grown on demand
struct Pinned {
  void* p = nullptr;
  size_t n = 0;
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
  void* get(size_t bytes) {
    if (bytes > n) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      n = 0;
      if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
      n = bytes;
    }
    return p;
  }
};
thread_local Pinned g_pinned;

bool env_on(const char* name) {
  const char* e = getenv(name);
  return e && e[0] == '1';
}
// RBRP_FORCE_SIMT=1: CUDA-core projection kernels instead of DMMA.  RBRP_NO_GRAPH=1: eager
// block loop.  RBRP_DEBUG_STAMPS=1: print the filter phase stamps of every block (eager).
bool force_simt() { return env_on("RBRP_FORCE_SIMT"); }
// smallest K (= k rounded up to 8) for which W = L L_1^{-1} runs as k_lhat64 passes
// rather than k_nt_mma (measured, scripts/w_bench.py: k = 240: 0.66 vs 0.98 ms, k = 128:
// 0.22 vs 0.25 ms; RBRP_W_MINK overrides)
// fp32: any K (the alternative is the CUDA-core tile GEMM)
template <typename T = double>
int64_t w_min_k() {
  const char* e = getenv("RBRP_W_MINK");
  return e ? atoll(e) : (sizeof(T) == 8 ? 128 : 16);
}
// RBRP_HOST_TIMING=1: host microseconds between the marks of one rbrp_id (profiling only)
struct HostMarks {
  bool on = env_on("RBRP_HOST_TIMING");
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  char buf[512];
  int len = 0;
  void mark(const char* what) {
    if (!on) return;
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    len += snprintf(buf + len, sizeof(buf) - len, " %s %.1f", what, us);
  }
  ~HostMarks() {
    if (on) fprintf(stderr, "rbrp host us:%s\n", buf);
  }
};
template <typename T>
int lp_max_bucket(const void* X, int64_t ldx, int64_t d) {
  return sizeof(T) == 8 ? lhat_paper_max_bucket(X, ldx, d) : lhat_paper_max_bucket_f32(X, ldx, d);
}

// per-phase CUDA events on the caller's stream (report.profile, eager loop only)
struct Prof {
  bool on = false;
  cudaStream_t s = nullptr;
  std::vector<int> phase;
  std::vector<cudaEvent_t> ev;   // pairs (start, end)
  void begin(int ph) {
    if (!on) return;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    ev.push_back(a);
    ev.push_back(b);
    phase.push_back(ph);
  }
  void end() {
    if (!on) return;
    cudaEventRecord(ev.back(), s);
  }
  void collect(float* out) {
    for (size_t i = 0; i < phase.size(); ++i) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]) == cudaSuccess) out[phase[i]] += ms;
    }
  }
  ~Prof() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

// device pointers of one call
template <typename T>
struct Ctx {
  const rbrp_problem* p;
  const Layout* Ly;
  rbrp_comm* comm;
  int64_t n, d, k_cap, chunk0, ldr;
  T* X;
  T* Xres;
  double *dvec, *cpre, *ctot, *cprefix, *Vg, *Gpart, *G, *Tg, *Ag, *R11, *Rtot, *mass;
  int32_t *cpos, *piv, *forced;
  T *Lm, *Qt;
  double* Qp;   // packed Q_b chunks of the 64-row-tile projection (k_pack_q)
  T* Qall;      // paper form: accumulated Q rows (k_cap x d)
  double* Ccgs; // paper form: CGS coefficients
  char* ws;     // workspace base
  bool paper;   // RBRP_FORM_PAPER: left-looking, X read only
  int64_t *St, *Srep, *S, *cand;
  double* L1;
  T* LinvT;
  void* Wsc;   // scratch of the W GEMM (gemm_nt_lp)
  void* Pinv;  // scratch of the clipped-pinv fallback (Remark 5.2)
  float* Qtc;  // packed Q_b chunk images of the tcgen05 fp32 projection
  bool tc32 = false;   // fp32 residual form on tcgen05 (k_proj_tc32)
  DevState* st;
  long long* dbg;
  BlockLog log;
  bool use_mma, use_forced;
  bool force_blk = false;   // replay: this block's pivots are forced (first entry >= 0)
  int nforced = 0;          // blocks run with forced pivots (RBRP_F_NEAR_TIE)
  int bucketB;
  int lp_max;      // largest bucket run by the 64-row tiled kernel k_lhat_paper (0: none)
  bool tiled;      // residual form on the 64-row tiled kernel (L-hat pass + update pass via L2)
  bool lazy;       // X_res not copied at init: block 1's projection reads X and writes X_res
};

// pointers of one shard's workspace
template <typename T>
void make_ctx(Ctx<T>& c, const rbrp_problem* p, void* Xv, char* ws, const Layout& Ly, rbrp_comm* comm) {
  c.p = p;
  c.Ly = &Ly;
  c.comm = comm;
  c.n = p->n_local;
  c.d = p->d;
  c.k_cap = Ly.k_cap;
  c.chunk0 = p->row_offset / RBRP_CHUNK;
  const bool inplace = (p->flags & RBRP_INPLACE) != 0;
  c.X = (T*)Xv;
  c.paper = (p->flags & RBRP_FORM_PAPER) != 0;
  c.Xres = (inplace || c.paper) ? c.X : (T*)(ws + Ly.Xres);   // paper form: X itself, read only
  c.ldr = (inplace || c.paper) ? p->ld : c.d;
  c.ws = ws;
  c.Qall = c.paper ? (T*)(ws + Ly.Qall) : nullptr;
  c.Ccgs = c.paper ? (double*)(ws + Ly.Ccgs) : nullptr;
  c.dvec = (double*)(ws + Ly.dvec);
  c.cpre = (double*)(ws + Ly.cpre);
  c.ctot = (double*)(ws + Ly.ctot);
  c.cpos = (int32_t*)(ws + Ly.cpos);
  c.cprefix = (double*)(ws + Ly.cprefix);
  c.Lm = (T*)(ws + Ly.L);
  c.Qt = (T*)(ws + Ly.Qt);
  c.Qp = (double*)(ws + Ly.Qp);
  c.Vg = (double*)(ws + Ly.Vg);
  c.Gpart = (double*)(ws + Ly.Gpart);
  c.G = (double*)(ws + Ly.G);
  c.Tg = (double*)(ws + Ly.Tg);
  c.Ag = (double*)(ws + Ly.Ag);
  c.R11 = (double*)(ws + Ly.R11);
  c.Rtot = (double*)(ws + Ly.Rtot);
  c.piv = (int32_t*)(ws + Ly.piv);
  c.mass = (double*)(ws + Ly.mass);
  c.St = (int64_t*)(ws + Ly.St);
  c.Srep = (int64_t*)(ws + Ly.Srep);
  c.S = (int64_t*)(ws + Ly.S);
  c.cand = (int64_t*)(ws + Ly.cand);
  c.forced = (int32_t*)(ws + Ly.forced);
  c.st = (DevState*)(ws + Ly.st);
  c.L1 = Ly.L1 != SIZE_MAX ? (double*)(ws + Ly.L1) : nullptr;
  c.LinvT = Ly.LinvT != SIZE_MAX ? (T*)(ws + Ly.LinvT) : nullptr;
  c.Wsc = Ly.Wsc != SIZE_MAX ? (void*)(ws + Ly.Wsc) : nullptr;
  c.Pinv = Ly.Pinv != SIZE_MAX ? (void*)(ws + Ly.Pinv) : nullptr;
  c.Qtc = Ly.Qtc != SIZE_MAX ? (float*)(ws + Ly.Qtc) : nullptr;
  c.dbg = env_on("RBRP_DEBUG_STAMPS") ? (long long*)(ws + Ly.dbg) : nullptr;
  c.log.bt = (int32_t*)(ws + Ly.lbt);
  c.log.bp = (int32_t*)(ws + Ly.lbp);
  c.log.rho = (double*)(ws + Ly.lrho);
  c.log.St = (int64_t*)(ws + Ly.lSt);
  c.log.piv = (int32_t*)(ws + Ly.lpiv);
  c.log.ts = (long long*)(ws + Ly.lts);
  c.log.maxlog = Ly.maxlog;
  c.log.b = p->b;
  c.use_forced = p->replay_pivots != nullptr;
  c.use_mma = sizeof(T) == 8 && !force_simt() && projection_mma_supported(c.Xres, c.ldr, c.Qt, c.d);
  c.bucketB = bucket_of((int)std::min<int64_t>(p->b, c.k_cap));
  // residual form: the 64-row tiled kernel (L-hat pass + update pass re-reading the tile
  // through L2); fp32: the same kernel with fp32 storage and fp64 DMMA arithmetic
  // (R19); RBRP_FP32_SIMT=1 keeps the CUDA-core fp32 kernels
  const bool lp_ok = sizeof(T) == 8 ? c.use_mma : (!force_simt() && !env_on("RBRP_FP32_SIMT"));
  c.tiled = !c.paper && lp_ok;
  c.lp_max = ((c.paper || c.tiled) && lp_ok && !env_on("RBRP_NO_FUSED")) ? lp_max_bucket<T>(c.Xres, c.ldr, c.d) : 0;
  // the tiled kernel handles every bucket of this problem, so it can take block 1 straight
  // from X (X_res is then never copied: one HBM read + write less per ID).  Single-GPU
  // path only (run_dist keeps the copy).
  // (b' > 32 runs as 32-column parts on the same kernel, enqueue_projection)
  const int lp_need = c.bucketB > 32 && !env_on("RBRP_NO_PARTS") ? 32 : c.bucketB;
  c.lazy = c.tiled && !inplace && c.Xres != c.X && c.lp_max >= lp_need && c.lp_max > 0 &&
           lp_max_bucket<T>(c.X, p->ld, c.d) >= lp_need && !env_on("RBRP_EAGER_COPY");
  // fp32 residual form: the tcgen05 3xTF32 kernel (RBRP_FP32_DMMA=1 keeps the fp64-DMMA one)
  if (sizeof(T) == 4 && !c.paper && c.Qtc && !force_simt() && !env_on("RBRP_FP32_DMMA") && !env_on("RBRP_FP32_SIMT") &&
      proj_tc32_supported(c.Xres, c.ldr, c.d)) {
    c.tc32 = true;
    c.tiled = false;
    c.lazy = !inplace && c.Xres != c.X && proj_tc32_supported(c.X, p->ld, c.d) && !env_on("RBRP_EAGER_COPY");
  }
}

// one sampling chunk on one GPU: k_sample computes the chunk scan itself (no k_chunk_scan
// launch; RBRP_NO_FUSE_SCAN=1 keeps the separate kernel)
template <typename T>
bool fuse_scan(const Ctx<T>& c) {
  return !c.comm && c.Ly->nchunks == 1 && c.n <= RBRP_CHUNK && c.chunk0 == 0 && !env_on("RBRP_NO_FUSE_SCAN");
}

template <typename T>
void make_sample_args(SampleArgs& sa, const Ctx<T>& c, int dist) {
  memset(&sa, 0, sizeof(sa));
  sa.st = c.st;
  sa.ctot = c.ctot;
  sa.cpos = c.cpos;
  sa.cprefix = c.cprefix;
  sa.nchunks = (int)c.Ly->nchunks;
  sa.cpre = c.cpre;
  sa.dvec = c.dvec;
  sa.n_local = c.n;
  sa.row_offset = c.p->row_offset;
  sa.S_t = c.St;
  sa.S_rep = c.Srep;
  sa.seed = c.p->seed;
  sa.first = 1;
  sa.piv = c.piv;
  sa.log = c.log;
  sa.cond = 0;
  sa.dist = dist;
  sa.cand = c.cand;
  sa.greedy = c.p->greedy ? 1 : 0;
  sa.S_top = c.p->greedy ? (const int64_t*)((char*)c.ws + c.Ly->Stop) : nullptr;
  sa.top_cnt = c.p->greedy ? (const int*)((char*)c.ws + c.Ly->Tcnt) : nullptr;
  sa.dbg = c.dbg ? c.dbg + 32 : nullptr;
  sa.fuse_scan = (!dist && fuse_scan(c)) ? 1 : 0;
}

// l.5: RBRP draw, or (RBGP, Remark 4.2) the top-b rows of d computed first by k_topb
template <typename T>
cudaError_t launch_block_sample(Ctx<T>& c, SampleArgs& sa, cudaStream_t s, int* nl) {
  if (sa.greedy) {
    ++*nl;
    cudaError_t e = launch_topb(c.dvec, c.n, c.p->row_offset, c.p->b, c.ws + c.Ly->Topb,
                                (int64_t*)(c.ws + c.Ly->Stop), (int*)(c.ws + c.Ly->Tcnt), c.st, s);
    if (e != cudaSuccess) return e;
  }
  ++*nl;
  return launch_sample(sa, s);
}

// b' <= 64 on the 64-row-tile kernel: the filter writes Q_b's packed images itself (no
// k_pack_q launch); RBRP_NO_FUSE_PACK=1 restores the separate launch
template <typename T>
bool fuse_pack(const Ctx<T>& c) {
  return !env_on("RBRP_NO_FUSE_PACK") && !c.tc32 && (c.paper || c.tiled) && c.lp_max > 0;
}

// a4 (Alg. 2 l.13 + l.16): the 64-row-tile kernel k_lhat_paper (L-hat pass + update pass
// per tile) for the buckets it supports, else the two-kernel DMMA / CUDA-core path.  Each
// launch is a no-op unless the block's b' falls in its bucket, so the sequence is
// graph-capturable.
template <typename T>
int enqueue_projection(Ctx<T>& c, cudaStream_t s, int* nl) {
  auto lk = [&](cudaError_t e) {
    ++*nl;
    return e == cudaSuccess ? (int)RBRP_OK : (int)RBRP_ECUDA;
  };
  int rc = RBRP_OK;
  if (c.tc32) {   // fp32 residual form on tcgen05: one launch (b' <= 64) or 64-column parts
    const int nparts = c.bucketB > 64 ? (c.bucketB + 63) / 64 : 0;
    for (int part = nparts ? 0 : -1; part < std::max(nparts, 0); ++part) {
      if ((rc = lk(launch_pack_tc32((const float*)c.Qt, c.d, c.Qtc, c.st, s, part)))) return rc;
      if ((rc = lk(launch_proj_tc32((float*)c.Xres, c.ldr, c.Qtc, (float*)c.Lm, c.k_cap, c.n, c.d, c.dvec, c.st, s,
                                    c.lazy ? (const float*)c.X : nullptr, c.p->ld, part))))
        return rc;
      if (part < 0) break;
    }
    return RBRP_OK;
  }
  const int fmax = (c.paper || c.tiled) ? c.lp_max : 0;
  if (fmax > 0 && !fuse_pack(c) && (rc = lk(launch_pack_q(c.Qt, c.d, c.Qp, c.st, s)))) return rc;
  bool need_downdate = false;
  // b' above the widest 64-row-tile kernel (64 columns fp64, 32 fp32): balanced parts of
  // <= lp_max columns in sequence (RBRP_NO_PARTS=1: the two-kernel path instead)
  const bool parts = (c.paper || c.tiled) && c.lp_max >= 32 && c.bucketB > c.lp_max && !env_on("RBRP_NO_PARTS");
  for (int bk = 16; bk <= c.bucketB; bk *= 2) {
    if (bk > c.lp_max && parts) continue;
    if (bk <= fmax) {
      rc = lk(launch_lhat_paper((const T*)c.Xres, c.ldr, c.Qp, c.Lm, c.k_cap, c.n, c.d, c.dvec, c.st, bk,
                                !c.paper, s, c.lazy ? (const T*)c.X : nullptr, c.p->ld));
    } else if (c.use_mma) {
      rc = lk(launch_lhat_mma((const double*)c.Xres, c.ldr, (const double*)c.Qt, c.n, c.d, (double*)c.Lm,
                              c.k_cap, c.st, bk, s));
      if (!rc && !c.paper)
        rc = lk(launch_update_mma((double*)c.Xres, c.ldr, (const double*)c.Qt, (const double*)c.Lm,
                                  c.k_cap, c.n, c.d, c.dvec, c.st, bk, s));
      need_downdate = c.paper;
    } else {
      rc = lk(launch_lhat<T>(c.Xres, c.ldr, c.Qt, c.n, c.d, c.Lm, c.k_cap, c.st, bk, s));
      if (!rc && !c.paper)
        rc = lk(launch_update<T>(c.Xres, c.ldr, c.Qt, c.Lm, c.k_cap, c.n, c.d, c.dvec, c.st, bk, s));
      need_downdate = c.paper;
    }
    if (rc) return rc;
  }
  // full parts of lp_max columns, then the remainder on the kernel of its bucket (every bucket
  // kernel is enqueued for every part; all but one exit at once)
  const int nparts = parts ? (c.bucketB + c.lp_max - 1) / c.lp_max : 0;
  for (int part = 0; part < nparts; ++part) {
    if ((rc = lk(launch_pack_q(c.Qt, c.d, c.Qp, c.st, s, part, 0, c.lp_max)))) return rc;
    for (int bk = 16; bk <= c.lp_max; bk *= 2) {
      if ((rc = lk(launch_lhat_paper((const T*)c.Xres, c.ldr, c.Qp, c.Lm, c.k_cap, c.n, c.d, c.dvec, c.st, bk,
                                     !c.paper, s, c.lazy ? (const T*)c.X : nullptr, c.p->ld, part, c.lp_max))))
        return rc;
    }
  }
  // paper form on the two-kernel path: l.16 downdate from the L-hat columns (the kernel
  // skips blocks whose bucket the fused kernel handled, which downdates in its epilogue)
  if (need_downdate) rc = lk(launch_downdate<T>(c.Lm, c.k_cap, c.n, c.dvec, c.st, fmax, s));
  return rc;
}

// The kernels of one block (Alg. 2 l.6-16), optionally followed by the next block's
// stop test and sample (l.3-5).  Every kernel reads its sizes from DevState and is a
// no-op once stop is set, so the sequence can be replayed blindly (graph body).
template <typename T>
int enqueue_block(Ctx<T>& c, SampleArgs& sa, cudaStream_t s, Prof* prof, int* nl, int* nproj,
                  bool with_sample) {
#define LK(x)                                  \
  do {                                         \
    ++*nl;                                     \
    if ((x) != cudaSuccess) return RBRP_ECUDA; \
  } while (0)
  const rbrp_problem* p = c.p;
  if (prof) prof->begin(2);
  FilterArgs fa;
  fa.st = c.st;
  fa.X = c.Xres;
  fa.ldx = c.ldr;
  fa.X0 = c.lazy ? c.X : nullptr;
  fa.ldx0 = p->ld;
  fa.Vg = nullptr;
  if (c.comm || c.paper) {
    if (c.comm) CK(cudaMemsetAsync(c.Vg, 0, (size_t)RBRP_MAX_B * c.d * 8, s));
    LK(launch_gather_rows<T>(c.Xres, c.ldr, c.St, c.n, p->row_offset, c.st, c.d, c.Vg, s));
    if (c.comm) {
      int rc = comm_allreduce_f64(c.comm, c.Vg, (int64_t)RBRP_MAX_B * c.d, s);
      if (rc) return rc;
    }
    // paper form, l.6: V = X(S_t,:)^T - Q Q^T X(S_t,:)^T (CGS2)
    if (c.paper) LK(launch_cgs2_rows<T>(c.Vg, c.d, c.Qall, c.k_cap, c.Ccgs, c.st, s));
    fa.Vg = c.Vg;
  }
  fa.S_t = c.St;
  fa.row_offset = p->row_offset;
  fa.d = c.d;
  fa.Gpart = c.Gpart;
  fa.G = c.G;
  fa.forced = (c.use_forced && c.force_blk) ? c.forced : nullptr;
  if (fa.forced) ++c.nforced;
  fa.piv = c.piv;
  fa.mass = c.mass;
  fa.R11 = c.R11;
  fa.Tg = c.Tg;
  fa.Ag = c.Ag;
  fa.Rtot = c.Rtot;
  fa.S = c.S;
  fa.Qt = c.Qt;
  fa.bp_pad = c.bucketB;
  fa.Qp = fuse_pack(c) ? c.Qp : nullptr;
  fa.dbg = c.dbg;
  LK(launch_filter_coop<T>(fa, s));
  if (prof) prof->end();
  // a4: projection + fused norms (l.13, l.16)
  if (prof) prof->begin(3);
  {
    int rc = enqueue_projection(c, s, nl);
    if (rc) return rc;
  }
  if (prof) prof->end();
  ++*nproj;
  if (prof) prof->begin(5);
  LK(launch_fixup<T>(c.paper ? nullptr : c.Xres, c.ldr, c.dvec, c.Lm, c.k_cap, c.Rtot, c.S, c.n, p->row_offset,
                     c.d, c.st, s));
  if (c.paper) {
    LK(launch_zero_prev<T>(c.Lm, c.k_cap, c.S, c.n, p->row_offset, c.st, s));
    LK(launch_append_q<T>(c.Qt, c.d, c.Qall, c.st, s));
  }
  if (!fuse_scan(c)) LK(launch_chunk_scan(c.dvec, c.n, c.chunk0, c.cpre, c.ctot, c.cpos, s));
  if (prof) prof->end();
  if (c.comm) {
    int rc = comm_allgather_chunks(c.comm, c.ctot, c.cpos, c.chunk0, (c.n + RBRP_CHUNK - 1) / RBRP_CHUNK,
                                   c.Ly->nchunks, s);
    if (rc) return rc;
  }
  if (with_sample) {
    if (prof) prof->begin(1);
    if (launch_block_sample(c, sa, s, nl) != cudaSuccess) return RBRP_ECUDA;
    if (prof) prof->end();
  }
#undef LK
  return RBRP_OK;
}

// ---------------------------------------------------------------------------------
// graph cache: one instantiated WHILE-loop graph per (problem, buffers, device)
// ---------------------------------------------------------------------------------
struct GraphKey {
  rbrp_problem p;
  const void* X;
  const void* ws;
  const void* aux;   // row-sharded graphs: the communicator
  uint64_t shards;   // row-sharded graphs: hash of every shard's X, workspace and rows
  uint64_t env;      // hash of the RBRP_* environment (the experiment knobs select kernels)
  int device, use_mma;
  bool operator==(const GraphKey& o) const { return memcmp(this, &o, sizeof(GraphKey)) == 0; }
};
// Entries are shared_ptr-owned: a caller keeps its entry alive across the launch even if
// another host thread evicts it from the cache meanwhile (cudaGraphExecDestroy of an
// in-flight graph frees it asynchronously on completion).
struct GraphEntry {
  GraphKey key;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  int launches_per_block = 0;
  unsigned long long stamp = 0;
  ~GraphEntry() {
    if (exec) cudaGraphExecDestroy(exec);
    if (g) cudaGraphDestroy(g);
  }
};
using GraphPtr = std::shared_ptr<GraphEntry>;
std::mutex g_graph_mu;
std::list<GraphPtr> g_graphs;
unsigned long long g_graph_clock = 0;
cudaStream_t g_capture_stream[256] = {};   // one capture stream per device (under g_graph_mu)

cudaStream_t capture_stream() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t& cs = g_capture_stream[dev & 255];
  if (!cs && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) cs = nullptr;
  return cs;
}

template <typename E>
void evict_lru(std::list<std::shared_ptr<E>>& cache, size_t cap) {
  while (cache.size() >= cap) {
    auto it = std::min_element(cache.begin(), cache.end(),
                               [](const std::shared_ptr<E>& a, const std::shared_ptr<E>& b) { return a->stamp < b->stamp; });
    cache.erase(it);   // the entry itself dies with its last holder
  }
}

// FNV-1a over the RBRP_* environment entries: a graph captured under one setting of the
// experiment knobs (§7.1 of DESIGN.md) is not replayed under another
uint64_t env_hash() {
  uint64_t h = 1469598103934665603ull;
  for (char** e = environ; e && *e; ++e) {
    if (strncmp(*e, "RBRP_", 5) != 0) continue;
    for (const char* c = *e; *c; ++c) {
      h ^= (unsigned char)*c;
      h *= 1099511628211ull;
    }
    h ^= 0xffu;
    h *= 1099511628211ull;
  }
  return h;
}

GraphKey make_key(const rbrp_problem* p, const void* X, const void* ws, int variant, const void* aux = nullptr,
                  uint64_t shards = 0) {
  GraphKey k;
  memset(&k, 0, sizeof(k));
  k.p = *p;
  k.p.replay_blocks = nullptr;
  k.p.replay_lens = nullptr;
  k.p.replay_pivots = nullptr;
  k.X = X;
  k.ws = ws;
  cudaGetDevice(&k.device);
  k.use_mma = variant;
  k.aux = aux;
  k.shards = shards;
  k.env = env_hash();
  return k;
}

// FNV-1a over the shard pointers and sizes: a graph captured for one set of in-process
// shards bakes every shard's X and workspace address into its kernels, not only shard 0's
uint64_t shard_hash(int nsh, const rbrp_problem* ps, void* const* Xs, char* const* wss) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    for (int i = 0; i < 8; ++i) {
      h ^= (v >> (8 * i)) & 0xffu;
      h *= 1099511628211ull;
    }
  };
  for (int i = 0; i < nsh; ++i) {
    mix((uint64_t)(uintptr_t)Xs[i]);
    mix((uint64_t)(uintptr_t)wss[i]);
    mix((uint64_t)ps[i].n_local);
    mix((uint64_t)ps[i].row_offset);
    mix((uint64_t)ps[i].ld);
  }
  return h;
}

// Returns the cached graph for key, building it if needed; nullptr if graphs are not
// usable (the caller then runs the eager loop — same kernels, host-driven).
template <typename T>
GraphPtr get_graph(Ctx<T>& c, SampleArgs sa, const GraphKey& key) {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  for (auto& e : g_graphs)
    if (e->key == key) {
      e->stamp = ++g_graph_clock;
      return e;
    }
  cudaStream_t cs = capture_stream();
  if (!cs) return nullptr;
  GraphPtr ep = std::make_shared<GraphEntry>();
  GraphEntry& e = *ep;
  e.key = key;
  cudaGraphConditionalHandle h;
  cudaGraphNode_t node;
  cudaGraph_t body = nullptr;
  if (cudaGraphCreate(&e.g, 0) != cudaSuccess) return nullptr;
  bool ok = cudaGraphConditionalHandleCreate(&h, e.g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
  if (ok) {
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    ok = cudaGraphAddNode(&node, e.g, nullptr, 0, &np) == cudaSuccess;
    if (ok) body = np.conditional.phGraph_out[0];
    ok = ok && body;
  }
  if (ok) {
    ok = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (ok) {
      sa.cond = (unsigned long long)h;
      sa.first = 0;
      sa.replay_len = -1;
      int nl = 0, nproj = 0;
      const int rc = enqueue_block<T>(c, sa, cs, nullptr, &nl, &nproj, true);
      cudaGraph_t cap = nullptr;
      const bool endok = cudaStreamEndCapture(cs, &cap) == cudaSuccess;
      ok = (rc == RBRP_OK) && endok;
      e.launches_per_block = nl;
    }
  }
  if (ok) ok = cudaGraphInstantiate(&e.exec, e.g, 0) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    return nullptr;   // ep's destructor releases what was created
  }
  evict_lru(g_graphs, 8);
  e.stamp = ++g_graph_clock;
  g_graphs.push_back(ep);
  return ep;
}

// Remark 5.2 trigger (reading R17): min |diag L_1| < 1e-12 max |diag L_1|
bool clip_needed(double dmin, double dmax) { return dmax > 0.0 && dmin < 1e-12 * dmax; }

// the nodes of g with no outgoing edge
std::vector<cudaGraphNode_t> sink_nodes(cudaGraph_t g) {
  size_t nn = 0, ne = 0;
  std::vector<cudaGraphNode_t> sinks;
  if (cudaGraphGetNodes(g, nullptr, &nn) != cudaSuccess) return sinks;
  std::vector<cudaGraphNode_t> nodes(nn);
  if (nn && cudaGraphGetNodes(g, nodes.data(), &nn) != cudaSuccess) return sinks;
  if (cudaGraphGetEdges(g, nullptr, nullptr, &ne) != cudaSuccess) return sinks;
  std::vector<cudaGraphNode_t> from(ne), to(ne);
  if (ne && cudaGraphGetEdges(g, from.data(), to.data(), &ne) != cudaSuccess) return sinks;
  for (auto n : nodes)
    if (std::find(from.begin(), from.end(), n) == from.end()) sinks.push_back(n);
  return sinks;
}

// Row-sharded block loop as one graph: outer WHILE (handle set by k_sample) whose body is
// [block kernels + collectives, k_sample per shard] followed by an inner WHILE node over the
// draw rounds (handle set by k_sample and k_draw_accept).  NCCL collectives are captured
// into the bodies.  nullptr if graphs are not usable here (the caller runs the eager loop).
template <typename T, class FB, class FS, class FR>
GraphPtr get_graph_dist(Ctx<T>* C, SampleArgs* SA, int nsh, rbrp_comm* comm, FB& blockf, FS& samplef, FR& roundf,
                        const GraphKey& key) {
  (void)C;
  (void)comm;
  std::lock_guard<std::mutex> lk(g_graph_mu);
  for (auto& e : g_graphs)
    if (e->key == key) {
      e->stamp = ++g_graph_clock;
      return e;
    }
  cudaStream_t cs = capture_stream();
  if (!cs) return nullptr;
  GraphPtr ep = std::make_shared<GraphEntry>();
  GraphEntry& e = *ep;
  e.key = key;
  if (cudaGraphCreate(&e.g, 0) != cudaSuccess) return nullptr;
  cudaGraphConditionalHandle h = 0, h2 = 0;
  cudaGraph_t body = nullptr, inner = nullptr;
  bool ok = cudaGraphConditionalHandleCreate(&h, e.g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
  if (ok) {
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    ok = cudaGraphAddNode(&node, e.g, nullptr, 0, &np) == cudaSuccess;
    if (ok) body = np.conditional.phGraph_out[0];
    ok = ok && body;
  }
  if (ok) ok = cudaGraphConditionalHandleCreate(&h2, body, 0, 0) == cudaSuccess;
  std::vector<SampleArgs> saved(SA, SA + nsh);
  for (int i = 0; i < nsh; ++i) {
    SA[i].cond = (unsigned long long)h;
    SA[i].cond2 = (unsigned long long)h2;
    SA[i].first = 0;
  }
  int nl = 0;
  if (ok) {   // outer body: the block, then the stop test / b_t of the next one
    ok = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (ok) {
      int rc = blockf(cs, &nl);
      if (!rc) rc = samplef(cs, -1, &nl);
      cudaGraph_t cap = nullptr;
      const bool endok = cudaStreamEndCapture(cs, &cap) == cudaSuccess;
      ok = rc == RBRP_OK && endok;
    }
  }
  if (ok) {   // ... then the draw rounds
    std::vector<cudaGraphNode_t> sinks = sink_nodes(body);
    cudaGraphNodeParams np2 = {};
    np2.type = cudaGraphNodeTypeConditional;
    np2.conditional.handle = h2;
    np2.conditional.type = cudaGraphCondTypeWhile;
    np2.conditional.size = 1;
    cudaGraphNode_t n2;
    ok = !sinks.empty() && cudaGraphAddNode(&n2, body, sinks.data(), sinks.size(), &np2) == cudaSuccess;
    if (ok) inner = np2.conditional.phGraph_out[0];
    ok = ok && inner;
  }
  if (ok) {
    ok = cudaStreamBeginCaptureToGraph(cs, inner, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (ok) {
      const int rc = roundf(cs, &nl);
      cudaGraph_t cap = nullptr;
      const bool endok = cudaStreamEndCapture(cs, &cap) == cudaSuccess;
      ok = rc == RBRP_OK && endok;
    }
  }
  for (int i = 0; i < nsh; ++i) SA[i] = saved[i];
  if (ok) ok = cudaGraphInstantiate(&e.exec, e.g, 0) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    return nullptr;
  }
  e.launches_per_block = nl;   // one draw round per block counted
  evict_lru(g_graphs, 8);
  e.stamp = ++g_graph_clock;
  g_graphs.push_back(ep);
  return ep;
}

// a6: W(S,:) = I, W(rest,:) = L_2 L_1^{-1} (Alg. 3; triangular inverse),
// or L_2 pinv_clip(L_1) when `clip` (Remark 5.2)
template <typename T>
int enqueue_W(Ctx<T>& c, const rbrp_problem* p, rbrp_comm* comm, void* W_out, int64_t k, cudaStream_t s,
              int* nl, bool clip = false) {
  const int64_t k_cap = c.k_cap;
  double* L1 = c.L1;
  T* LinvT = c.LinvT;
  ++*nl;
  CK(launch_gather_L1<T>(c.Lm, k_cap, c.S, k, c.n, p->row_offset, L1, s));
  if (comm) {
    int rc = comm_allreduce_f64(comm, L1, k * k, s);
    if (rc) return rc;
  }
  // K padded to a multiple of 8 for the FP64 tensor path: L_1^{-T} gets zero columns
  // [k, kp) and L's columns [k, kp) are zeroed (never written by the loop)
  const int64_t kp = (k + 7) / 8 * 8;
  if (clip) {
    *nl += 4;
    CK(launch_pinv_clip<T>(L1, k, LinvT, kp, c.Pinv, nullptr, s));   // dense pinv_clip(L_1)^T
  } else {
    ++*nl;
    CK(launch_trinv<T>(L1, k, LinvT, kp, c.st, s, c.Pinv));
  }
  const bool w_small = !force_simt() && kp <= k_cap && w_small_supported<T>(kp) && !env_on("RBRP_W_NOSMALL") &&
                       !env_on("RBRP_W_SIMT");
  if (kp > k && kp <= k_cap && c.n > 0 && !w_small)   // k_w_small reads columns [k, kp) as zeros
    CK(cudaMemset2DAsync(c.Lm + k, (size_t)k_cap * sizeof(T), 0, (size_t)(kp - k) * sizeof(T), (size_t)c.n, s));
  cudaError_t merr = cudaSuccess;
  ++*nl;
  if (w_small) {
    // K <= 128: L_1^{-T} resident in shared memory, one pass over L (k_w_small)
    CK(launch_w_small<T>(c.Lm, k_cap, LinvT, c.n, k, kp, (T*)W_out, k_cap, !clip, s));
  } else if (!force_simt() && kp <= k_cap && c.Wsc && !env_on("RBRP_W_NTMMA") && !env_on("RBRP_W_SIMT") &&
      gemm_lp_supported(c.Lm, k_cap, LinvT, kp, kp, w_min_k<T>())) {
    // lower_b: L_1^{-T} has zero chunks to skip; the clipped pinv is dense.  fp32: the same
    // passes with fp32 storage and fp64 DMMA arithmetic
    --*nl;
    CK(gemm_nt_lp(c.Lm, k_cap, LinvT, kp, (T*)W_out, k_cap, c.n, k, kp, c.Wsc, s, !clip, w_min_k<T>(), nl));
  } else if (sizeof(T) == 8 && !force_simt() && kp <= k_cap &&
             gemm_nt_mma((const double*)c.Lm, k_cap, (const double*)LinvT, kp, (double*)W_out, k_cap, c.n, k, kp, s,
                         &merr)) {
    CK(merr);
  } else {
    CK(launch_gemm_nt<T>(c.Lm, k_cap, LinvT, kp, (T*)W_out, k_cap, c.n, k, k, s));
  }
  ++*nl;
  CK(launch_w_identity<T>((T*)W_out, k_cap, c.S, k, c.n, p->row_offset, s));
  return RBRP_OK;
}

struct WGraph {
  GraphKey key;
  const void* W;
  int64_t k;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t exec = nullptr;
  int launches = 0;
  unsigned long long stamp = 0;
  ~WGraph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (g) cudaGraphDestroy(g);
  }
};
using WGraphPtr = std::shared_ptr<WGraph>;
std::list<WGraphPtr> g_wgraphs;

template <typename T>
WGraphPtr get_w_graph(Ctx<T>& c, const rbrp_problem* p, const GraphKey& key, void* W_out, int64_t k) {
  if (env_on("RBRP_NO_GRAPH")) return nullptr;
  std::lock_guard<std::mutex> lk(g_graph_mu);
  for (auto& e : g_wgraphs)
    if (e->key == key && e->W == W_out && e->k == k) {
      e->stamp = ++g_graph_clock;
      return e;
    }
  cudaStream_t cs = capture_stream();
  if (!cs) return nullptr;
  WGraphPtr ep = std::make_shared<WGraph>();
  WGraph& e = *ep;
  e.key = key;
  e.W = W_out;
  e.k = k;
  bool ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed) == cudaSuccess;
  if (ok) {
    const int rc = enqueue_W<T>(c, p, nullptr, W_out, k, cs, &e.launches);
    const bool endok = cudaStreamEndCapture(cs, &e.g) == cudaSuccess;
    ok = rc == RBRP_OK && endok && e.g;
  }
  if (ok) ok = cudaGraphInstantiate(&e.exec, e.g, 0) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    return nullptr;
  }
  evict_lru(g_wgraphs, 8);
  e.stamp = ++g_graph_clock;
  g_wgraphs.push_back(ep);
  return ep;
}

template <typename T>
int run(const rbrp_problem* p, void* Xv, char* ws, const Layout& Ly, rbrp_comm* comm,
        cudaStream_t s, int64_t* S_out, void* W_out, rbrp_report* rep) {
  HostMarks hm;
  Ctx<T> c;
  make_ctx<T>(c, p, Xv, ws, Ly, comm);
  hm.mark("ctx");
  const bool inplace = (p->flags & RBRP_INPLACE) != 0;
  const bool stamps = env_on("RBRP_DEBUG_STAMPS");
  const int64_t k_cap = c.k_cap;

  // pinned staging: [state][S_t][piv][log ...][S]
  const int mb = Ly.maxlog, b = p->b;
  size_t o = 0;
  auto carve = [&](size_t bytes) { size_t r = o; o = align256(o + bytes); return r; };
  const size_t o_st = carve(sizeof(DevState)), o_St = carve(RBRP_MAX_B * 8),
               o_piv = carve(RBRP_MAX_B * 4), o_bt = carve(mb * 4), o_bp = carve(mb * 4),
               o_rho = carve(mb * 8), o_lSt = carve((size_t)mb * b * 8), o_lpiv = carve((size_t)mb * b * 4),
               o_ts = carve((size_t)mb * 16), o_S = carve((size_t)k_cap * 8 + 8);
  char* hp = (char*)g_pinned.get(o);
  if (!hp) return RBRP_ECUDA;
  DevState* hst = (DevState*)(hp + o_st);
  int64_t* hSt = (int64_t*)(hp + o_St);
  int32_t* hpiv = (int32_t*)(hp + o_piv);

  memset(hst, 0, sizeof(DevState));
  hst->tau = p->tol > 0.0 ? p->tol : -1.0;
  hst->tau_b = p->tau_b;
  hst->k_cap = k_cap;
  hst->b = p->b;
  hst->ldiag_min = DBL_MAX;
  hst->ldiag_max = 0.0;
  CK(launch_set_state(*hst, c.st, s));   // the initial state as a kernel parameter

  Prof prof;
  prof.on = rep && rep->profile;
  prof.s = s;
  int nl = 0, nproj = 0;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));
  hm.mark("e0");

  // a0: d^(0), X_res <- X (Alg. 2 l.1-2)
  prof.begin(0);
  ++nl;
  CK(launch_init_norms<T>(c.X, p->ld, c.Xres, c.n, c.d, c.dvec, c.st, !inplace && !c.paper && !c.lazy, s));
  if (!fuse_scan(c)) {
    ++nl;
    CK(launch_chunk_scan(c.dvec, c.n, c.chunk0, c.cpre, c.ctot, c.cpos, s));
  }
  prof.end();
  if (comm) {
    int rc = comm_allgather_chunks(comm, c.ctot, c.cpos, c.chunk0, (c.n + RBRP_CHUNK - 1) / RBRP_CHUNK,
                                   Ly.nchunks, s);
    if (rc) return rc;
  }

  // replay: the ids of block blk are staged into Srep; the sampler copies them to S_t
  int64_t replay_pos = 0;
  auto stage_replay = [&](int blk) -> int {
    if (!p->replay_nblocks) return -1;
    if (blk >= p->replay_nblocks) return -2;
    const int len = p->replay_lens[blk];
    if (len < 1 || len > p->b) return RBRP_EREPLAY - 1000;
    if (cudaStreamSynchronize(s) != cudaSuccess) return RBRP_ECUDA - 1000;   // staging reuse
    for (int i = 0; i < len; ++i) {
      const int64_t id = p->replay_blocks[replay_pos + i];
      if (id < 0 || id >= p->n_global) return RBRP_EREPLAY - 1000;
      hSt[i] = id;
    }
    if (cudaMemcpyAsync(c.Srep, hSt, len * 8, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return RBRP_ECUDA - 1000;
    c.force_blk = p->replay_pivots && p->replay_pivots[replay_pos] >= 0;
    if (c.force_blk) {
      for (int i = 0; i < len; ++i) {
        hpiv[i] = p->replay_pivots[replay_pos + i];
        if (hpiv[i] < 0 || hpiv[i] >= len) return RBRP_EREPLAY - 1000;
      }
      if (cudaMemcpyAsync(c.forced, hpiv, len * 4, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return RBRP_ECUDA - 1000;
    }
    replay_pos += len;
    return len;
  };

  SampleArgs sa;
  make_sample_args<T>(sa, c, 0);
  int rl = stage_replay(0);
  if (rl < -100) return rl + 1000;
  sa.replay_len = rl;
  prof.begin(1);
  CK(launch_block_sample(c, sa, s, &nl));
  prof.end();

  sa.first = 0;
  const bool eager = p->replay_nblocks > 0 || prof.on || stamps || comm || env_on("RBRP_NO_GRAPH");
  GraphPtr ge;   // held until the end of the call (stays valid if another thread evicts it)
  // the key records the kernel variant too (environment knobs select alternatives)
  if (!eager) ge = get_graph<T>(c, sa, make_key(p, Xv, ws, (c.use_mma ? 1 : 0) | (c.tc32 ? 2 : 0) | (c.tiled ? 4 : 0) |
                                                              (c.lazy ? 8 : 0) | (c.paper ? 16 : 0)));
  if (ge) {
    // the whole block loop as one graph launch (conditional WHILE node), enqueued right
    // behind a0 and the first sample: no host round trip in between (a non-finite or
    // all-zero X stops the loop on the device -- the sampler's stop test fails on a NaN
    // or zero total -- and is reported after it)
    CK(cudaGraphLaunch(ge->exec, s));
  } else {
    CK(cudaMemcpyAsync(hst, c.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hst->nonfinite) return RBRP_ENONFINITE;
    if (!(hst->D0 > 0.0)) return RBRP_EDEGENERATE;
    int blk = 0;
    while (!hst->stop) {
      int rc = enqueue_block<T>(c, sa, s, prof.on ? &prof : nullptr, &nl, &nproj, false);
      if (rc) return rc;
      ++blk;
      rl = stage_replay(blk);
      if (rl < -100) return rl + 1000;
      sa.replay_len = rl;
      prof.begin(1);
      CK(launch_block_sample(c, sa, s, &nl));
      prof.end();
      CK(cudaMemcpyAsync(hst, c.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (stamps) {
        long long t[11];
        if (cudaMemcpy(t, c.dbg, sizeof(t), cudaMemcpyDeviceToHost) == cudaSuccess) {
          fprintf(stderr, "rbrp filter phases (us):");
          for (int i = 1; i < 11; ++i) fprintf(stderr, " %.2f", (t[i] - t[0]) * 1e-3);
          fprintf(stderr, "\n");
          long long u[8];
          if (cudaMemcpy(u, c.dbg + 32, sizeof(u), cudaMemcpyDeviceToHost) == cudaSuccess) {
            fprintf(stderr, "rbrp sample phases (us):");
            for (int i = 1; i < 8; ++i)
              if (i != 6) fprintf(stderr, " %.2f", (u[i] - u[0]) * 1e-3);
            fprintf(stderr, " rounds %lld\n", u[6]);
          }
        }
      }
    }
  }

  // read the state (k, flags) before W (written into the pinned staging by a kernel)
  hm.mark("loop_enqueued");
  {
    const CopySeg sg = {c.st, hst, sizeof(DevState)};
    ++nl;
    CK(launch_copy_segments(&sg, 1, s));
  }
  CK(cudaStreamSynchronize(s));
  hm.mark("loop_done");
  if (hst->nonfinite) return RBRP_ENONFINITE;
  if (!(hst->D0 > 0.0)) return RBRP_EDEGENERATE;
  const int64_t k = hst->k;
  const int nblocks = std::min(hst->t, Ly.maxlog);
  if (ge) {
    nl += ge->launches_per_block * hst->t;
    nproj += hst->t;
  }
  // a6: W (Alg. 3); in graph mode the W kernels are replayed from a cached graph (keyed by
  // the loop's graph, W_out and k), so the host does not launch them one by one while the
  // GPU waits behind the stop-test read-back
  uint32_t host_flags = 0;
  if (!(p->flags & RBRP_NO_W) && W_out && k > 0) {
    prof.begin(6);
    const bool clip = clip_needed(hst->ldiag_min, hst->ldiag_max);   // Remark 5.2 (R17)
    if (clip) host_flags |= RBRP_F_W_CLIPPED;
    WGraphPtr wg = (ge && !comm && !prof.on && !clip) ? get_w_graph<T>(c, p, ge->key, W_out, k) : nullptr;
    if (wg) {
      CK(cudaGraphLaunch(wg->exec, s));
      nl += wg->launches;
    } else {
      const int rc = enqueue_W<T>(c, p, comm, W_out, k, s, &nl, clip);
      if (rc) return rc;
    }
    prof.end();
  }
  // the report (S, state, block log) into the pinned staging buffer: one kernel writing the
  // host-mapped memory instead of one copy per array
  int64_t* hS = (int64_t*)(hp + o_S);
  const int nlog = std::max(nblocks, 1);
  const bool want_blocks = rep && (rep->block_idx || rep->block_piv);
  {
    CopySeg sg[kMaxCopySegs];
    int ns = 0;
    sg[ns++] = {c.S, hS, (size_t)std::max<int64_t>(k, 1) * 8};
    sg[ns++] = {c.st, hst, sizeof(DevState)};
    sg[ns++] = {c.log.bt, hp + o_bt, (size_t)nlog * 4};
    sg[ns++] = {c.log.bp, hp + o_bp, (size_t)nlog * 4};
    sg[ns++] = {c.log.rho, hp + o_rho, (size_t)nlog * 8};
    sg[ns++] = {c.log.ts, hp + o_ts, (size_t)nlog * 16};
    if (want_blocks) {
      sg[ns++] = {c.log.St, hp + o_lSt, (size_t)nlog * b * 8};
      sg[ns++] = {c.log.piv, hp + o_lpiv, (size_t)nlog * b * 4};
    }
    ++nl;
    CK(launch_copy_segments(sg, ns, s));
  }
  if (rep && rep->d_out && c.n > 0)   // the final d^(t) (residual squared row norms)
    CK(cudaMemcpyAsync(rep->d_out, c.dvec, (size_t)c.n * 8, cudaMemcpyDeviceToDevice, s));
  hm.mark("w_enqueued");
  CK(cudaEventRecord(e1, s));
  CK(cudaStreamSynchronize(s));
  hm.mark("done");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  memcpy(S_out, hS, (size_t)k * 8);
  if (rep) {
    rep->k = k;
    rep->fro2 = hst->D0;
    rep->resid_rel = hst->total / hst->D0;
    rep->nblocks = hst->t;
    rep->flags = hst->flags | host_flags | (c.nforced ? (uint32_t)RBRP_F_NEAR_TIE : 0u);
    rep->ms_total = ms;
    for (int i = 0; i < 8; ++i) rep->ms_phase[i] = 0.f;
    prof.collect(rep->ms_phase);
    rep->launches = nl;
    rep->proj_calls = nproj;
    const int32_t* lbt = (const int32_t*)(hp + o_bt);
    const int32_t* lbp = (const int32_t*)(hp + o_bp);
    const double* lrho = (const double*)(hp + o_rho);
    const long long* lts = (const long long*)(hp + o_ts);
    const int64_t* lSt = (const int64_t*)(hp + o_lSt);
    const int32_t* lpiv = (const int32_t*)(hp + o_lpiv);
    double proj = 0.0;
    for (int t = 0; t < nblocks; ++t) {
      const double pms = (lbp[t] > 0 && lts[2 * t + 1] > lts[2 * t]) ? (lts[2 * t + 1] - lts[2 * t]) * 1e-6 : 0.0;
      proj += pms;
      if (rep->proj_ms_blk && t < rep->max_blocks) rep->proj_ms_blk[t] = (float)pms;
      if (t < rep->max_blocks) {
        if (rep->b_t) rep->b_t[t] = lbt[t];
        if (rep->b_prime) rep->b_prime[t] = lbp[t];
        if (rep->rho) rep->rho[t] = lrho[t];
        for (int i = 0; want_blocks && i < b; ++i) {
          if (rep->block_idx) rep->block_idx[(int64_t)t * b + i] = lSt[(int64_t)t * b + i];
          if (rep->block_piv) rep->block_piv[(int64_t)t * b + i] = lpiv[(int64_t)t * b + i];
        }
      }
    }
    rep->proj_ms = (float)proj;
    rep->graph = ge ? 1 : 0;
  }
  return RBRP_OK;
}

// ---------------------------------------------------------------------------------
// Row-sharded run: nsh shards handled by this process.  With an NCCL
// communicator (one process per GPU) nsh == 1 and the exchange points are NCCL
// collectives; without one, nsh > 1 shards live on the current device (in-process
// emulation of nsh ranks: the exchange buffers are shared and written by the owners only,
// which is exactly what the collectives produce).  Per block: C1 chunk totals, C2
// candidate rows of every draw round (max), C3 V rows (sum), once for W: C5 L_1 (sum).
// Q_b is not broadcast: every shard runs the (deterministic) filter on identical data.
// ---------------------------------------------------------------------------------
template <typename T>
int run_dist(int nsh, const rbrp_problem* ps, void* const* Xs, char* const* wss, const Layout* Lys,
             rbrp_comm* comm, cudaStream_t s, int64_t* S_out, void* const* W_outs, rbrp_report* rep) {
  std::vector<Ctx<T>> C(nsh);
  std::vector<SampleArgs> SA(nsh);
  for (int h = 0; h < nsh; ++h) make_ctx<T>(C[h], &ps[h], Xs[h], wss[h], Lys[h], comm);
  const bool emul = comm == nullptr;
  if (emul)
    for (int h = 1; h < nsh; ++h) {   // exchange buffers shared with shard 0
      C[h].ctot = C[0].ctot;
      C[h].cpos = C[0].cpos;
      C[h].cprefix = C[0].cprefix;
      C[h].Vg = C[0].Vg;
      C[h].cand = C[0].cand;
      C[h].Srep = C[0].Srep;
      C[h].L1 = C[0].L1;
    }
  for (int h = 0; h < nsh; ++h) make_sample_args<T>(SA[h], C[h], 1);
  const rbrp_problem* p = &ps[0];
  const int64_t k_cap = C[0].k_cap;
  const int b = p->b, mb = Lys[0].maxlog;
  size_t o = 0;
  auto carve = [&](size_t bytes) { size_t r = o; o = align256(o + bytes); return r; };
  const size_t o_st = carve(sizeof(DevState) * nsh), o_St = carve(RBRP_MAX_B * 8),
               o_piv = carve(RBRP_MAX_B * 4), o_bt = carve(mb * 4), o_bp = carve(mb * 4),
               o_rho = carve(mb * 8), o_lSt = carve((size_t)mb * b * 8), o_lpiv = carve((size_t)mb * b * 4),
               o_ts = carve((size_t)mb * 16), o_S = carve((size_t)k_cap * 8 + 8);
  char* hp = (char*)g_pinned.get(o);
  if (!hp) return RBRP_ECUDA;
  DevState* hst = (DevState*)(hp + o_st);
  int64_t* hSt = (int64_t*)(hp + o_St);
  int32_t* hpiv = (int32_t*)(hp + o_piv);
  int nl = 0, nproj = 0;
#define LKD(x)                                 \
  do {                                         \
    ++nl;                                      \
    if ((x) != cudaSuccess) return RBRP_ECUDA; \
  } while (0)
#define RCD(x)              \
  do {                      \
    const int rc_ = (x);    \
    if (rc_) return rc_;    \
  } while (0)
  for (int h = 0; h < nsh; ++h) {
    DevState* hs = hst + h;
    memset(hs, 0, sizeof(DevState));
    hs->tau = p->tol > 0.0 ? p->tol : -1.0;
    hs->tau_b = p->tau_b;
    hs->k_cap = k_cap;
    hs->b = p->b;
    hs->ldiag_min = DBL_MAX;
    hs->ldiag_max = 0.0;
    CK(cudaMemcpyAsync(C[h].st, hs, sizeof(DevState), cudaMemcpyHostToDevice, s));
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));
  auto coll_chunks = [&](cudaStream_t ss) -> int {
    if (!comm) return RBRP_OK;
    return comm_allgather_chunks(comm, C[0].ctot, C[0].cpos, C[0].chunk0,
                                 (C[0].n + RBRP_CHUNK - 1) / RBRP_CHUNK, Lys[0].nchunks, ss);
  };
#define LKS(x)                                 \
  do {                                         \
    ++*nlp;                                    \
    if ((x) != cudaSuccess) return RBRP_ECUDA; \
  } while (0)
  // the kernels and collectives of one block on `ss`: a3 (V rows from their owners, C3;
  // the filter on every shard), a4 + fix-up + chunk scan per shard, C1.  Every kernel reads
  // its sizes from DevState and is a no-op once stop is set (graph-capturable).
  auto enqueue_dblock = [&](cudaStream_t ss, int* nlp) -> int {
    if (comm && cudaMemsetAsync(C[0].Vg, 0, (size_t)p->b * C[0].d * 8, ss) != cudaSuccess) return RBRP_ECUDA;
    for (int h = 0; h < nsh; ++h)   // lazy X_res: block 1's rows come from X itself (device-side test)
      LKS(launch_gather_rows<T>(C[h].Xres, C[h].ldr, C[h].St, C[h].n, ps[h].row_offset, C[h].st, C[h].d, C[h].Vg,
                                ss, C[h].lazy ? (const T*)C[h].X : nullptr, ps[h].ld));
    if (comm) {
      const int rc = comm_allreduce_f64(comm, C[0].Vg, (int64_t)p->b * C[0].d, ss);
      if (rc) return rc;
    }
    // paper form, l.6 (CGS2): once per distinct V buffer (in-process shards share one)
    if (C[0].paper) {
      for (int h = 0; h < nsh; ++h) {
        bool seen = false;
        for (int h2 = 0; h2 < h; ++h2) seen = seen || (C[h2].Vg == C[h].Vg);
        if (!seen) LKS(launch_cgs2_rows<T>(C[h].Vg, C[h].d, C[h].Qall, C[h].k_cap, C[h].Ccgs, C[h].st, ss));
      }
    }
    for (int h = 0; h < nsh; ++h) {
      Ctx<T>& c = C[h];
      FilterArgs fa;
      fa.st = c.st;
      fa.X = c.Xres;
      fa.ldx = c.ldr;
      fa.X0 = nullptr;
      fa.ldx0 = 0;
      fa.Vg = c.Vg;
      fa.S_t = c.St;
      fa.row_offset = ps[h].row_offset;
      fa.d = c.d;
      fa.Gpart = c.Gpart;
      fa.G = c.G;
      fa.forced = (c.use_forced && c.force_blk) ? c.forced : nullptr;
      if (fa.forced && h == 0) ++c.nforced;
      fa.piv = c.piv;
      fa.mass = c.mass;
      fa.R11 = c.R11;
      fa.Tg = c.Tg;
      fa.Ag = c.Ag;
      fa.Rtot = c.Rtot;
      fa.S = c.S;
      fa.Qt = c.Qt;
      fa.bp_pad = c.bucketB;
      fa.Qp = fuse_pack(c) ? c.Qp : nullptr;
      fa.dbg = nullptr;
      LKS(launch_filter_coop<T>(fa, ss));
    }
    // a4: projection, rank-local
    for (int h = 0; h < nsh; ++h) {
      Ctx<T>& c = C[h];
      {
        const int rc = enqueue_projection(c, ss, nlp);
        if (rc) return rc;
      }
      LKS(launch_fixup<T>(c.paper ? nullptr : c.Xres, c.ldr, c.dvec, c.Lm, c.k_cap, c.Rtot, c.S, c.n,
                          ps[h].row_offset, c.d, c.st, ss));
      if (c.paper) {
        LKS(launch_zero_prev<T>(c.Lm, c.k_cap, c.S, c.n, ps[h].row_offset, c.st, ss));
        LKS(launch_append_q<T>(c.Qt, c.d, c.Qall, c.st, ss));
      }
      LKS(launch_chunk_scan(c.dvec, c.n, c.chunk0, c.cpre, c.ctot, c.cpos, ss));
    }
    return coll_chunks(ss);
  };
  // stop test + b_t of the next block (l.3-4) on every shard
  auto enqueue_dsample = [&](cudaStream_t ss, int rl, int* nlp) -> int {
    for (int h = 0; h < nsh; ++h) {
      SA[h].replay_len = rl;
      if (emul) SA[h].S_rep = C[0].Srep;
      LKS(launch_sample(SA[h], ss));
      SA[h].first = 0;
    }
    return RBRP_OK;
  };
  // one draw round (l.5): kSampleRound draws resolved by their owners (C2: max), accepted
  // in draw order on every shard
  auto enqueue_dround = [&](cudaStream_t ss, int* nlp) -> int {
    const int ncand = emul ? 1 : nsh;
    for (int h = 0; h < ncand; ++h)
      if (cudaMemsetAsync(C[h].cand, 0xff, kSampleRound * 8, ss) != cudaSuccess) return RBRP_ECUDA;
    for (int h = 0; h < nsh; ++h) LKS(launch_draw_resolve(SA[h], ss));
    if (comm) {
      const int rc = comm_allreduce_max_i64(comm, C[0].cand, kSampleRound, ss);
      if (rc) return rc;
    }
    for (int h = 0; h < nsh; ++h) LKS(launch_draw_accept(SA[h], ss));
    return RBRP_OK;
  };
#undef LKS
  // a0
  for (int h = 0; h < nsh; ++h) {
    const bool inplace = (ps[h].flags & RBRP_INPLACE) != 0;
    LKD(launch_init_norms<T>(C[h].X, ps[h].ld, C[h].Xres, C[h].n, C[h].d, C[h].dvec, C[h].st,
                               !inplace && !C[h].paper && !C[h].lazy, s));
    LKD(launch_chunk_scan(C[h].dvec, C[h].n, C[h].chunk0, C[h].cpre, C[h].ctot, C[h].cpos, s));
  }
  RCD(coll_chunks(s));
  // replay ids: one staging buffer (shard 0's Srep; shared in emulation, per rank with NCCL)
  int64_t replay_pos = 0;
  auto stage_replay = [&](int blk) -> int {
    if (!p->replay_nblocks) return -1;
    if (blk >= p->replay_nblocks) return -2;
    const int len = p->replay_lens[blk];
    if (len < 1 || len > p->b) return RBRP_EREPLAY - 1000;
    if (cudaStreamSynchronize(s) != cudaSuccess) return RBRP_ECUDA - 1000;
    for (int i = 0; i < len; ++i) {
      const int64_t id = p->replay_blocks[replay_pos + i];
      if (id < 0 || id >= p->n_global) return RBRP_EREPLAY - 1000;
      hSt[i] = id;
    }
    if (cudaMemcpyAsync(C[0].Srep, hSt, len * 8, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return RBRP_ECUDA - 1000;
    const bool fb = p->replay_pivots && p->replay_pivots[replay_pos] >= 0;
    for (int h = 0; h < nsh; ++h) C[h].force_blk = fb;
    if (fb) {
      for (int i = 0; i < len; ++i) {
        hpiv[i] = p->replay_pivots[replay_pos + i];
        if (hpiv[i] < 0 || hpiv[i] >= len) return RBRP_EREPLAY - 1000;
      }
      for (int h = 0; h < nsh; ++h)
        if (cudaMemcpyAsync(C[h].forced, hpiv, len * 4, cudaMemcpyHostToDevice, s) != cudaSuccess)
          return RBRP_ECUDA - 1000;
    }
    replay_pos += len;
    return len;
  };
  // eager sampling: stop test, then draw rounds until the block is complete (one host read
  // of the loop state per round)
  auto sample = [&](int rl) -> int {
    RCD(enqueue_dsample(s, rl, &nl));
    if (rl >= 0 || rl == -2) return RBRP_OK;
    for (int round = 0;; ++round) {
      RCD(enqueue_dround(s, &nl));
      CK(cudaMemcpyAsync(hst, C[0].st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (hst->stop || hst->sample_done) break;
    }
    return RBRP_OK;
  };
  int rl = stage_replay(0);
  if (rl < -100) return rl + 1000;
  RCD(sample(rl));
  // errors: any shard saw NaN/Inf
  if (comm) RCD(comm_allreduce_sum_i32(comm, &C[0].st->nonfinite, 1, s));
  for (int h = 0; h < nsh; ++h) CK(cudaMemcpyAsync(hst + h, C[h].st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int h = 0; h < nsh; ++h)
    if (hst[h].nonfinite) return RBRP_ENONFINITE;
  if (!(hst->D0 > 0.0)) return RBRP_EDEGENERATE;

  // Graph mode (no replay): the whole block loop -- block kernels, collectives, the stop
  // test and the draw rounds -- is one CUDA-graph launch: an outer conditional WHILE node
  // (condition set by k_sample) whose body ends in an inner WHILE node over the draw rounds
  // (condition set by k_sample and k_draw_accept).  No host round trip per block.
  GraphPtr dg;
  if (!hst->stop && !p->replay_nblocks && !env_on("RBRP_NO_GRAPH"))
    dg = get_graph_dist<T>(C.data(), SA.data(), nsh, comm, enqueue_dblock, enqueue_dsample, enqueue_dround,
                           make_key(p, Xs[0], wss[0], 64 | (nsh << 8) | (C[0].lazy ? 8 : 0) | (C[0].paper ? 16 : 0) |
                                                           (C[0].tc32 ? 2 : 0) | (C[0].use_mma ? 1 : 0), comm,
                                    shard_hash(nsh, ps, Xs, wss)));
  if (dg) {
    CK(cudaGraphLaunch(dg->exec, s));
    CK(cudaMemcpyAsync(hst, C[0].st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (comm) RCD(comm_check(comm));
    nl += dg->launches_per_block * hst->t;
    nproj += hst->t;
  }
  int blk = 0;
  while (!hst->stop) {
    RCD(enqueue_dblock(s, &nl));
    ++nproj;
    ++blk;
    rl = stage_replay(blk);
    if (rl < -100) return rl + 1000;
    RCD(sample(rl));
    CK(cudaMemcpyAsync(hst, C[0].st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (comm) RCD(comm_check(comm));   // a failed collective surfaces as RBRP_ENCCL
  }
  const int64_t k = hst->k;
  const int nblocks = std::min(hst->t, mb);
  // a6: W — L_1 rows from their owners (C5), then W rank-local
  const bool want_W = !(p->flags & RBRP_NO_W) && W_outs && k > 0;
  const bool clip = want_W && clip_needed(hst->ldiag_min, hst->ldiag_max);   // Remark 5.2 (R17)
  if (want_W) {
    if (comm || nsh > 0) CK(cudaMemsetAsync(C[0].L1, 0, (size_t)k * k * 8, s));
    for (int h = 0; h < nsh; ++h)
      LKD(launch_gather_L1<T>(C[h].Lm, k_cap, C[h].S, k, C[h].n, ps[h].row_offset, C[h].L1, s));
    if (comm) RCD(comm_allreduce_f64(comm, C[0].L1, k * k, s));
    int lt_src = -1;   // in-process shards: the shard whose L_1^{-T} the others copy
    for (int h = 0; h < nsh; ++h) {
      Ctx<T>& c = C[h];
      if (!W_outs[h]) continue;
      const int64_t kp = (k + 7) / 8 * 8;
      // the Jacobi SVD and the blocked inverse work on L_1 in place: in-process shards (one
      // shared L_1) compute L_1^{-T} once and copy it
      if (emul && lt_src >= 0) {
        CK(cudaMemcpyAsync(c.LinvT, C[lt_src].LinvT, (size_t)k * kp * sizeof(T), cudaMemcpyDeviceToDevice, s));
      } else if (clip) {
        nl += 4;
        CK(launch_pinv_clip<T>(c.L1, k, c.LinvT, kp, c.Pinv, nullptr, s));
        lt_src = h;
      } else {
        LKD(launch_trinv<T>(c.L1, k, c.LinvT, kp, c.st, s, c.Pinv));
        lt_src = h;
      }
      if (kp > k && kp <= k_cap && c.n > 0)
        CK(cudaMemset2DAsync(c.Lm + k, (size_t)k_cap * sizeof(T), 0, (size_t)(kp - k) * sizeof(T), (size_t)c.n, s));
      cudaError_t merr = cudaSuccess;
      ++nl;
      if (!force_simt() && kp <= k_cap && w_small_supported<T>(kp) && !env_on("RBRP_W_NOSMALL") &&
          !env_on("RBRP_W_SIMT")) {
        CK(launch_w_small<T>(c.Lm, k_cap, c.LinvT, c.n, k, kp, (T*)W_outs[h], k_cap, !clip, s));
      } else if (!force_simt() && kp <= k_cap && c.Wsc && !env_on("RBRP_W_NTMMA") && !env_on("RBRP_W_SIMT") &&
          gemm_lp_supported(c.Lm, k_cap, c.LinvT, kp, kp, w_min_k<T>())) {
        --nl;
        CK(gemm_nt_lp(c.Lm, k_cap, c.LinvT, kp, (T*)W_outs[h], k_cap, c.n, k, kp, c.Wsc, s, !clip, w_min_k<T>(), &nl));
      } else if (sizeof(T) == 8 && !force_simt() && kp <= k_cap &&
                 gemm_nt_mma((const double*)c.Lm, k_cap, (const double*)c.LinvT, kp, (double*)W_outs[h], k_cap,
                             c.n, k, kp, s, &merr)) {
        CK(merr);
      } else {
        CK(launch_gemm_nt<T>(c.Lm, k_cap, c.LinvT, kp, (T*)W_outs[h], k_cap, c.n, k, k, s));
      }
      LKD(launch_w_identity<T>((T*)W_outs[h], k_cap, c.S, k, c.n, ps[h].row_offset, s));
    }
  }
  int64_t* hS = (int64_t*)(hp + o_S);
  CK(cudaMemcpyAsync(hS, C[0].S, (size_t)std::max<int64_t>(k, 1) * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hst, C[0].st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  const int nlog = std::max(nblocks, 1);
  const BlockLog& lg = C[0].log;
  CK(cudaMemcpyAsync(hp + o_bt, lg.bt, nlog * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hp + o_bp, lg.bp, nlog * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hp + o_rho, lg.rho, nlog * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hp + o_ts, lg.ts, nlog * 16, cudaMemcpyDeviceToHost, s));
  const bool want_blocks = rep && (rep->block_idx || rep->block_piv);
  if (want_blocks) {
    CK(cudaMemcpyAsync(hp + o_lSt, lg.St, (size_t)nlog * b * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hp + o_lpiv, lg.piv, (size_t)nlog * b * 4, cudaMemcpyDeviceToHost, s));
  }
  if (rep && rep->d_out && nsh == 1 && C[0].n > 0)
    CK(cudaMemcpyAsync(rep->d_out, C[0].dvec, (size_t)C[0].n * 8, cudaMemcpyDeviceToDevice, s));
  CK(cudaEventRecord(e1, s));
  CK(cudaStreamSynchronize(s));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  memcpy(S_out, hS, (size_t)k * 8);
  if (rep) {
    rep->k = k;
    rep->fro2 = hst->D0;
    rep->resid_rel = hst->total / hst->D0;
    rep->nblocks = hst->t;
    rep->flags = hst->flags | (clip ? (uint32_t)RBRP_F_W_CLIPPED : 0u) | (C[0].nforced ? (uint32_t)RBRP_F_NEAR_TIE : 0u);
    rep->ms_total = ms;
    for (int i = 0; i < 8; ++i) rep->ms_phase[i] = 0.f;
    rep->launches = nl;
    rep->proj_calls = nproj;
    const int32_t* lbt = (const int32_t*)(hp + o_bt);
    const int32_t* lbp = (const int32_t*)(hp + o_bp);
    const double* lrho = (const double*)(hp + o_rho);
    const long long* lts = (const long long*)(hp + o_ts);
    double proj = 0.0;
    for (int t = 0; t < nblocks; ++t) {
      const double pms = (lbp[t] > 0 && lts[2 * t + 1] > lts[2 * t]) ? (lts[2 * t + 1] - lts[2 * t]) * 1e-6 : 0.0;
      proj += pms;
      if (rep->proj_ms_blk && t < rep->max_blocks) rep->proj_ms_blk[t] = (float)pms;
      if (t < rep->max_blocks) {
        if (rep->b_t) rep->b_t[t] = lbt[t];
        if (rep->b_prime) rep->b_prime[t] = lbp[t];
        if (rep->rho) rep->rho[t] = lrho[t];
        for (int i = 0; want_blocks && i < b; ++i) {
          if (rep->block_idx) rep->block_idx[(int64_t)t * b + i] = ((const int64_t*)(hp + o_lSt))[(int64_t)t * b + i];
          if (rep->block_piv) rep->block_piv[(int64_t)t * b + i] = ((const int32_t*)(hp + o_lpiv))[(int64_t)t * b + i];
        }
      }
    }
    rep->proj_ms = (float)proj;
    rep->graph = dg ? 1 : 0;
  }
#undef LKD
#undef RCD
  return RBRP_OK;
}

}  // namespace

namespace {
struct FwLayout {
  size_t L1, LinvT, Pinv, S, diag, nclip, Wsc, total;
};
FwLayout fw_layout(rbrp_dtype dtype, int64_t k) {
  FwLayout f;
  const size_t w = dtype == RBRP_F64 ? 8 : 4;
  const int64_t kp = (k + 7) / 8 * 8;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + std::max<size_t>(bytes, 1));
    return o;
  };
  f.L1 = take((size_t)k * k * 8);
  f.LinvT = take((size_t)k * kp * w);
  f.Pinv = take(pinv_scratch_bytes(k));
  f.S = take((size_t)k * 8);
  f.diag = take(16);
  f.nclip = take(8);
  f.Wsc = take(gemm_lp_scratch_bytes(k, kp));
  f.total = off;
  return f;
}

template <typename T>
int form_w_run(const T* L, int64_t ldl, int64_t n, const int64_t* S, int64_t k, int method, T* W, int64_t ldw,
               char* ws, cudaStream_t s, uint32_t* flags, int32_t* nclip) {
  const FwLayout f = fw_layout(sizeof(T) == 8 ? RBRP_F64 : RBRP_F32, k);
  double* L1 = (double*)(ws + f.L1);
  T* LinvT = (T*)(ws + f.LinvT);
  int64_t* Sd = (int64_t*)(ws + f.S);
  double* dg = (double*)(ws + f.diag);
  int* ncl = (int*)(ws + f.nclip);
  const int64_t kp = (k + 7) / 8 * 8;
  CK(cudaMemcpyAsync(Sd, S, (size_t)k * 8, cudaMemcpyHostToDevice, s));
  CK(launch_gather_L1<T>(L, ldl, Sd, k, n, 0, L1, s));
  bool clip = method == 2;
  if (method == 0) {   // Remark 5.2 trigger (reading R17), decided on the host
    double h[2];
    CK(launch_diag_test(L1, k, dg, s));
    CK(cudaMemcpyAsync(h, dg, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    clip = clip_needed(h[0], h[1]);
  }
  CK(cudaMemsetAsync(ncl, 0, 4, s));
  if (clip) {
    CK(launch_pinv_clip<T>(L1, k, LinvT, kp, ws + f.Pinv, ncl, s));
  } else {
    CK(launch_trinv<T>(L1, k, LinvT, kp, nullptr, s, ws + f.Pinv));
  }
  // the ID's W GEMM (k_lhat64 / k_lhat_paper passes, or k_nt_mma for small fp64 k) when L's
  // rows can be read as k = kp columns (k % 8 == 0), else the CUDA-core tile GEMM
  cudaError_t merr = cudaSuccess;
  if (k == kp && !force_simt() && w_small_supported<T>(kp) && !env_on("RBRP_W_NOSMALL")) {
    CK(launch_w_small<T>(L, ldl, (const T*)LinvT, n, k, kp, W, ldw, !clip, s));
  } else if (k == kp && !force_simt() && gemm_lp_supported(L, ldl, (const T*)LinvT, kp, kp, w_min_k<T>())) {
    CK(gemm_nt_lp(L, ldl, (const T*)LinvT, kp, W, ldw, n, k, kp, ws + f.Wsc, s, !clip, w_min_k<T>()));
  } else if (sizeof(T) == 8 && k == kp && !force_simt() &&
             gemm_nt_mma((const double*)L, ldl, (const double*)LinvT, kp, (double*)W, ldw, n, k, kp, s, &merr)) {
    CK(merr);
  } else {
    CK(launch_gemm_nt<T>(L, ldl, LinvT, kp, W, ldw, n, k, k, s));
  }
  CK(launch_w_identity<T>(W, ldw, Sd, k, n, 0, s));
  int hn = 0;
  CK(cudaMemcpyAsync(&hn, ncl, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (flags) *flags = clip ? (uint32_t)RBRP_F_W_CLIPPED : 0u;
  if (nclip) *nclip = hn;
  return RBRP_OK;
}
}  // namespace

extern "C" {

int rbrp_version(void) { return (RBRP_VERSION_MAJOR << 16) | RBRP_VERSION_MINOR; }

const char* rbrp_strerror(int status) {
  switch (status) {
    case RBRP_OK: return "RBRP_OK";
    case RBRP_EINVAL: return "RBRP_EINVAL: invalid argument";
    case RBRP_ENONFINITE: return "RBRP_ENONFINITE: X contains NaN or Inf";
    case RBRP_EDEGENERATE: return "RBRP_EDEGENERATE: ||X||_F = 0";
    case RBRP_ENOMEM: return "RBRP_ENOMEM: workspace too small";
    case RBRP_ECUDA: return "RBRP_ECUDA: CUDA error";
    case RBRP_ENCCL: return "RBRP_ENCCL: NCCL error or NCCL unavailable";
    case RBRP_EREPLAY: return "RBRP_EREPLAY: inconsistent replay log";
    case RBRP_ENOTSUP: return "RBRP_ENOTSUP: option not built";
    default: return "RBRP: unknown status";
  }
}

int rbrp_workspace_size(const rbrp_problem* p, size_t* bytes) {
  int rc = validate(p);
  if (rc) return rc;
  if (!bytes) return RBRP_EINVAL;
  *bytes = make_layout(p).total;
  return RBRP_OK;
}

int rbrp_id(const rbrp_problem* p, void* X, void* workspace, size_t ws_bytes, rbrp_comm* comm,
            void* stream, int64_t* S_out, void* W_out, rbrp_report* rep) {
  int rc = validate(p);
  if (rc) return rc;
  if (!S_out || (p->n_local > 0 && !X) || !workspace) return RBRP_EINVAL;
  if (comm && (p->row_offset % RBRP_CHUNK) != 0) return RBRP_EINVAL;
  if (filter_coop_nsplit(p->d) > 148) return RBRP_ENOTSUP;   // d > 4736: one CTA per 32 columns
  Layout Ly = make_layout(p);
  if (ws_bytes < Ly.total) return RBRP_ENOMEM;
  if ((uintptr_t)workspace % 256) return RBRP_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (comm) {
    if (p->greedy) return RBRP_ENOTSUP;
    char* ws = (char*)workspace;
    void* Xs[1] = {X};
    void* Ws[1] = {W_out};
    if (p->dtype == RBRP_F64) return run_dist<double>(1, p, Xs, &ws, &Ly, comm, s, S_out, Ws, rep);
    return run_dist<float>(1, p, Xs, &ws, &Ly, comm, s, S_out, Ws, rep);
  }
  if (p->dtype == RBRP_F64)
    return run<double>(p, X, (char*)workspace, Ly, comm, s, S_out, W_out, rep);
  return run<float>(p, X, (char*)workspace, Ly, comm, s, S_out, W_out, rep);
}

// End-to-end entry with host buffers: X (host) -> a private device copy in the workspace
// (run in place: the copy becomes the residual), rbrp_id, W (device, in the workspace)
// -> W_host.  All copies are stream-ordered cudaMemcpy2DAsync calls on `stream`.
static rbrp_problem host_problem(const rbrp_problem* p) {
  rbrp_problem q = *p;
  q.flags |= RBRP_INPLACE;
  q.ld = p->d;
  return q;
}

int rbrp_workspace_size_host(const rbrp_problem* p, size_t* bytes) {
  int rc = validate(p);
  if (rc) return rc;
  if (!bytes) return RBRP_EINVAL;
  const rbrp_problem q = host_problem(p);
  const size_t w = p->dtype == RBRP_F64 ? 8 : 4;
  const size_t xb = align256((size_t)p->n_local * p->d * w);
  const size_t wb = (p->flags & RBRP_NO_W) ? 0 : align256((size_t)p->n_local * k_cap_of(p) * w);
  *bytes = xb + wb + make_layout(&q).total;
  return RBRP_OK;
}

int rbrp_id_host(const rbrp_problem* p, const void* X_host, void* workspace, size_t ws_bytes, rbrp_comm* comm,
                 void* stream, int64_t* S_out, void* W_host, rbrp_report* rep) {
  int rc = validate(p);
  if (rc) return rc;
  if (!S_out || (p->n_local > 0 && !X_host) || !workspace) return RBRP_EINVAL;
  if ((uintptr_t)workspace % 256) return RBRP_EINVAL;
  size_t need = 0;
  if ((rc = rbrp_workspace_size_host(p, &need))) return rc;
  if (ws_bytes < need) return RBRP_ENOMEM;
  const rbrp_problem q = host_problem(p);
  const size_t w = p->dtype == RBRP_F64 ? 8 : 4;
  const int64_t k_cap = k_cap_of(p);
  const bool want_W = !(p->flags & RBRP_NO_W) && W_host;
  char* ws = (char*)workspace;
  void* Xd = ws;
  const size_t xb = align256((size_t)p->n_local * p->d * w);
  void* Wd = (p->flags & RBRP_NO_W) ? nullptr : (void*)(ws + xb);
  const size_t wb = (p->flags & RBRP_NO_W) ? 0 : align256((size_t)p->n_local * k_cap * w);
  cudaStream_t s = (cudaStream_t)stream;
  if (p->n_local > 0)
    CK(cudaMemcpy2DAsync(Xd, (size_t)p->d * w, X_host, (size_t)p->ld * w, (size_t)p->d * w, (size_t)p->n_local,
                         cudaMemcpyHostToDevice, s));
  rc = rbrp_id(&q, Xd, ws + xb + wb, ws_bytes - xb - wb, comm, stream, S_out, want_W ? Wd : nullptr, rep);
  if (rc) return rc;
  const int64_t k = rep ? rep->k : 0;
  if (want_W && p->n_local > 0) {
    int64_t kk = k;
    if (!rep) {   // k = number of valid entries written to S_out is not known without a report
      kk = k_cap;
    }
    if (kk > 0)
      CK(cudaMemcpy2DAsync(W_host, (size_t)k_cap * w, Wd, (size_t)k_cap * w, (size_t)kk * w, (size_t)p->n_local,
                           cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  return RBRP_OK;
}

int rbrp_form_w_workspace_size(rbrp_dtype dtype, int64_t k, size_t* bytes) {
  if ((dtype != RBRP_F32 && dtype != RBRP_F64) || k < 1 || !bytes) return RBRP_EINVAL;
  *bytes = fw_layout(dtype, k).total;
  return RBRP_OK;
}

int rbrp_form_w(rbrp_dtype dtype, const void* L, int64_t ldl, int64_t n, const int64_t* S, int64_t k,
                int32_t method, void* W_out, int64_t ldw, void* workspace, size_t ws_bytes, void* stream,
                uint32_t* flags, int32_t* nclip) {
  if ((dtype != RBRP_F32 && dtype != RBRP_F64) || k < 1 || n < k || ldl < k || ldw < k || !L || !S || !W_out ||
      !workspace || method < 0 || method > 2)
    return RBRP_EINVAL;
  if ((uintptr_t)workspace % 256) return RBRP_EINVAL;
  if (ws_bytes < fw_layout(dtype, k).total) return RBRP_ENOMEM;
  for (int64_t i = 0; i < k; ++i)
    if (S[i] < 0 || S[i] >= n) return RBRP_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == RBRP_F64)
    return form_w_run<double>((const double*)L, ldl, n, S, k, method, (double*)W_out, ldw, (char*)workspace, s,
                              flags, nclip);
  return form_w_run<float>((const float*)L, ldl, n, S, k, method, (float*)W_out, ldw, (char*)workspace, s, flags,
                           nclip);
}

int rbrp_id_sharded(const rbrp_problem* p, int nshards, const int64_t* shard_rows, void* const* X,
                    void* const* workspace, size_t ws_bytes, void* stream, int64_t* S_out,
                    void* const* W_out, rbrp_report* rep) {
  if (!p || nshards < 1 || nshards > 64 || !shard_rows || !X || !workspace || !S_out) return RBRP_EINVAL;
  if (p->greedy) return RBRP_ENOTSUP;
  if (filter_coop_nsplit(p->d) > 148) return RBRP_ENOTSUP;
  std::vector<rbrp_problem> ps(nshards, *p);
  std::vector<Layout> Ly(nshards);
  std::vector<char*> ws(nshards);
  int64_t off = 0;
  for (int h = 0; h < nshards; ++h) {
    ps[h].n_local = shard_rows[h];
    ps[h].row_offset = off;
    if (shard_rows[h] < 0 || (h + 1 < nshards && shard_rows[h] % RBRP_CHUNK)) return RBRP_EINVAL;
    off += shard_rows[h];
    int rc = validate(&ps[h]);
    if (rc) return rc;
    if (shard_rows[h] > 0 && !X[h]) return RBRP_EINVAL;
    Ly[h] = make_layout(&ps[h]);
    if (ws_bytes < Ly[h].total) return RBRP_ENOMEM;
    ws[h] = (char*)workspace[h];
    if (!ws[h] || (uintptr_t)ws[h] % 256) return RBRP_EINVAL;
  }
  if (off != p->n_global) return RBRP_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->dtype == RBRP_F64)
    return run_dist<double>(nshards, ps.data(), X, ws.data(), Ly.data(), nullptr, s, S_out, W_out, rep);
  return run_dist<float>(nshards, ps.data(), X, ws.data(), Ly.data(), nullptr, s, S_out, W_out, rep);
}

}  // extern "C"
