// rbrp.cu — C ABI of librbrp.so (include/rbrp.h) and the host orchestration of
// Alg. 2 + Alg. 3.
//
// The host only sequences kernels on the caller's stream; every decision of the loop
// (stop test l.3, b_t l.4, sampling l.5, b' l.8, |S| l.14) is taken on the device in
// DevState.  One device->host read of DevState per block (the data-dependent stop).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

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
  size_t Xres = SIZE_MAX, dvec, cpre, ctot, cpos, cprefix, L, Qt, Vg, Gpart, G, Tg, Ag, R11, Rtot,
         piv, mass, St, S, forced, cand, st, L1 = SIZE_MAX, LinvT = SIZE_MAX, total;
  int nsplit, cw;
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
  L.cw = 32;
  L.nsplit = (int)((d + L.cw - 1) / L.cw);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + std::max<size_t>(bytes, 1));
    return o;
  };
  const size_t B = RBRP_MAX_B;
  if (!(p->flags & RBRP_INPLACE)) L.Xres = take((size_t)n * d * w);
  L.dvec = take((size_t)n * 8);
  L.cpre = take((size_t)n * 8);
  L.ctot = take((size_t)L.nchunks * 8);
  L.cpos = take((size_t)L.nchunks * 4);
  L.cprefix = take((size_t)L.nchunks * 8);
  L.L = take((size_t)n * L.k_cap * w);
  L.Qt = take(B * d * w);
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
  L.S = take((size_t)L.k_cap * 8);
  L.forced = take(B * 4);
  L.cand = take(4096 * 8);
  L.st = take(sizeof(DevState));
  if (!(p->flags & RBRP_NO_W)) {
    L.L1 = take((size_t)L.k_cap * L.k_cap * 8);
    L.LinvT = take((size_t)L.k_cap * L.k_cap * w);
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

// RBRP_FORCE_SIMT=1 selects the CUDA-core (DFMA/FFMA) projection kernels instead of DMMA
bool dbg_stamps() {
  const char* e = getenv("RBRP_DEBUG_STAMPS");
  return e && e[0] == '1';
}
bool force_simt() {
  const char* e = getenv("RBRP_FORCE_SIMT");
  return e && e[0] == '1';
}

// per-phase CUDA events on the caller's stream (report.profile)
struct Prof {
  bool on = false;
  cudaStream_t s = nullptr;
  std::vector<int> phase;
  std::vector<cudaEvent_t> ev;   // pairs (start, end)
  int open_phase = -1;
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

template <typename T>
int run(const rbrp_problem* p, void* Xv, char* ws, const Layout& Ly, rbrp_comm* comm,
        cudaStream_t s, int64_t* S_out, void* W_out, rbrp_report* rep) {
  const int64_t n = p->n_local, d = p->d, k_cap = Ly.k_cap;
  const bool inplace = (p->flags & RBRP_INPLACE) != 0;
  T* X = (T*)Xv;
  T* Xres = inplace ? X : (T*)(ws + Ly.Xres);
  const int64_t ldr = inplace ? p->ld : d;
  double* dvec = (double*)(ws + Ly.dvec);
  double* cpre = (double*)(ws + Ly.cpre);
  double* ctot = (double*)(ws + Ly.ctot);
  int32_t* cpos = (int32_t*)(ws + Ly.cpos);
  double* cprefix = (double*)(ws + Ly.cprefix);
  T* Lm = (T*)(ws + Ly.L);
  T* Qt = (T*)(ws + Ly.Qt);
  double* Vg = (double*)(ws + Ly.Vg);
  double* Gpart = (double*)(ws + Ly.Gpart);
  double* G = (double*)(ws + Ly.G);
  double* Tg = (double*)(ws + Ly.Tg);
  double* Ag = (double*)(ws + Ly.Ag);
  double* R11 = (double*)(ws + Ly.R11);
  double* Rtot = (double*)(ws + Ly.Rtot);
  int32_t* piv = (int32_t*)(ws + Ly.piv);
  double* mass = (double*)(ws + Ly.mass);
  int64_t* St = (int64_t*)(ws + Ly.St);
  int64_t* S = (int64_t*)(ws + Ly.S);
  int32_t* forced = (int32_t*)(ws + Ly.forced);
  DevState* st = (DevState*)(ws + Ly.st);

  // pinned staging: [state A][state B][S_t][piv][S]
  const size_t off_B = 256, off_St = 512, off_piv = off_St + RBRP_MAX_B * 8,
               off_S = off_piv + RBRP_MAX_B * 4;
  char* hp = (char*)g_pinned.get(off_S + (size_t)k_cap * 8 + 64);
  if (!hp) return RBRP_ECUDA;
  DevState* hA = (DevState*)hp;
  DevState* hB = (DevState*)(hp + off_B);
  int64_t* hSt = (int64_t*)(hp + off_St);
  int32_t* hpiv = (int32_t*)(hp + off_piv);
  int64_t* hS = (int64_t*)(hp + off_S);

  DevState h0;
  memset(&h0, 0, sizeof(h0));
  h0.tau = p->tol > 0.0 ? p->tol : -1.0;
  h0.tau_b = p->tau_b;
  h0.k_cap = k_cap;
  h0.b = p->b;
  *hA = h0;
  CK(cudaMemcpyAsync(st, hA, sizeof(DevState), cudaMemcpyHostToDevice, s));

  Prof prof;
  prof.on = rep && rep->profile;
  prof.s = s;
  int nl = 0, nproj = 0;
#define LK(x) \
  do {        \
    ++nl;     \
    CK(x);    \
  } while (0)
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));

  const int64_t chunk0 = p->row_offset / RBRP_CHUNK;
  // a0: d^(0), X_res <- X (Alg. 2 l.1-2)
  prof.begin(0);
  LK(launch_init_norms<T>(X, p->ld, Xres, n, d, dvec, st, !inplace, s));
  LK(launch_chunk_scan(dvec, n, chunk0, cpre, ctot, cpos, s));
  prof.end();
  if (comm) {
    int rc = comm_allgather_chunks(comm, ctot, cpos, chunk0, (n + RBRP_CHUNK - 1) / RBRP_CHUNK, Ly.nchunks, s);
    if (rc) return rc;
  }

  int64_t replay_pos = 0;
  auto stage_replay = [&](int blk) -> int {
    if (!p->replay_nblocks) return -1;
    if (blk >= p->replay_nblocks) return -2;
    const int len = p->replay_lens[blk];
    if (len < 1 || len > p->b) return RBRP_EREPLAY - 1000;
    for (int i = 0; i < len; ++i) {
      const int64_t id = p->replay_blocks[replay_pos + i];
      if (id < 0 || id >= p->n_global) return RBRP_EREPLAY - 1000;
      hSt[i] = id;
    }
    if (cudaMemcpyAsync(St, hSt, len * 8, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return RBRP_ECUDA - 1000;
    if (p->replay_pivots) {
      for (int i = 0; i < len; ++i) hpiv[i] = p->replay_pivots[replay_pos + i];
      if (cudaMemcpyAsync(forced, hpiv, len * 4, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return RBRP_ECUDA - 1000;
    }
    replay_pos += len;
    // the staging buffers are reused below: wait for the copies
    if (cudaStreamSynchronize(s) != cudaSuccess) return RBRP_ECUDA - 1000;
    return len;
  };

  SampleArgs sa;
  sa.st = st;
  sa.ctot = ctot;
  sa.cpos = cpos;
  sa.cprefix = cprefix;
  sa.nchunks = (int)Ly.nchunks;
  sa.cpre = cpre;
  sa.dvec = dvec;
  sa.n_local = n;
  sa.row_offset = p->row_offset;
  sa.S_t = St;
  sa.seed = p->seed;
  sa.first = 1;
  int rl = stage_replay(0);
  if (rl < -100) return rl + 1000;
  sa.replay_len = rl;
  prof.begin(1);
  LK(launch_sample(sa, s));
  prof.end();
  CK(cudaMemcpyAsync(hB, st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (hB->nonfinite) return RBRP_ENONFINITE;
  if (!(hB->D0 > 0.0)) return RBRP_EDEGENERATE;

  const int bucketB = bucket_of((int)std::min<int64_t>(p->b, k_cap));
  const bool use_forced = p->replay_pivots != nullptr;
  const bool use_mma = sizeof(T) == 8 && !force_simt() && projection_mma_supported(Xres, ldr, Qt, d);
  int nblocks = 0;
  while (!hB->stop) {
    // a3: gather V = X_res(S_t,:)^T, Gram, pivoted Cholesky + filter (l.6-9)
    prof.begin(2);
    FilterArgs fa;
    fa.st = st;
    fa.X = Xres;
    fa.ldx = ldr;
    fa.Vg = nullptr;
    if (comm) {
      LK(launch_gather_rows<T>(Xres, ldr, St, n, p->row_offset, st, d, Vg, s));
      int rc = comm_allreduce_f64(comm, Vg, (int64_t)RBRP_MAX_B * d, s);
      if (rc) return rc;
      fa.Vg = Vg;
    }
    fa.S_t = St;
    fa.row_offset = p->row_offset;
    fa.d = d;
    fa.Gpart = Gpart;
    fa.G = G;
    fa.forced = use_forced ? forced : nullptr;
    fa.piv = piv;
    fa.mass = mass;
    fa.R11 = R11;
    fa.Tg = Tg;
    fa.Ag = Ag;
    fa.Rtot = Rtot;
    fa.S = S;
    fa.Qt = Qt;
    fa.bp_pad = bucketB;
    fa.dbg = dbg_stamps() ? (long long*)(ws + Ly.cand) : nullptr;
    LK(launch_filter_coop<T>(fa, s));
    prof.end();
    // a4: projection + fused norms (l.13, l.16)
    prof.begin(3);
    for (int bk = 16; bk <= bucketB; bk *= 2) {
      if (use_mma)
        LK(launch_lhat_mma((const double*)Xres, ldr, (const double*)Qt, n, d, (double*)Lm, k_cap,
                           st, bk, s));
      else
        LK(launch_lhat<T>(Xres, ldr, Qt, n, d, Lm, k_cap, st, bk, s));
    }
    prof.end();
    prof.begin(4);
    for (int bk = 16; bk <= bucketB; bk *= 2) {
      if (use_mma)
        LK(launch_update_mma((double*)Xres, ldr, (const double*)Qt, (const double*)Lm, k_cap, n, d,
                             dvec, st, bk, s));
      else
        LK(launch_update<T>(Xres, ldr, Qt, Lm, k_cap, n, d, dvec, st, bk, s));
    }
    prof.end();
    ++nproj;
    prof.begin(5);
    LK(launch_fixup<T>(Xres, ldr, dvec, Lm, k_cap, Rtot, S, n, p->row_offset, d, st, s));
    LK(launch_chunk_scan(dvec, n, chunk0, cpre, ctot, cpos, s));
    prof.end();
    if (comm) {
      int rc = comm_allgather_chunks(comm, ctot, cpos, chunk0, (n + RBRP_CHUNK - 1) / RBRP_CHUNK, Ly.nchunks, s);
      if (rc) return rc;
    }
    // log this block before the next sample overwrites S_t
    const bool logit = rep && nblocks < rep->max_blocks;
    CK(cudaMemcpyAsync(hA, st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
    if (logit && (rep->block_idx || rep->block_piv)) {
      CK(cudaMemcpyAsync(hSt, St, RBRP_MAX_B * 8, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(hpiv, piv, RBRP_MAX_B * 4, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      const int bt = hA->b_t;
      for (int i = 0; i < p->b; ++i) {
        if (rep->block_idx) rep->block_idx[(int64_t)nblocks * p->b + i] = i < bt ? hSt[i] : -1;
        if (rep->block_piv) rep->block_piv[(int64_t)nblocks * p->b + i] = i < bt ? hpiv[i] : -1;
      }
    }
    // next block: stop test + sample (l.3-5)
    rl = stage_replay(nblocks + 1);
    if (rl < -100) return rl + 1000;
    sa.replay_len = rl;
    sa.first = 0;
    prof.begin(1);
    LK(launch_sample(sa, s));
    prof.end();
    CK(cudaMemcpyAsync(hB, st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (dbg_stamps()) {   // diagnostics: phase stamps of this block's filter call (ns)
      long long t[11];
      if (cudaMemcpy(t, ws + Ly.cand, sizeof(t), cudaMemcpyDeviceToHost) == cudaSuccess) {
        fprintf(stderr, "rbrp filter b_t=%d b'=%d phases (us):", hA->b_t, hA->b_prime);
        for (int i = 1; i < 11; ++i) fprintf(stderr, " %.2f", (t[i] - t[0]) * 1e-3);
        fprintf(stderr, "\n");
      }
    }
    if (logit) {
      if (rep->b_t) rep->b_t[nblocks] = hA->b_t;
      if (rep->b_prime) rep->b_prime[nblocks] = hA->b_prime;
      if (rep->rho) rep->rho[nblocks] = hB->total / hB->D0;
    }
    ++nblocks;
  }

  const int64_t k = hB->k;
  // a6: W (Alg. 3)
  if (!(p->flags & RBRP_NO_W) && W_out && k > 0) {
    double* L1 = (double*)(ws + Ly.L1);
    T* LinvT = (T*)(ws + Ly.LinvT);
    prof.begin(6);
    LK(launch_gather_L1<T>(Lm, k_cap, S, k, n, p->row_offset, L1, s));
    if (comm) {
      int rc = comm_allreduce_f64(comm, L1, k * k, s);
      if (rc) return rc;
    }
    LK(launch_trinv<T>(L1, k, LinvT, st, s));
    cudaError_t merr = cudaSuccess;
    if (sizeof(T) == 8 && !force_simt() &&
        gemm_nt_mma((const double*)Lm, k_cap, (const double*)LinvT, k, (double*)W_out, k_cap, n, k,
                    k, s, &merr)) {
      ++nl;
      CK(merr);
    } else {
      LK(launch_gemm_nt<T>(Lm, k_cap, LinvT, k, (T*)W_out, k_cap, n, k, k, s));
    }
    LK(launch_w_identity<T>((T*)W_out, k_cap, S, k, n, p->row_offset, s));
    prof.end();
  }
  CK(cudaMemcpyAsync(hS, S, (size_t)std::max<int64_t>(k, 1) * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hB, st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  CK(cudaEventRecord(e1, s));
  CK(cudaStreamSynchronize(s));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  memcpy(S_out, hS, (size_t)k * 8);
  if (rep) {
    rep->k = k;
    rep->fro2 = hB->D0;
    rep->resid_rel = hB->total / hB->D0;
    rep->nblocks = nblocks;
    rep->flags = hB->flags;
    rep->ms_total = ms;
    for (int i = 0; i < 8; ++i) rep->ms_phase[i] = 0.f;
    prof.collect(rep->ms_phase);
    rep->launches = nl;
    rep->proj_calls = nproj;
  }
#undef LK
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
  if (p->flags & RBRP_FORM_PAPER) return RBRP_ENOTSUP;
  if (p->greedy) return RBRP_ENOTSUP;
  if (comm && (p->row_offset % RBRP_CHUNK) != 0) return RBRP_EINVAL;
  if (comm) return RBRP_ENOTSUP;   // distributed sampler: not yet built
  if (filter_coop_nsplit(p->d) > 148) return RBRP_ENOTSUP;   // d > 4736: one CTA per 32 columns
  Layout Ly = make_layout(p);
  if (ws_bytes < Ly.total) return RBRP_ENOMEM;
  if ((uintptr_t)workspace % 256) return RBRP_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->dtype == RBRP_F64)
    return run<double>(p, X, (char*)workspace, Ly, comm, s, S_out, W_out, rep);
  return run<float>(p, X, (char*)workspace, Ly, comm, s, S_out, W_out, rep);
}

}  // extern "C"
