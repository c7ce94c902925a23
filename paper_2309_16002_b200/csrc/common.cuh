// common.cuh — internal definitions shared by the librbrp kernels (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>

#include "../../include/rbrp.h"

namespace rbrp {

constexpr int kChunk = RBRP_CHUNK;   // rows per sampling chunk
constexpr int kMaxB = RBRP_MAX_B;    // largest block size
constexpr int64_t kJMax = 1 << 20;   // cap on draws per block (R6)

// Loop state kept on the device so that every decision of Alg. 2 (stop test,
// b_t, b') is taken by a kernel and the host only reads it once per block.
struct DevState {
  double D0;          // ||d^(0)||_1 (Alg. 2 l.2)
  double total;       // ||d^(t)||_1 (fixed-order chunk prefix, last entry)
  double tau;         // tolerance (<= 0: fixed rank)
  double tau_b;       // filter tolerance (< 0: 1/b_t)
  int64_t k;          // |S|
  int64_t k_cap;      // capacity / fixed rank
  int64_t npos;       // rows with d > 0
  int32_t t;          // block counter (l.4)
  int32_t b;          // block size parameter
  int32_t b_t;        // candidates in the current block
  int32_t b_prime;    // kept by the filter (l.8)
  int32_t stop;       // 1: loop ended
  uint32_t flags;     // RBRP_F_* bits
  int32_t nonfinite;  // set by k_init_norms
  int32_t draws;      // Philox draws consumed by the current block
  int32_t rank_def;   // pivoted Cholesky hit a non-positive pivot
  int32_t nlogged;    // blocks written to the device log
  uint32_t done_ctas; // CTA completion counter of the projection update kernel
  int32_t exhausted;  // distributed sampling: support <= b_t (take all positive rows)
  long long ts0, ts1; // %globaltimer at projection start / end (current block)
  int64_t jb;         // distributed sampling: next Philox draw index of the block
  int32_t sample_c;   // distributed sampling: candidates accepted so far
  int32_t sample_done;
  double ldiag_min;   // min / max |L_1(i,i)| = |R_V(i,i)| over the kept skeletons (k_fixup);
  double ldiag_max;   // the Remark 5.2 trigger of the clipped-pinv W (reading R17)
};

__device__ __forceinline__ long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (long long)t;
}

// the last CTA of a grid to call this records the projection end time
__device__ __forceinline__ void proj_end_stamp(DevState* st) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&st->done_ctas, 1u);
    if (prev == gridDim.x - 1) {
      st->ts1 = gtimer();
      st->done_ctas = 0;
    }
  }
}

// per-block device log (read by the host once, at the end of rbrp_id)
struct BlockLog {
  int32_t* bt;        // [maxlog]
  int32_t* bp;        // [maxlog]
  double* rho;        // [maxlog]
  int64_t* St;        // [maxlog][b]
  int32_t* piv;       // [maxlog][b]
  long long* ts;      // [maxlog][2]
  int maxlog, b;
};

// fp64 warp reduction in a fixed butterfly order (bitwise deterministic)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T> struct VecT;
template <> struct VecT<double> { using v2 = double2; };
template <> struct VecT<float> { using v2 = float2; };

// One-time per-device host initialisation (kernel attributes such as the dynamic
// shared-memory limit are per device, and a process may drive several GPUs from several
// host threads): f() runs under the lock the first time the current device calls once().
struct PerDevice {
  std::mutex mu;
  uint64_t done[4] = {0, 0, 0, 0};   // devices 0..255
  template <class F>
  cudaError_t once(F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    uint64_t& w = done[(dev >> 6) & 3];
    const uint64_t bit = 1ull << (dev & 63);
    if (w & bit) return cudaSuccess;
    const cudaError_t e = f();
    if (e == cudaSuccess) w |= bit;
    return e;
  }
};

// SM count of the current device (cached per device)
inline int device_sms() {
  static std::atomic<int> cache[256];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& c = cache[dev & 255];
  int v = c.load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
  c.store(v, std::memory_order_relaxed);
  return v;
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// b' > pw projected in parts (Q_b's rows are orthonormal, so the parts in sequence equal one
// projection up to rounding): full parts of pw rows of Q_b, then the remainder, part p = rows
// [r0, r0 + cnt) = [p pw, min((p + 1) pw, b')); pw = the widest projection kernel (64 for
// fp64, 32 for the fp32 DMMA fallback).  The remainder runs on the kernel of its own bucket
// (a 31-column remainder on the 32-column kernel: balanced parts of 48 would leave a quarter
// of the 64-column kernel's warps idle).  Returns false if part p does not exist for this b'.
__host__ __device__ inline bool part_range(int bpa, int part, int* r0, int* cnt, int pw = 32) {
  if (bpa <= pw) return false;
  const int np = (bpa + pw - 1) / pw;
  if (part >= np) return false;
  *r0 = part * pw;
  *cnt = bpa - *r0 < pw ? bpa - *r0 : pw;
  return true;
}

// padded block-width bucket used to instantiate the projection kernels
__host__ __device__ inline int bucket_of(int bp) {
  return bp <= 16 ? 16 : bp <= 32 ? 32 : bp <= 64 ? 64 : 128;
}

}  // namespace rbrp
