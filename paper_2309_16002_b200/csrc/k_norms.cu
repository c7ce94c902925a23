// k_norms.cu — a0 init (Alg. 2 l.1-2) and the chunked sampling CDF.
//
// k_init_norms: d^(0)(i) = ||x_i||_2^2 in fp64, X_res <- X, NaN/Inf detection.
//   One warp per row, 16-byte vector loads, 4 loads in flight per lane; HBM-bound
//   (algorithmic bytes per row: d*w read + d*w written (copy) + 8).
// k_chunk_scan: chunk-local inclusive prefix of d over RBRP_CHUNK rows and the
//   chunk totals, in a fixed summation order (bitwise reproducible for any number
//   of ranks: DESIGN.md R8 / SURVEY §8(e)).
#include "launch.cuh"

namespace rbrp {

template <typename T> struct V16;
template <> struct V16<double> {
  using type = double2;
  static constexpr int n = 2;
  __device__ static double sq(const double2& v) { return v.x * v.x + v.y * v.y; }
  __device__ static bool finite(const double2& v) { return isfinite(v.x) && isfinite(v.y); }
};
template <> struct V16<float> {
  using type = float4;
  static constexpr int n = 4;
  __device__ static double sq(const float4& v) {
    double a = v.x, b = v.y, c = v.z, e = v.w;
    return a * a + b * b + c * c + e * e;
  }
  __device__ static bool finite(const float4& v) {
    return isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
  }
};

template <typename T, bool VEC>
__global__ void __launch_bounds__(256) k_init_norms(const T* __restrict__ X, int64_t ldx,
                                                    T* __restrict__ Xres, int64_t n, int64_t d,
                                                    double* __restrict__ dvec, DevState* st,
                                                    int copy) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool ok = true;
  for (int64_t r = warp; r < n; r += nwarps) {
    const T* x = X + r * ldx;
    T* y = Xres + r * d;
    double s = 0.0;
    if (VEC) {
      using V = typename V16<T>::type;
      const V* xv = reinterpret_cast<const V*>(x);
      V* yv = reinterpret_cast<V*>(y);
      const int64_t nv = d / V16<T>::n;
      for (int64_t v = lane; v < nv; v += 128) {
        V a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (v + 32 * u < nv) a[u] = __ldcs(xv + v + 32 * u);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (v + 32 * u < nv) {
            s += V16<T>::sq(a[u]);
            ok = ok && V16<T>::finite(a[u]);
            if (copy) yv[v + 32 * u] = a[u];
          }
      }
    } else {
      for (int64_t c = lane; c < d; c += 32) {
        T a = x[c];
        double ad = (double)a;
        s += ad * ad;
        ok = ok && isfinite(ad);
        if (copy) y[c] = a;
      }
    }
    s = warp_sum(s);
    if (lane == 0) dvec[r] = s;
  }
  if (!ok) atomicOr(&st->nonfinite, 1);
}

template <typename T>
cudaError_t launch_init_norms(const T* X, int64_t ldx, T* Xres, int64_t n, int64_t d, double* dvec,
                              DevState* st, bool copy, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int per = 16 / (int)sizeof(T);
  bool vec = (d % per == 0) && (ldx % per == 0) && ((uintptr_t)X % 16 == 0) &&
             ((uintptr_t)Xres % 16 == 0);
  int64_t warps = n;
  int blocks = (int)std::min<int64_t>((warps + 7) / 8, 148 * 16);
  if (vec)
    k_init_norms<T, true><<<blocks, 256, 0, s>>>(X, ldx, Xres, n, d, dvec, st, copy ? 1 : 0);
  else
    k_init_norms<T, false><<<blocks, 256, 0, s>>>(X, ldx, Xres, n, d, dvec, st, copy ? 1 : 0);
  return cudaGetLastError();
}

// One CTA per chunk of RBRP_CHUNK rows; thread t owns rows [4t, 4t+4).
__global__ void __launch_bounds__(1024) k_chunk_scan(const double* __restrict__ dvec, int64_t n_local,
                                                     int64_t chunk0, double* __restrict__ cpre,
                                                     double* __restrict__ ctot,
                                                     int32_t* __restrict__ cpos) {
  __shared__ double wsum[32];
  __shared__ int cnt;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kChunk + 4 * tid;
  if (tid == 0) cnt = 0;
  double v[4];
  double s = 0.0;
  int c = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    v[e] = (base + e < n_local) ? dvec[base + e] : 0.0;
    s += v[e];
    c += v[e] > 0.0;
  }
  // warp inclusive scan (fixed pattern)
  double incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  double excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = 0.0;
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  const int wc = __reduce_add_sync(0xffffffffu, c);   // one shared atomic per warp
  if (lane == 0 && wc) atomicAdd(&cnt, wc);
  if (w == 0) {
    double x = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      double y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    wsum[lane] = x;
  }
  __syncthreads();
  double p = (w > 0 ? wsum[w - 1] : 0.0) + excl;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    p += v[e];
    if (base + e < n_local) cpre[base + e] = p;
  }
  if (tid == 1023) ctot[chunk0 + blockIdx.x] = p;   // = cpre of the chunk's last row
  __syncthreads();
  if (tid == 0) cpos[chunk0 + blockIdx.x] = cnt;
}

cudaError_t launch_chunk_scan(const double* dvec, int64_t n_local, int64_t chunk0, double* cpre,
                              double* ctot, int32_t* cpos, cudaStream_t s) {
  int nch = ceil_div(n_local, kChunk);
  if (nch == 0) return cudaSuccess;
  k_chunk_scan<<<nch, 1024, 0, s>>>(dvec, n_local, chunk0, cpre, ctot, cpos);
  return cudaGetLastError();
}

template cudaError_t launch_init_norms<double>(const double*, int64_t, double*, int64_t, int64_t,
                                               double*, DevState*, bool, cudaStream_t);
template cudaError_t launch_init_norms<float>(const float*, int64_t, float*, int64_t, int64_t,
                                              double*, DevState*, bool, cudaStream_t);

}  // namespace rbrp
