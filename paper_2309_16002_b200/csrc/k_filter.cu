// k_filter.cu — a3 helper for the row-sharded path: gather the candidate rows
// (Alg. 2 l.6) so that an allreduce gives every rank V; the filter itself is
// k_filter_coop.cu.
//
#include "launch.cuh"

namespace rbrp {

// V rows: Vg(i,:) = X_res(S_t[i],:) in fp64, written by the owner of row S_t[i] only
// (multi-GPU: Vg is zeroed first and an allreduce(sum) then gives every rank the full V,
// SURVEY §8(e) C3; in-process shards share one Vg).
template <typename T>
__global__ void __launch_bounds__(256) k_gather_rows(const T* __restrict__ X, int64_t ldx,
                                                     const int64_t* __restrict__ rows,
                                                     int64_t n_local, int64_t row_offset,
                                                     const DevState* st, int64_t d,
                                                     double* __restrict__ Vg, const T* __restrict__ X0,
                                                     int64_t ldx0) {
  if (st->stop) return;
  const int i = blockIdx.x;
  if (i >= st->b_t) return;
  const int64_t r = rows[i] - row_offset;
  if (r < 0 || r >= n_local) return;   // another rank's row: left as is (zeroed before)
  if (X0 && st->t == 1) {   // lazy X_res copy: block 1's rows come from X itself
    X = X0;
    ldx = ldx0;
  }
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) Vg[(int64_t)i * d + c] = (double)X[r * ldx + c];
}

template <typename T>
cudaError_t launch_gather_rows(const T* X, int64_t ldx, const int64_t* rows, int64_t n_local,
                               int64_t row_offset, const DevState* st, int64_t d, double* Vg,
                               cudaStream_t s, const T* X0, int64_t ldx0) {
  k_gather_rows<T><<<kMaxB, 256, 0, s>>>(X, ldx, rows, n_local, row_offset, st, d, Vg, X0, ldx0);
  return cudaGetLastError();
}
template cudaError_t launch_gather_rows<double>(const double*, int64_t, const int64_t*, int64_t,
                                                int64_t, const DevState*, int64_t, double*,
                                                cudaStream_t, const double*, int64_t);
template cudaError_t launch_gather_rows<float>(const float*, int64_t, const int64_t*, int64_t,
                                               int64_t, const DevState*, int64_t, double*,
                                               cudaStream_t, const float*, int64_t);

}  // namespace rbrp
