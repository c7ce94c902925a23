// k_pack.cu — Q_b packed in the shared-memory image of the 64-row-tile projection
// kernel (k_lhat_paper.cu): one 1-D bulk copy per 64-column chunk instead of a gather.
//
// Q_b are the rows of the kept basis of Alg. 2 l.9; the projection of l.13/l.16
// streams them chunk by chunk from L2 for every 64-row tile of X_res.
// Two images per chunk (both zero-padded to PACK_ROWS rows and to the chunk width):
//   image 1 (L-hat pass, B fragments indexed by (row j, column pair)): row j, column c at
//           j * KC + (c ^ f(j)), f(j) = 8 (j & 1) ^ 4 ((j >> 1) & 3)  (conflict-free);
//   image 2 (update pass, B fragments indexed by (row pair p, column)): the 16-byte unit
//           (Q(2p, c), Q(2p+1, c)) of pair p and column c at p * KC + (c ^ 2 (p & 3)).
#include <algorithm>

#include "launch.cuh"

namespace rbrp {

namespace pk {
constexpr int KC = 64;          // columns per chunk (k_lhat_paper lp::KC)
constexpr int PACK_ROWS = 64;   // rows of the packed buffer (lp::PACK_ROWS)
}  // namespace pk


// part < 0: rows [0, b'), b' <= 64.  part >= 0 (b' > pw split into balanced parts of <= pw
// rows, part_range): rows [r0, r0 + cnt).
template <typename QT>
__global__ void k_pack_q(const QT* __restrict__ Qt, int64_t d, double* __restrict__ Qp,
                         const DevState* st, int part, int64_t ldq, int pw) {
  if (st->stop) return;
  const int bpa = st->b_prime;
  int bp, r0 = 0;
  if (part < 0) {
    bp = bpa;
    if (bp <= 0 || bp > pk::PACK_ROWS) return;
  } else {
    if (!part_range(bpa, part, &r0, &bp, pw)) return;
  }
  const int c = blockIdx.x, j = blockIdx.y, col = threadIdx.x;   // blockDim = KC
  const int64_t gc = (int64_t)c * pk::KC + col;
  const double v = (j < bp && gc < d) ? (double)Qt[(int64_t)(r0 + j) * ldq + gc] : 0.0;
  Qp[((int64_t)c * pk::PACK_ROWS + j) * pk::KC + pack_qswz(j, col)] = v;
  const int pr = j >> 1;
  double* Q2 = Qp + (int64_t)gridDim.x * pk::PACK_ROWS * pk::KC + (int64_t)c * pk::PACK_ROWS * pk::KC;
  Q2[(pr * pk::KC + (col ^ (2 * (pr & 3)))) * 2 + (j & 1)] = v;
}

struct CopySegs {
  CopySeg seg[kMaxCopySegs];
};
__global__ void k_copy_segments(CopySegs a) {
  const CopySeg sg = a.seg[blockIdx.y];
  const uint32_t* src = (const uint32_t*)sg.src;
  uint32_t* dst = (uint32_t*)sg.dst;
  const size_t nw = sg.bytes / 4;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

cudaError_t launch_copy_segments(const CopySeg* segs, int nseg, cudaStream_t s) {
  if (nseg <= 0) return cudaSuccess;
  if (nseg > kMaxCopySegs) return cudaErrorInvalidValue;
  CopySegs a = {};
  size_t mx = 0;
  for (int i = 0; i < nseg; ++i) {
    if (segs[i].bytes % 4) return cudaErrorInvalidValue;
    a.seg[i] = segs[i];
    mx = segs[i].bytes > mx ? segs[i].bytes : mx;
  }
  const unsigned gx = (unsigned)std::min<size_t>(std::max<size_t>((mx / 4 + 255) / 256, 1), 64);
  k_copy_segments<<<dim3(gx, (unsigned)nseg), 256, 0, s>>>(a);
  return cudaGetLastError();
}

__global__ void k_set_state(DevState v, DevState* st) {
  if (threadIdx.x == 0) *st = v;
}

cudaError_t launch_set_state(const DevState& v, DevState* st, cudaStream_t s) {
  k_set_state<<<1, 32, 0, s>>>(v, st);
  return cudaGetLastError();
}

static int pk_nc(int64_t d) { return (int)((d + pk::KC - 1) / pk::KC); }

size_t fused_pack_bytes(int64_t d) { return 2 * (size_t)pk_nc(d) * pk::PACK_ROWS * pk::KC * 8; }   // two images

cudaError_t launch_pack_q(const float* Qt, int64_t d, double* Qp, DevState* st, cudaStream_t s, int part,
                          int64_t ldq, int pw) {
  dim3 grid((unsigned)pk_nc(d), pk::PACK_ROWS);
  k_pack_q<float><<<grid, pk::KC, 0, s>>>(Qt, d, Qp, st, part, ldq > 0 ? ldq : d, pw);
  return cudaGetLastError();
}

cudaError_t launch_pack_q(const double* Qt, int64_t d, double* Qp, DevState* st, cudaStream_t s, int part,
                          int64_t ldq, int pw) {
  dim3 grid((unsigned)pk_nc(d), pk::PACK_ROWS);
  k_pack_q<double><<<grid, pk::KC, 0, s>>>(Qt, d, Qp, st, part, ldq > 0 ? ldq : d, pw);
  return cudaGetLastError();
}

}  // namespace rbrp
