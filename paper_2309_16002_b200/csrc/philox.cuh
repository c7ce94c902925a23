// philox.cuh — Philox4x32-10 (Salmon et al., SC'11) and the U53 uniform map used by
// the sampler (reading R8): draw j of block t uses counter (j, t, 0, 0) and
// key (seed_lo, seed_hi); u = ((w1 << 32 | w0) >> 11) * 2^-53 in [0, 1).
#pragma once
#include <stdint.h>

namespace rbrp {

__host__ __device__ inline uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

__host__ __device__ inline uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    const uint32_t hi0 = mulhi32(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

__host__ __device__ inline double u53(uint4 w) {
  const uint64_t x = (((uint64_t)w.y << 32) | w.x) >> 11;
  return (double)x * 0x1.0p-53;
}

}  // namespace rbrp
