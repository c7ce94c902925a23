// mb_tmem_m64.cu — where does tcgen05.mma kind::tf32 with M = 64 (cta_group::1, A from TMEM)
// read its A rows and write its D rows in TMEM?  A(lane, 0) = lane + 1, B(n, 0) = 1 (n < 8), all
// other entries 0, so D(m, n) = the A value of the lane the MMA uses as row m.  Prints, for
// every TMEM lane, column 0 of D.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(float* out, int M) {
  __shared__ __align__(1024) float bsm[8 * 32];   // 8 rows x 128 B, SW128
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 8 * 32; i += blockDim.x) bsm[i] = 0.f;
  __syncthreads();
  if (tid < 8) bsm[tid * 32 + ((0 ^ (tid & 7)) * 4)] = 1.0f;   // B(n, k = 0) = 1
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(su32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tb = tslot;
  // A: TMEM columns [32, 40): lane l (of warp quarter w) row value l + 1 at k = 0
  {
    const uint32_t ta = tb + ((uint32_t)(32 * w) << 16) + 32;
    uint32_t r[8];
    for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(i == 0 ? (float)(32 * w + lane + 1) : 0.f);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(ta), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
    // D region [0, 8): zero
    uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(
                     tb + ((uint32_t)(32 * w) << 16)),
                 "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7])
                 : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (w == 0) {
    const uint32_t sa = su32(bsm);
    const uint64_t bdesc = (uint64_t)((sa & 0x3FFFFu) >> 4) | ((uint64_t)(16 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
                           (1ull << 46) | (2ull << 61);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(8 >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    asm volatile(
        "{\n .reg .pred p, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, 0, 0;\n"
        " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tb),
        "r"(tb + 32), "l"(bdesc), "r"(idesc)
        : "memory");
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(&bar))
        : "memory");
  }
  asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(su32(&bar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(tb + ((uint32_t)(32 * w) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  for (int i = 0; i < 8; ++i) out[tid * 8 + i] = __uint_as_float(r[i]);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(tb) : "memory");
}

int main() {
  float* out;
  cudaMallocManaged(&out, 128 * 8 * 4);
  for (int M : {128, 64}) {
    for (int i = 0; i < 128 * 8; ++i) out[i] = -1;
    k<<<1, 128>>>(out, M);
    cudaError_t e = cudaDeviceSynchronize();
    printf("M=%d err=%s\n", M, cudaGetErrorString(e));
    for (int l = 0; l < 128; ++l) {
      printf("%4.0f", out[l * 8]);
      if (l % 32 == 31) printf("   | lanes %d-%d, cols 0..7 of lane %d: %g %g %g %g\n", l - 31, l, l, out[l * 8],
                               out[l * 8 + 1], out[l * 8 + 7], out[l * 8 + 3]);
    }
  }
  return 0;
}
