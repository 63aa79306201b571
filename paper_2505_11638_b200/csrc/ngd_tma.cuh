// TMA / mbarrier helpers shared by the DMMA GEMM kernels (ngd_gemm.cu, ngd_phbg.cu).
#pragma once
#include <cuda.h>
#include <cstdint>

namespace ngd {
namespace tma {

__device__ __forceinline__ unsigned smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem(m)), "r"(count));
}
__device__ __forceinline__ void expect_tx(unsigned long long* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(unsigned long long* m) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem(m)) : "memory");
}
__device__ __forceinline__ void wait(unsigned long long* m, unsigned parity) {
  const unsigned a = smem(m);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void load2d(void* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem(m))
      : "memory");
}
__device__ __forceinline__ void load1d(void* dst, const void* src, unsigned bytes, unsigned long long* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem(dst)),
               "l"(src), "r"(bytes), "r"(smem(m))
               : "memory");
}
// orders this thread's earlier generic-proxy accesses to shared memory before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// element (mn, k) of a 128 x 16 stage tile loaded as one K-major TMA box (128-byte swizzle)
__device__ __forceinline__ int kmaj_off(int mn, int k) { return mn * 16 + ((((k >> 1) ^ (mn & 7)) << 1) | (k & 1)); }

}  // namespace tma
}  // namespace ngd
