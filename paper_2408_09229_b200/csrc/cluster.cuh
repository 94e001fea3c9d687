// cluster.cuh -- thread-block-cluster primitives (sm_90+/sm_100a PTX) for
// the split fill: two CTAs of a cluster sample disjoint halves of the axes
// of the same runs and swap per-run partials through distributed shared
// memory (st.async into the partner CTA, completion counted on the
// partner's mbarrier).
#pragma once
#include <cstdint>

namespace vpb {

__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// the shared::cluster address of `laddr` (a shared::cta address) in CTA `rank`
__device__ __forceinline__ uint32_t mapa_u32(uint32_t laddr, unsigned rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(laddr), "r"(rank));
  return r;
}

// whole-cluster barrier (every thread of every CTA), release/acquire
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init_cluster() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one arrival on the local barrier that also expects `bytes` of transactions
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// 16 bytes into the partner CTA's shared memory, counted on its barrier
__device__ __forceinline__ void st_async_f64x2(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
          raddr),
      "d"(a), "d"(b), "r"(rbar)
      : "memory");
}
__device__ __forceinline__ int ld_dsmem_s32(uint32_t raddr) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(raddr) : "memory");
  return v;
}

}  // namespace vpb
