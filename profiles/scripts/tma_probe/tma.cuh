// tma.cuh -- Tensor Memory Accelerator plumbing of the TMA probe (probe.cu); not part of
// the library: the probe showed why TMA does not fit the lean kernels.
//
// Every level array and class-type row of a dyadic hierarchy has an ODD
// pitch (2^k + 1 or 2^k elements at arbitrary offsets), so 2-D/3-D tensor
// maps cannot describe them (globalStrides must be multiples of 16 bytes).
// A 1-D tiled tensor map over the whole buffer can: its box may start at any
// element coordinate (the TMA unit absorbs the misalignment and zero-fills
// out-of-bounds elements), so a warp fetches each 32-element row segment it
// needs with ONE cp.async.bulk.tensor.1d -- no per-lane address arithmetic,
// no superset rows, no boundary branches -- into a shared-memory ring
// completed on an mbarrier with the transaction byte count.
#pragma once

#include <cuda.h>

#include <cstdint>

namespace mgrg {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
// make the barrier inits visible to the async proxy (the TMA unit)
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// one 1-D box of a tiled tensor map at element coordinate c -> smem
__device__ __forceinline__ void tma_load_1d(void *smem, const CUtensorMap *map, int32_t c,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2}], [%3];\n" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(smem_u32(bar))
      : "memory");
}

} // namespace mgrg
