// TMA bulk-copy helper shared by the sm_100a kernels (cp.async.bulk, SASS
// UBLKCP): the problem image, global -> shared, completing on an mbarrier.
#pragma once

#include <cstdint>

namespace loomk {

// The problem image arrives in shared memory through one TMA bulk copy
// (cp.async.bulk, SASS UBLKCP) completing on an mbarrier.
__device__ __forceinline__ void load_blob(uint8_t* smem, const uint8_t* g, uint32_t bytes, uint64_t* mbar) {
  const uint32_t mb = static_cast<uint32_t>(__cvta_generic_to_shared(mbar));
  const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    constexpr uint32_t kChunk = 16384;
    for (uint32_t off = 0; off < bytes; off += kChunk) {
      const uint32_t n = min(kChunk, bytes - off);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst + off),
          "l"(g + off), "r"(n), "r"(mb)
          : "memory");
    }
  }
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LOOM_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      "@!p bra LOOM_WAIT_%=;\n"
      "}\n" ::"r"(mb)
      : "memory");
}

}  // namespace loomk
