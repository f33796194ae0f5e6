// tma.cuh — Blackwell (sm_100a) tile staging: mbarrier transaction barriers and the TMA tensor copy
// global -> shared (cp.async.bulk.tensor ... mbarrier::complete_tx::bytes).  One thread issues the
// copies of a stage; the consumers wait on the stage's mbarrier phase.  No register staging, no
// per-thread address arithmetic for the fill, completion tracked in bytes.  (Plain cp.async.bulk row
// copies of 128-160 bytes were measured slower than per-thread cp.async: DESIGN.md §7.)
#pragma once
#include <cstdint>

namespace topt {
namespace tma {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make the initialised barriers visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one arrival that also announces `bytes` of incoming transactions for the current phase
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// block until the phase with parity `parity` of `bar` has completed
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// TMA bulk copy of `bytes` (multiple of 16, 16-byte aligned ends) global -> shared, completing on
// `bar` — for LARGE contiguous chunks only (per-request cost dominates 128-byte rows)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// TMA tensor copy: the box at coordinates (c0..c3) of the 4D tensor map `tm` -> shared `dst`
// (128-byte aligned), completing on `bar`
__device__ __forceinline__ void tensor4_g2s(void* dst, const void* tm, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace tma
}  // namespace topt
