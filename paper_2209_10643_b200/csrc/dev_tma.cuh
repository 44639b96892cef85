// dev_tma.cuh -- device helpers for TMA tensor loads and mbarriers (sm_100a),
// plus the host-side tensor-map encoder (driver entry point, no -lcuda).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace upir {

// ------------------------------------------------------------------ device
__device__ __forceinline__ unsigned tma_smem(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tma_mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(tma_smem(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void tma_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void tma_mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tma_smem(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tma_smem(bar)) : "memory");
}
__device__ __forceinline__ void tma_mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TW_%=;\n}\n" ::"r"(tma_smem(bar)),
      "r"(parity)
      : "memory");
}
// Wait that suspends the thread in the barrier unit (try_wait with a
// suspend-time hint) instead of spinning: for a producer thread whose wait
// spans a whole tile of consumer work, whose probe loop would otherwise take
// issue slots from the unit warps of its SM sub-partition (ncu: 40 M
// SYNCS/NANOSLEEP/BRA instructions per 7x7 stencil sweep with a nanosleep
// back-off).
__device__ __forceinline__ void tma_mbar_wait_backoff(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TWS_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra TWS_%=;\n}\n" ::"r"(tma_smem(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void tma_fence_proxy() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// 2-D tiled TMA load of the box at (c0 = inner/column, c1 = row) into smem.
__device__ __forceinline__ void tma_load_2d(void *dst, const void *tmap, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          tma_smem(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(tma_smem(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const void *tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(tmap) : "memory");
}

// ------------------------------------------------------------------ host
// Encode a 2-D row-major tensor map (dims {cols, rows}, row pitch in bytes).
bool encode_tmap_2d(CUtensorMap *out, CUtensorMapDataType dt, const void *base, uint64_t cols, uint64_t rows,
                    uint64_t pitch_bytes, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swz,
                    CUtensorMapL2promotion l2);

}  // namespace upir
