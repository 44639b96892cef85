// dev_peer.cuh -- system-scope signalling between ranks over NVLink peer
// memory (CUDA IPC mappings of the other ranks' buffers / peer windows).
// Writers publish with a release RMW after their data stores; readers poll
// with acquire loads (PTX memory model, .sys scope).
#pragma once
#include <stdint.h>

namespace upir {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(unsigned long long *p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin until *p >= target (acquire): later loads see what the writers
// published before their release.  A peer that never arrives (a rank that
// died or skipped a collective loop) traps the kernel after 60 s -- a
// reported CUDA error instead of a hung device.
__device__ __forceinline__ void wait_geq_sys(const unsigned long long *p, unsigned long long target) {
  if (ld_acquire_sys(p) >= target) return;
  const unsigned long long t0 = global_ns();
  while (ld_acquire_sys(p) < target) {
    __nanosleep(128);
    if (global_ns() - t0 > 60ull * 1000000000ull) __trap();
  }
}
// Order this thread's earlier generic-proxy accesses (incl. the acquire
// above) before later async-proxy (TMA) reads of global memory.
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

}  // namespace upir
