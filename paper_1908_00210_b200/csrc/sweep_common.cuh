// Device helpers shared by the sweep kernels.
#pragma once

#include <cstdint>

namespace gdi {

// visit_node's decision (reference anneal.cpp:104-127) on a precomputed
// diff = 4A * (G - own) - B * field: diff < 0 -> +1, > 0 -> -1, tie -> coin;
// then the random flip.
__device__ __forceinline__ int decide(int diff, bool coin, bool flip) {
  const int c = diff < 0 ? 1 : diff > 0 ? -1 : (coin ? 1 : -1);
  return flip ? -c : c;
}

// CTA-scope release/acquire on shared-memory words, by their shared::cta
// address (generic-address atomics compile to slower generic loads/stores).
__device__ __forceinline__ unsigned saddr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ int ld_acquire(unsigned a) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(unsigned a) {
  int v;
  asm volatile("ld.relaxed.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned a, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// Relaxed store; callers order it after a preceding fence or release.
__device__ __forceinline__ void st_relaxed(unsigned a, int v) {
  asm volatile("st.relaxed.cta.shared::cta.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

}  // namespace gdi
