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

// In-order decisions of 32 consecutive visits (one per lane) against one
// counter: visit i sees G_i = G + (the changes of visits 0..i-1), as in the
// sequential visit_node (anneal.cpp:95-118). A visit's choice depends on G
// only through one threshold: with X = a4*own + b*field, diff = a4*G - X, so
// c = +1 iff G <= U (U = floor((X - 1)/a4), or floor(X/a4) when the tie coin
// says +1), and G_{i+1} = G_i + (G_i <= U_i ? dL_i : dR_i).
//
// warp_seq_decide: the in-order scan over the 32 thresholds (two dependent
// instructions per step); each lane gets the counter its own visit sees.
// Exact for any number of changes. Callers first
// evaluate every lane against G and then against G + the changes of the lanes
// before it under that evaluation: when no decision moves, those are the
// in-order decisions (most chunks), and only otherwise run the scan (an
// evaluation loop inside this function, and a scan starting at the first
// unsettled lane, both measured slower). Returns the lane's final spin (own
// when !live); advances G. (a4, b and the fields are bounded so that
// a4 * (|G| + 1) + b * |field| < 2^31.)
__device__ __forceinline__ int floor_div(int x, int a) { return x >= 0 ? x / a : -((-x + a - 1) / a); }
// The scan is run by lane 0 alone on the thresholds staged in shared memory
// (buf: 32 int2 + 32 int per warp, 16-byte aligned; 128-bit loads and
// stores): ~4 instructions per step once, instead of every lane running it
// redundantly on shuffled thresholds (~10 instructions per step, two
// shuffles): K2 pooled G22 18.7 -> 18.0 ms, G55 41.2 -> 37.5 ms, K4 M1
// 1.239 -> 1.221 ms.
__device__ __forceinline__ int warp_seq_decide(int own, int f, bool live, bool coin, bool flip, int& G, int a4,
                                                     int bb, int lane, int2* buf, int* gout) {
  const int X = a4 * own + bb * f;
  int U;
  if (a4 == 1)
    U = coin ? X : X - 1;
  else if (a4 > 0)
    U = floor_div(coin ? X : X - 1, a4);
  else
    U = (X > 0 || (X == 0 && coin)) ? 0x7fffffff : static_cast<int>(0x80000000u);
  const int cL = flip ? -1 : 1;
  const int dL = live ? cL - own : 0, dR = live ? -cL - own : 0;
  buf[lane] = make_int2(U, (dL + 2) | ((dR + 2) << 4));
  __syncwarp();
  int g = G;
  if (lane == 0) {
    const int4* b4 = reinterpret_cast<const int4*>(buf);
    int4* g4 = reinterpret_cast<int4*>(gout);
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int4 e0 = b4[2 * q], e1 = b4[2 * q + 1];  // entries 4q .. 4q + 3
      int4 out;
      out.x = g;
      g += g <= e0.x ? (e0.y & 15) - 2 : (e0.y >> 4) - 2;
      out.y = g;
      g += g <= e0.z ? (e0.w & 15) - 2 : (e0.w >> 4) - 2;
      out.z = g;
      g += g <= e1.x ? (e1.y & 15) - 2 : (e1.y >> 4) - 2;
      out.w = g;
      g += g <= e1.z ? (e1.w & 15) - 2 : (e1.w >> 4) - 2;
      g4[q] = out;
    }
  }
  __syncwarp();
  const int mine = gout[lane];
  G = __shfl_sync(0xffffffffu, g, 0);
  __syncwarp();  // (buf / gout reused by the next call)
  return live ? (mine <= U ? cL : -cL) : own;
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
