// Microbenchmark (not product code): cycles per xoshiro256++ draw for one
// serial stream per lane, as used by the k1 producers.
#include <cstdio>
#include <cstdint>
#include "../paper_1908_00210_b200/csrc/device_rng.cuh"
using namespace gdi;

__device__ __forceinline__ uint64_t rotl_sh(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

// closed-form step on 32-bit halves (lo, hi) with funnel shifts:
//   s0' = s0^s1^s3, s1' = s0^s1^s2, s2' = s0^s2^(s1<<17), s3' = rotl(s1^s3, 45)
struct X32 {
  uint32_t a0, a1, b0, b1, c0, c1, d0, d1;  // s0..s3 as (lo, hi)
  __device__ __forceinline__ uint64_t next() {
    const uint64_t s0 = ((uint64_t)a1 << 32) | a0, s3 = ((uint64_t)d1 << 32) | d0;
    const uint64_t sum = s0 + s3;
    const uint32_t sl = (uint32_t)sum, sh = (uint32_t)(sum >> 32);
    const uint64_t res = (((uint64_t)__funnelshift_l(sl, sh, 23) << 32) | __funnelshift_l(sh, sl, 23)) + s0;
    const uint32_t tl = b0 << 17, th = __funnelshift_l(b0, b1, 17);
    const uint32_t x0 = b0 ^ d0, x1 = b1 ^ d1;  // s1 ^ s3
    const uint32_t na0 = a0 ^ x0, na1 = a1 ^ x1;
    const uint32_t nb0 = a0 ^ b0 ^ c0, nb1 = a1 ^ b1 ^ c1;
    const uint32_t nc0 = a0 ^ c0 ^ tl, nc1 = a1 ^ c1 ^ th;
    const uint32_t nd0 = __funnelshift_l(x0, x1, 13), nd1 = __funnelshift_l(x1, x0, 13);  // rotl 45
    a0 = na0; a1 = na1; b0 = nb0; b1 = nb1; c0 = nc0; c1 = nc1; d0 = nd0; d1 = nd1;
    return res;
  }
};

// variant 2: same closed form, shifts/rotations/adds on the FMA pipe
// (IMAD.WIDE by 2^k splits a 32-bit word across the 64-bit product; ORs of
// disjoint bit ranges become adds), XORs on the ALU pipe
__device__ __forceinline__ uint64_t wide(uint32_t x, uint32_t m) { return (uint64_t)x * m; }  // IMAD.WIDE.U32
__device__ __forceinline__ uint32_t lo32(uint64_t v) { return (uint32_t)v; }
__device__ __forceinline__ uint32_t hi32(uint64_t v) { return (uint32_t)(v >> 32); }
struct X2 {
  uint32_t a0, a1, b0, b1, c0, c1, d0, d1;
  __device__ __forceinline__ uint64_t next() {
    // sum = s0 + s3 (64-bit), res = rotl(sum, 23) + s0
    const uint64_t sum = (((uint64_t)a1 << 32) | a0) + (((uint64_t)d1 << 32) | d0);
    const uint64_t pl = wide((uint32_t)sum, 1u << 23), ph = wide((uint32_t)(sum >> 32), 1u << 23);
    const uint64_t rot = ((uint64_t)(lo32(ph) + hi32(pl)) << 32) | (lo32(pl) + hi32(ph));
    const uint64_t res = rot + (((uint64_t)a1 << 32) | a0);
    // t = s1 << 17
    const uint64_t tb = wide(b0, 1u << 17);
    const uint32_t tl = lo32(tb), th = b1 * (1u << 17) + hi32(tb);
    const uint32_t x0 = b0 ^ d0, x1 = b1 ^ d1;
    const uint32_t na0 = a0 ^ x0, na1 = a1 ^ x1;
    const uint32_t nb0 = a0 ^ b0 ^ c0, nb1 = a1 ^ b1 ^ c1;
    const uint32_t nc0 = a0 ^ c0 ^ tl, nc1 = a1 ^ c1 ^ th;
    // rotl(x, 45) = rotl(swap halves, 13)
    const uint64_t q0 = wide(x0, 1u << 13), q1 = wide(x1, 1u << 13);
    const uint32_t nd0 = lo32(q1) + hi32(q0), nd1 = lo32(q0) + hi32(q1);
    a0 = na0; a1 = na1; b0 = nb0; b1 = nb1; c0 = nc0; c1 = nc1; d0 = nd0; d1 = nd1;
    return res;
  }
};

template <int V>
__global__ void bench(uint64_t seed, int iters, unsigned long long* out, long long* cyc) {
  uint64_t acc = 0;
  long long t0 = clock64();
  if (V == 0) {
    Xoshiro r = Xoshiro::stream(seed + threadIdx.x, 1);
    for (int i = 0; i < iters; i++) acc ^= r.next();
  } else if (V == 2) {
    Xoshiro r = Xoshiro::stream(seed + threadIdx.x, 1);
    X2 x{(uint32_t)r.s0, (uint32_t)(r.s0 >> 32), (uint32_t)r.s1, (uint32_t)(r.s1 >> 32),
         (uint32_t)r.s2, (uint32_t)(r.s2 >> 32), (uint32_t)r.s3, (uint32_t)(r.s3 >> 32)};
    for (int i = 0; i < iters; i++) acc ^= x.next();
  } else {
    Xoshiro r = Xoshiro::stream(seed + threadIdx.x, 1);
    X32 x{(uint32_t)r.s0, (uint32_t)(r.s0 >> 32), (uint32_t)r.s1, (uint32_t)(r.s1 >> 32),
          (uint32_t)r.s2, (uint32_t)(r.s2 >> 32), (uint32_t)r.s3, (uint32_t)(r.s3 >> 32)};
    for (int i = 0; i < iters; i++) acc ^= x.next();
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  unsigned long long* d;
  long long* c;
  cudaMalloc(&d, 1024 * 8);
  cudaMalloc(&c, 8);
  for (int v = 0; v < 3; v++) {
    const int iters = 1 << 20;
    long long cyc = 0;
    unsigned long long h0[2];
    if (v == 0) bench<0><<<1, 32>>>(7, iters, d, c); else if (v == 1) bench<1><<<1, 32>>>(7, iters, d, c); else bench<2><<<1, 32>>>(7, iters, d, c);
    cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h0, d, 16, cudaMemcpyDeviceToHost);
    printf("variant %d: %.2f cycles/draw (one warp, 32 lanes)  check %016llx\n", v, (double)cyc / iters, h0[0]);
  }
  return 0;
}
