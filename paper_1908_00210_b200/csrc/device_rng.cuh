// Device random number generators.
//
//  * Xoshiro: xoshiro256++ with splitmix64 seeding, bit-identical to the
//    reference ising::Rng (reference proj/include/ising/rng.hpp:10-65). Used
//    by the exact kernel, whose output must match the CPU reference bit for
//    bit; the state lives in 8 registers of every lane that owns a replica.
//  * philox4x32_10: counter-based generator keyed by (seed, replica) with the
//    counter (sweep, vertex); used by the throughput kernel, where each
//    vertex visit needs an independent draw without sequential state.
#pragma once

#include <cstdint>

namespace gdi {

__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) {
  return (x << k) | (x >> (64 - k));
}

struct Xoshiro {
  uint64_t s0, s1, s2, s3;

  __host__ __device__ __forceinline__ static uint64_t splitmix(uint64_t& x) {
    uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }

  // rng.hpp:12-15 and :19-21
  __host__ __device__ __forceinline__ static Xoshiro stream(uint64_t seed, uint64_t id) {
    uint64_t x = seed ^ (0xd1b54a32d192ed03ULL * (id + 1));
    Xoshiro r;
    r.s0 = splitmix(x);
    r.s1 = splitmix(x);
    r.s2 = splitmix(x);
    r.s3 = splitmix(x);
    return r;
  }

  // rng.hpp:23-33
  __host__ __device__ __forceinline__ uint64_t next() {
    const uint64_t out = rotl64(s0 + s3, 23) + s0;
    const uint64_t t = s1 << 17;
    s2 ^= s0;
    s3 ^= s1;
    s1 ^= s2;
    s0 ^= s3;
    s2 ^= t;
    s3 = rotl64(s3, 45);
    return out;
  }
};

// Philox4x32-10 (Salmon et al., SC'11). Returns four 32-bit words.
struct Philox4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                 uint32_t c3, uint32_t k0, uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  constexpr uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int round = 0; round < 10; round++) {
    const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
    const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += W0;
    k1 += W1;
  }
  return {c0, c1, c2, c3};
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

} // namespace gdi
