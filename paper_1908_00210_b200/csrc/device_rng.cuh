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
    step();
    return out;
  }

  // the state transition alone (next() without its output). The reference's
  // in-place sequence (s2 ^= s0; s3 ^= s1; s1 ^= s2; s0 ^= s3; s2 ^= t;
  // s3 = rotl(s3, 45)) written as three-input XORs of the old words, one LOP3
  // per 32-bit half each (the compiler did not merge the in-place form)
  __host__ __device__ __forceinline__ static uint64_t xor3(uint64_t a, uint64_t b, uint64_t c) {
#ifdef __CUDA_ARCH__
    uint32_t lo, hi;  // explicit lop3: common-subexpression elimination would otherwise split these
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(lo) : "r"(static_cast<uint32_t>(a)), "r"(static_cast<uint32_t>(b)),
        "r"(static_cast<uint32_t>(c)));
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(hi) : "r"(static_cast<uint32_t>(a >> 32)),
        "r"(static_cast<uint32_t>(b >> 32)), "r"(static_cast<uint32_t>(c >> 32)));
    return (static_cast<uint64_t>(hi) << 32) | lo;
#else
    return a ^ b ^ c;
#endif
  }
  __host__ __device__ __forceinline__ void step() {
    const uint64_t t = s1 << 17;
    const uint64_t n1 = xor3(s1, s2, s0);  // s1 ^ (s2 ^ s0)
    const uint64_t n0 = xor3(s0, s3, s1);  // s0 ^ (s3 ^ s1)
    const uint64_t n2 = xor3(s2, s0, t);   // (s2 ^ s0) ^ t
    const uint64_t n3 = s3 ^ s1;
    s0 = n0;
    s1 = n1;
    s2 = n2;
    s3 = rotl64(n3, 45);
  }

  // Jump ahead J draws: the transition is linear over GF(2), so J steps are
  // one 256x256 bit matrix (xoshiro_jump_matrix). jm = the matrix in shared
  // memory as 256 columns of 8 uint32 (the state words' little-endian
  // halves); column c = the state J steps after the unit state with only
  // bit c set (bit c = bit c%32 of half c/32). Every lane reads the same
  // column at the same time (shared-memory broadcast).
  __device__ __forceinline__ void jump(const uint32_t* jm) {
    uint32_t o0 = 0, o1 = 0, o2 = 0, o3 = 0, o4 = 0, o5 = 0, o6 = 0, o7 = 0;
    const uint32_t w[8] = {static_cast<uint32_t>(s0), static_cast<uint32_t>(s0 >> 32),
                           static_cast<uint32_t>(s1), static_cast<uint32_t>(s1 >> 32),
                           static_cast<uint32_t>(s2), static_cast<uint32_t>(s2 >> 32),
                           static_cast<uint32_t>(s3), static_cast<uint32_t>(s3 >> 32)};
#pragma unroll
    for (int q = 0; q < 8; q++) {
      uint32_t x = w[q];
      const uint4* col = reinterpret_cast<const uint4*>(jm) + 2 * (q * 32 + 31);
#pragma unroll 8
      for (int b = 31; b >= 0; b--) {  // top bit first: m = all ones if bit b is set
        const uint32_t m = static_cast<uint32_t>(static_cast<int32_t>(x) >> 31);
        x <<= 1;
        const uint4 c0 = col[0], c1 = col[1];
        col -= 2;
        o0 ^= c0.x & m;
        o1 ^= c0.y & m;
        o2 ^= c0.z & m;
        o3 ^= c0.w & m;
        o4 ^= c1.x & m;
        o5 ^= c1.y & m;
        o6 ^= c1.z & m;
        o7 ^= c1.w & m;
      }
    }
    s0 = o0 | (static_cast<uint64_t>(o1) << 32);
    s1 = o2 | (static_cast<uint64_t>(o3) << 32);
    s2 = o4 | (static_cast<uint64_t>(o5) << 32);
    s3 = o6 | (static_cast<uint64_t>(o7) << 32);
  }
};

// Jump with the matrix pre-combined two columns at a time: tab = 128 chunks
// x 4 entries x 8 uint32, entry k of chunk c = XOR of the columns 2c, 2c+1
// selected by the bits of k (xoshiro_jump_table2). Half the ALU work of
// Xoshiro::jump; a chunk's 4 entries are one 128-byte shared-memory row, so
// the lanes' different entries never conflict.
__device__ __forceinline__ void xoshiro_jump2(Xoshiro& r, const uint32_t* tab) {
  uint32_t o0 = 0, o1 = 0, o2 = 0, o3 = 0, o4 = 0, o5 = 0, o6 = 0, o7 = 0;
  const uint32_t w[8] = {static_cast<uint32_t>(r.s0), static_cast<uint32_t>(r.s0 >> 32),
                         static_cast<uint32_t>(r.s1), static_cast<uint32_t>(r.s1 >> 32),
                         static_cast<uint32_t>(r.s2), static_cast<uint32_t>(r.s2 >> 32),
                         static_cast<uint32_t>(r.s3), static_cast<uint32_t>(r.s3 >> 32)};
#pragma unroll
  for (int q = 0; q < 8; q++) {
    uint32_t x = w[q];
    const uint4* row = reinterpret_cast<const uint4*>(tab) + q * 16 * 8;
#pragma unroll 4
    for (int i = 0; i < 16; i++) {
      const uint4* e = row + i * 8 + (x & 3u) * 2;
      x >>= 2;
      const uint4 c0 = e[0], c1 = e[1];
      o0 ^= c0.x;
      o1 ^= c0.y;
      o2 ^= c0.z;
      o3 ^= c0.w;
      o4 ^= c1.x;
      o5 ^= c1.y;
      o6 ^= c1.z;
      o7 ^= c1.w;
    }
  }
  r.s0 = o0 | (static_cast<uint64_t>(o1) << 32);
  r.s1 = o2 | (static_cast<uint64_t>(o3) << 32);
  r.s2 = o4 | (static_cast<uint64_t>(o5) << 32);
  r.s3 = o6 | (static_cast<uint64_t>(o7) << 32);
}

// Host: the two-column table for xoshiro_jump2 from a jump matrix (256 x 4
// uint64 columns) -> 128 x 4 x 4 uint64.
inline void xoshiro_jump_table2(const uint64_t* mat, uint64_t* tab) {
  for (int c = 0; c < 128; c++)
    for (int k = 0; k < 4; k++)
      for (int w = 0; w < 4; w++)
        tab[(c * 4 + k) * 4 + w] = ((k & 1) ? mat[(2 * c) * 4 + w] : 0) ^ ((k & 2) ? mat[(2 * c + 1) * 4 + w] : 0);
}

// Host: the J-step jump matrix for Xoshiro::jump (256 columns x 4 uint64).
inline void xoshiro_jump_matrix(uint64_t J, uint64_t* out) {
  for (int c = 0; c < 256; c++) {
    uint64_t e[4] = {0, 0, 0, 0};
    e[c / 64] = 1ull << (c % 64);
    Xoshiro r{e[0], e[1], e[2], e[3]};
    for (uint64_t i = 0; i < J; i++) r.step();
    out[4 * c + 0] = r.s0;
    out[4 * c + 1] = r.s1;
    out[4 * c + 2] = r.s2;
    out[4 * c + 3] = r.s3;
  }
}

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

// Throughput-mode draws (K2, K4): one Philox4x32-10 call per four visits of a
// lane (counter (sweep, 32 * quad + lane, 2, 0), key = the replica seed), 32
// bits per visit: tie coin = bit 0, a 31-bit uniform against the flip
// threshold's top 31 bits (tm >> 33; tm = thr * 2^11 + 2047).

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

} // namespace gdi
