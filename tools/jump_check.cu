// Host check of the xoshiro256++ jump-ahead used by k1_window's producer
// (device_rng.cuh): for each distance J, the J-step bit matrix and its
// two-column table, applied the way the device code applies them, must equal
// J plain steps from several states. Prints "ok" or the first mismatch.
#include <cstdio>
#include <vector>

#include "device_rng.cuh"

using namespace gdi;

static void apply_matrix(const uint64_t* m, const Xoshiro& in, Xoshiro& out) {
  const uint64_t w[4] = {in.s0, in.s1, in.s2, in.s3};
  uint64_t o[4] = {0, 0, 0, 0};
  for (int c = 0; c < 256; c++)
    if ((w[c / 64] >> (c % 64)) & 1)
      for (int k = 0; k < 4; k++) o[k] ^= m[4 * c + k];
  out = Xoshiro{o[0], o[1], o[2], o[3]};
}

static void apply_table2(const uint64_t* t, const Xoshiro& in, Xoshiro& out) {
  const uint64_t w[4] = {in.s0, in.s1, in.s2, in.s3};
  uint64_t o[4] = {0, 0, 0, 0};
  for (int c = 0; c < 128; c++) {
    const int k = static_cast<int>((w[(2 * c) / 64] >> ((2 * c) % 64)) & 3);
    for (int q = 0; q < 4; q++) o[q] ^= t[(c * 4 + k) * 4 + q];
  }
  out = Xoshiro{o[0], o[1], o[2], o[3]};
}

int main() {
  for (uint64_t J : {1ull, 64ull, 96ull * 7, 192ull * 3, 256ull}) {
    std::vector<uint64_t> m(1024), t(2048);
    xoshiro_jump_matrix(J, m.data());
    xoshiro_jump_table2(m.data(), t.data());
    for (uint64_t seed : {1ull, 77ull, 0xdeadbeefull}) {
      Xoshiro ref = Xoshiro::stream(seed, 1), a, b;
      const Xoshiro start = ref;
      for (uint64_t i = 0; i < J; i++) ref.next();
      apply_matrix(m.data(), start, a);
      apply_table2(t.data(), start, b);
      const bool ok = a.s0 == ref.s0 && a.s1 == ref.s1 && a.s2 == ref.s2 && a.s3 == ref.s3 && b.s0 == ref.s0 &&
                      b.s1 == ref.s1 && b.s2 == ref.s2 && b.s3 == ref.s3;
      if (!ok) {
        std::printf("mismatch J=%llu seed=%llu\n", static_cast<unsigned long long>(J),
                    static_cast<unsigned long long>(seed));
        return 1;
      }
    }
  }
  std::printf("ok\n");
  return 0;
}
