// Open-addressing set of undirected vertex pairs, used for duplicate-edge
// detection by the G-set parser, Graph::from_edges and the generators. It
// only has to answer "was this pair new?" exactly like the reference's
// std::unordered_set dedupe (graph.cpp:53-61, gen.cpp:19-29); iteration
// order is never observed.
#pragma once

#include <cstdint>
#include <vector>

namespace ising::detail {

class PairSet {
public:
  explicit PairSet(std::size_t expected) {
    std::size_t cap = 16;
    while (cap < expected * 2 + 16) cap <<= 1;
    slots_.assign(cap, kEmpty);
    mask_ = cap - 1;
  }

  static std::uint64_t key(std::int32_t a, std::int32_t b) {
    if (a > b) std::swap(a, b);
    return (static_cast<std::uint64_t>(static_cast<std::uint32_t>(a)) << 32) |
           static_cast<std::uint32_t>(b);
  }

  // True when the pair was not present before.
  bool insert(std::uint64_t k) {
    std::uint64_t h = k * 0x9e3779b97f4a7c15ULL;
    std::size_t i = static_cast<std::size_t>(h ^ (h >> 31)) & mask_;
    for (;;) {
      std::uint64_t& slot = slots_[i];
      if (slot == kEmpty) {
        slot = k;
        return true;
      }
      if (slot == k) return false;
      i = (i + 1) & mask_;
    }
  }

private:
  static constexpr std::uint64_t kEmpty = ~0ULL;
  std::vector<std::uint64_t> slots_;
  std::size_t mask_ = 0;
};

} // namespace ising::detail
