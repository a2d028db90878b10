// Internal helper shared by libising and the pybind module: the reference's
// adjacency array is already the interleaved layout gdi_graph_create_pairs
// takes (graph.hpp:67: Neighbor{int32 node, int32 weight}).
#pragma once

#include <cstddef>
#include <cstdint>

#include "ising/ising.hpp"

namespace ising {

static_assert(sizeof(Neighbor) == 2 * sizeof(std::int32_t) && offsetof(Neighbor, node) == 0 &&
                  offsetof(Neighbor, weight) == sizeof(std::int32_t),
              "Neighbor must be two packed int32s (node, weight)");

inline const std::int32_t* adjacency_pairs(const Graph& g) {
  return reinterpret_cast<const std::int32_t*>(g.csr_adjacency().data());
}

}  // namespace ising
