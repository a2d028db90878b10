// Device-side graph loader (layout.cu): upload + validation, and the kernel
// layouts derived from the CSR on the GPU.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "devbuf.hpp"
#include "kernels.cuh"

namespace gdi {

// Result of the device validation pass (graph.cpp:47-61 invariants + stats).
struct GraphScan {
  unsigned bad;       // bit 0: offsets not monotone, 1: endpoint out of range, 2: self loop
  unsigned non_unit;  // some weight != 1
  unsigned non_pm1;   // some weight not in {-1, +1}
  int max_degree;
  unsigned long long max_abs_field;  // max_i sum_j |w_ij|
};

struct ThruLayout {
  DevBuf order, sell, sell_off, sell_w, edges, edge_w;
  // the CSR in position space (row p = vertex order[p], neighbours as their
  // positions, bit 31 = weight -1 on +-1 graphs) and vertex -> position
  DevBuf poff, pcol, ppos;
  long long slots = 0;  // int4 cells of SELL
};

struct PipeLayout {
  DevBuf win_pos, win_neg, fwd_pos, fwd_neg;
  // k1_window rows: SELL-32 over the natural vertex order (chunk c = vertices
  // 32c..32c+31, entry k of lane l at (wsell_off[c] + k) * 32 + l; padding
  // index n; -1 weights in bit 31 of the index)
  DevBuf wsell, wsell_off;
};

// K3 evaluation layout: the canonical edge list (u < v, row order), +1
// weights first: narrow = n <= 65536, each edge one word u | v << 16, else
// int2. wkind 1 (+-1): edges [0, mpos) have weight +1, [mpos, m) weight -1;
// wkind 2: per-edge int32 weights in w.
struct EvalLayout {
  DevBuf edges, w;
  long long m = 0, mpos = 0;
  bool narrow = false;
};

// Uploads the reference CSR (int64 offsets, int32 neighbours, optional int32
// weights), converts the offsets to int32 and validates on the device.
// `w` is released when every weight is 1.
// pairs != nullptr: interleaved {neighbour, weight} entries (the reference's
// Neighbor array, graph.hpp:67), split on the device; nbr / weights unused.
cudaError_t upload_and_scan(const int64_t* offsets, const int32_t* nbr, const int32_t* weights, const int32_t* pairs,
                            int n, int64_t nnz, DevBuf& off32, DevBuf& col, DevBuf& w, GraphScan* scan,
                            cudaStream_t st);

// K2/K4 layout. wkind: 0 unit, 1 +-1 (sign bit), 2 general weights.
// Returns cudaErrorInvalidValue when SELL would exceed 2^31 int4 cells.
cudaError_t build_thru_layout(const DevCsr& g, int64_t m, int wkind, ThruLayout* L, cudaStream_t st);

// K4 rows: the SELL layout with neighbour positions in the visit order
// (padding -> position 32 * ceil(n / 32), a zero word), the degree of the
// vertex at every position, and the canonical edges in position space (min
// position | -1 weight in bit 31, max position) sorted by the larger
// position (+ weights for general graphs): the finishing kernel's cut pass.
cudaError_t build_part_layout(const DevCsr& g, const ThruLayout& T, long long m, int wkind, DevBuf& psell,
                              DevBuf& pdeg, DevBuf& pedges, DevBuf& pedge_w, cudaStream_t st);
// number of position-space edges whose larger position is < lim
cudaError_t part_edges_below(const DevBuf& pedges, long long m, int lim, long long* count);

// k1_block row records (degree <= 4, n <= 32767 / 65535): per vertex its
// in-window +1 / -1 masks and 16-bit columns (bit 15 = weight -1).
cudaError_t build_block_rows(const DevCsr& g, DevBuf& rows, cudaStream_t st);

// K3 layout (see EvalLayout).
cudaError_t build_eval_layout(const DevCsr& g, int64_t m, int wkind, EvalLayout* L, cudaStream_t st);

// k1_window layout (every |w| == 1, n >= 2 * win).
cudaError_t build_pipe_layout(const DevCsr& g, int win, PipeLayout* L, cudaStream_t st);

}  // namespace gdi
