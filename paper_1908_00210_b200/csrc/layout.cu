// Graph loader on the device (SURVEY.md §8(f)3 "loader throughput").
//
// gdi_graph_create uploads the reference CSR (graph.hpp:66-67: int64 row
// offsets, int32 neighbours, int32 weights) once and everything else is
// derived on the GPU:
//   * validation + statistics (graph.cpp:47-61 invariants: monotone offsets,
//     endpoints in range, no self loops; unit / +-1 weights, max degree,
//     max_i sum_j |w_ij| for the 32-bit decision bound), one thread per row;
//   * the throughput layout (K2/K4): degree-binned visit order (stable radix
//     sort, descending degree, ties by index), SELL-32 rows over it, and the
//     canonical u < v edge list for the barrier cut;
//   * the k1_window layout: per row the 32-bit window masks of the L vertices
//     visited just before it, the forward masks, SELL-32 rows over the natural
//     order.
// The layouts are built lazily, the first time a session needs one. A host
// version of all this took ~0.4 s for the 1M-vertex graph, more than the
// whole 20-sweep anneal; here it is a few milliseconds.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "devbuf.hpp"
#include "layout.hpp"

namespace gdi {

namespace {

constexpr int kB = 256;

inline unsigned blocks(long long n) { return static_cast<unsigned>((n + kB - 1) / kB < 1 ? 1 : (n + kB - 1) / kB); }

__global__ void k_validate(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                           const int32_t* __restrict__ w, int n, int32_t* off32, GraphScan* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned bad = 0;
  bool unit = true, pm1 = true;
  long long row = 0;
  int deg = 0;
  if (i < n) {
    const int64_t o0 = off[i], o1 = off[i + 1];
    off32[i] = static_cast<int32_t>(o0);
    if (i == n - 1) off32[n] = static_cast<int32_t>(o1);
    if (o1 < o0) bad |= 1u;
    for (int64_t e = o0; e < o1; e++) {
      const int32_t v = col[e];
      if (v < 0 || v >= n) bad |= 2u;
      if (v == i) bad |= 4u;
      const long long wv = w ? w[e] : 1;
      unit &= wv == 1;
      pm1 &= wv == 1 || wv == -1;
      row += wv < 0 ? -wv : wv;
    }
    deg = static_cast<int>(o1 > o0 ? o1 - o0 : 0);
  }
  // one atomic per warp and statistic (1M threads hitting the same words
  // serialised: 0.7 ms for the 1M-vertex graph)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    row = max(row, __shfl_xor_sync(0xffffffffu, row, o));
    deg = max(deg, __shfl_xor_sync(0xffffffffu, deg, o));
  }
  unit = __all_sync(0xffffffffu, unit);
  pm1 = __all_sync(0xffffffffu, pm1);
  if ((threadIdx.x & 31) != 0) return;
  if (bad) atomicOr(&out->bad, bad);
  if (!unit) atomicOr(&out->non_unit, 1u);
  if (!pm1) atomicOr(&out->non_pm1, 1u);
  atomicMax(&out->max_abs_field, static_cast<unsigned long long>(row));
  atomicMax(&out->max_degree, deg);
}

// ---- throughput layout -------------------------------------------------------

__global__ void k_degree(const int32_t* off, int n, int32_t* deg, int32_t* idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    deg[i] = off[i + 1] - off[i];
    idx[i] = i;
  }
}

// SELL-32 slots of chunk c: the chunk's longest row (its first, the order is
// degree-descending) rounded up to int4 groups, times 32 lanes
__global__ void k_chunk_slots(const int32_t* deg_sorted, int n, int chunks, long long* cnt) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < chunks) cnt[c] = static_cast<long long>((deg_sorted[32 * c] + 3) / 4) * 32;
  if (c == chunks) cnt[c] = 0;
}

__global__ void k_to_i32(const long long* a, int count, int32_t* b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) b[i] = static_cast<int32_t>(a[i]);
}

__global__ void k_fill_i32(int32_t* p, long long count, int32_t v) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    p[i] = v;
}

// thread = (chunk, lane): copies its row into the lane's column of the chunk
template <int WK>
__global__ void k_sell_fill(const int32_t* off, const int32_t* col, const int32_t* w, const int32_t* ord,
                            const int32_t* soff, int n, int32_t* sell, int32_t* sellw) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int c = t >> 5, l = t & 31, v = ord[t];
  const int o0 = off[v], o1 = off[v + 1];
  for (int e = o0; e < o1; e++) {
    const int k = e - o0;
    const long long slot = static_cast<long long>(soff[c]) + (k >> 2) * 32 + l;
    int32_t idx = col[e];
    if (WK == 1 && w[e] < 0) idx |= static_cast<int32_t>(0x80000000u);
    sell[slot * 4 + (k & 3)] = idx;
    if (WK == 2) sellw[slot * 4 + (k & 3)] = w[e];
  }
}

__global__ void k_up_count(const int32_t* off, const int32_t* col, int n, int32_t* cnt) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u > n) return;
  if (u == n) {
    cnt[u] = 0;
    return;
  }
  int c = 0;
  for (int e = off[u]; e < off[u + 1]; e++) c += col[e] > u;
  cnt[u] = c;
}

__global__ void k_edges_fill(const int32_t* off, const int32_t* col, const int32_t* w, const int32_t* eoff, int n,
                             int2* edges, int32_t* ew) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  int p = eoff[u];
  for (int e = off[u]; e < off[u + 1]; e++)
    if (col[e] > u) {
      edges[p] = make_int2(u, col[e]);
      if (ew) ew[p] = w[e];
      p++;
    }
}

// ---- k1_block row records ---------------------------------------------------

// vertex v: {in-window +1 mask, in-window -1 mask, columns 0-1, columns 2-3}
// (16-bit columns, bit 15 = weight -1, 0xffff = empty; degree <= 4). Mask
// bit k-1: vertex v-k of v's own aligned 32-window is a neighbour.
__global__ void k_block_rows(const int32_t* off, const int32_t* col, const int32_t* w, int n, uint4* rows) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  unsigned mp = 0u, mn = 0u, c[4] = {0xffffu, 0xffffu, 0xffffu, 0xffffu};
  const int lo = v & ~31;
  for (int e = off[v], k = 0; e < off[v + 1] && k < 4; e++, k++) {
    const int u = col[e];
    const bool neg = w && w[e] < 0;
    c[k] = static_cast<unsigned>(u) | (neg ? 0x8000u : 0u);
    if (u < v && u >= lo) (neg ? mn : mp) |= 1u << (v - u - 1);
  }
  rows[v] = make_uint4(mp, mn, c[0] | (c[1] << 16), c[2] | (c[3] << 16));
}

// ---- K2 position-space CSR -----------------------------------------------------

__global__ void k_pos_deg(const int32_t* order, const int32_t* off, int n, int32_t* pos, int32_t* pdeg) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) {
    const int v = order[p];
    pos[v] = p;
    pdeg[p] = off[v + 1] - off[v];
  }
  if (p == n) pdeg[n] = 0;
}

__global__ void k_pos_fill(const int32_t* order, const int32_t* off, const int32_t* col, const int32_t* w,
                           const int32_t* pos, const int32_t* poff, int n, int32_t* pcol) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int v = order[p];
  int o = poff[p];
  for (int e = off[v]; e < off[v + 1]; e++)
    pcol[o++] = pos[col[e]] | (w && w[e] < 0 ? static_cast<int32_t>(0x80000000u) : 0);
}

// ---- K3 evaluation layout ----------------------------------------------------

// upper-triangle entries of row u by weight class: cnt[0][u] (+1 or any
// weight), cnt[1][u] (-1, wkind 1); row n is the scan's terminator
__global__ void k_eval_count(const int32_t* off, const int32_t* col, const int32_t* w, int n, bool split,
                             int32_t* cpos, int32_t* cneg) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u > n) return;
  int p = 0, q = 0;
  if (u < n)
    for (int e = off[u]; e < off[u + 1]; e++)
      if (col[e] > u) (split && w[e] < 0 ? q : p)++;
  cpos[u] = p;
  cneg[u] = q;
}

template <bool NARROW>
__global__ void k_eval_fill(const int32_t* off, const int32_t* col, const int32_t* w, int n, bool split,
                            bool weights, const int32_t* opos, const int32_t* oneg, long long mpos, void* edges,
                            int32_t* ew) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  long long p = opos[u], q = mpos + oneg[u];
  for (int e = off[u]; e < off[u + 1]; e++) {
    const int v = col[e];
    if (v <= u) continue;
    const long long at = split && w[e] < 0 ? q++ : p++;
    if (NARROW)
      static_cast<uint32_t*>(edges)[at] = static_cast<uint32_t>(u) | (static_cast<uint32_t>(v) << 16);
    else
      static_cast<int2*>(edges)[at] = make_int2(u, v);
    if (weights) ew[at] = w[e];
  }
}

// ---- k1_window layout (k1_window.cu) ----------------------------------------

// window distance of neighbour j from row i: k = (i - j) mod n in 1..n-1
__device__ __forceinline__ int wdist(int i, int j, int n) {
  const int k = i - j;
  return k < 0 ? k + n : k;
}

// window masks of row i: bit k-1 of wpos / wneg = the vertex visited k places
// before i (cyclically) is a +1 / -1 neighbour, k = 1..L
__global__ void k_win_masks(const int32_t* off, const int32_t* col, const int32_t* w, int n, int L, uint32_t* wpos,
                            uint32_t* wneg) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t mp = 0u, mn = 0u;
  for (int e = off[i]; e < off[i + 1]; e++) {
    const int k = wdist(i, col[e], n);
    if (k >= 1 && k <= L) (w && w[e] < 0 ? mn : mp) |= 1u << (k - 1);
  }
  wpos[i] = mp;
  wneg[i] = mn;
}

template <typename T>
cudaError_t exclusive_scan(const T* in, T* out, int count, cudaStream_t st) {
  size_t bytes = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, count, st);
  if (e) return e;
  DevBuf tmp;
  if ((e = tmp.alloc(bytes))) return e;
  if ((e = cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, count, st))) return e;
  return cudaStreamSynchronize(st);  // tmp is released on return
}

// k1_window rows (natural order): chunk c's slot count = its longest row
__global__ void k_wchunk_rows(const int32_t* off, int n, int chunks, int32_t* cnt) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > chunks) return;
  if (c == chunks) {
    cnt[c] = 0;
    return;
  }
  int mx = 0;
  for (int v = 32 * c; v < 32 * c + 32 && v < n; v++) mx = max(mx, off[v + 1] - off[v]);
  cnt[c] = mx;
}

__global__ void k_wsell_fill(const int32_t* off, const int32_t* col, const int32_t* w, const int32_t* woff, int n,
                             int32_t* wsell) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int c = v >> 5, l = v & 31;
  const int base = woff[c];
  for (int e = off[v]; e < off[v + 1]; e++) {
    int32_t idx = col[e];
    if (w && w[e] < 0) idx |= static_cast<int32_t>(0x80000000u);
    wsell[static_cast<long long>(base + (e - off[v])) * 32 + l] = idx;
  }
}

__global__ void k_split_pairs(const int2* pairs, long long nnz, int32_t* col, int32_t* w) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int2 p = pairs[e];
    col[e] = p.x;
    w[e] = p.y;
  }
}

}  // namespace

cudaError_t upload_and_scan(const int64_t* offsets, const int32_t* nbr, const int32_t* weights, const int32_t* pairs,
                            int n, int64_t nnz, DevBuf& off32, DevBuf& col, DevBuf& w, GraphScan* scan,
                            cudaStream_t st) {
  cudaError_t e;
  DevBuf off64, d_scan;
  if ((e = off64.alloc((n + 1) * sizeof(int64_t)))) return e;
  if ((e = off32.alloc((n + 1) * sizeof(int32_t)))) return e;
  if ((e = col.alloc((nnz > 0 ? nnz : 1) * sizeof(int32_t)))) return e;
  if ((e = d_scan.alloc(sizeof(GraphScan)))) return e;
  if ((e = cudaMemcpyAsync(off64.p, offsets, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st))) return e;
  if (pairs) {  // one upload of the interleaved entries, split on the device
    DevBuf dp;
    if ((e = dp.alloc((nnz > 0 ? nnz : 1) * 2 * sizeof(int32_t)))) return e;
    if ((e = w.alloc((nnz > 0 ? nnz : 1) * sizeof(int32_t)))) return e;
    if (nnz && (e = cudaMemcpyAsync(dp.p, pairs, nnz * 2 * sizeof(int32_t), cudaMemcpyHostToDevice, st))) return e;
    if (nnz) {
      k_split_pairs<<<blocks(nnz), kB, 0, st>>>(dp.as<int2>(), nnz, col.as<int32_t>(), w.as<int32_t>());
      if ((e = cudaGetLastError())) return e;
    }
    weights = w.as<int32_t>();  // (device pointer) marks "weights present" below
    if ((e = cudaStreamSynchronize(st))) return e;  // dp is released on return
  } else {
    if (nnz && (e = cudaMemcpyAsync(col.p, nbr, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, st))) return e;
    if (weights) {
      if ((e = w.alloc(nnz * sizeof(int32_t)))) return e;
      if (nnz && (e = cudaMemcpyAsync(w.p, weights, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, st))) return e;
    }
  }
  if ((e = cudaMemsetAsync(d_scan.p, 0, sizeof(GraphScan), st))) return e;
  k_validate<<<blocks(n), kB, 0, st>>>(off64.as<int64_t>(), col.as<int32_t>(), w.as<int32_t>(), n,
                                        off32.as<int32_t>(), d_scan.as<GraphScan>());
  if ((e = cudaGetLastError())) return e;
  if ((e = cudaMemcpyAsync(scan, d_scan.p, sizeof(GraphScan), cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaStreamSynchronize(st))) return e;
  if (!weights || !scan->non_unit) w.reset();  // unit weights: no weight array downstream
  return cudaSuccess;
}

cudaError_t build_thru_layout(const DevCsr& g, int64_t m, int wkind, ThruLayout* L, cudaStream_t st) {
  const int n = g.n, chunks = (n + 31) / 32;
  cudaError_t e;
  // degree-binned order: stable radix sort on degree, descending
  DevBuf deg, deg_s, idx;
  if ((e = deg.alloc(n * sizeof(int32_t))) || (e = deg_s.alloc(n * sizeof(int32_t))) ||
      (e = idx.alloc(n * sizeof(int32_t))) || (e = L->order.alloc(n * sizeof(int32_t))))
    return e;
  k_degree<<<blocks(n), kB, 0, st>>>(g.off, n, deg.as<int32_t>(), idx.as<int32_t>());
  {
    size_t bytes = 0;
    if ((e = cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, deg.as<int32_t>(), deg_s.as<int32_t>(),
                                                       idx.as<int32_t>(), L->order.as<int32_t>(), n, 0, 32, st)))
      return e;
    DevBuf tmp;
    if ((e = tmp.alloc(bytes))) return e;
    if ((e = cub::DeviceRadixSort::SortPairsDescending(tmp.p, bytes, deg.as<int32_t>(), deg_s.as<int32_t>(),
                                                       idx.as<int32_t>(), L->order.as<int32_t>(), n, 0, 32, st)))
      return e;
    if ((e = cudaStreamSynchronize(st))) return e;
  }
  // chunk offsets (int4 units) by an exclusive scan of the chunk sizes
  DevBuf cnt, soff64;
  if ((e = cnt.alloc((chunks + 1) * sizeof(long long))) || (e = soff64.alloc((chunks + 1) * sizeof(long long))))
    return e;
  k_chunk_slots<<<blocks(chunks + 1), kB, 0, st>>>(deg_s.as<int32_t>(), n, chunks, cnt.as<long long>());
  if ((e = exclusive_scan(cnt.as<long long>(), soff64.as<long long>(), chunks + 1, st))) return e;
  long long total = 0;
  if ((e = cudaMemcpy(&total, soff64.as<long long>() + chunks, sizeof total, cudaMemcpyDeviceToHost))) return e;
  if (total > 0x7fffffffLL) return cudaErrorInvalidValue;  // reported as capacity by the caller
  L->slots = total;
  if ((e = L->sell_off.alloc((chunks + 1) * sizeof(int32_t)))) return e;
  k_to_i32<<<blocks(chunks + 1), kB, 0, st>>>(soff64.as<long long>(), chunks + 1, L->sell_off.as<int32_t>());
  const long long cells = (total > 0 ? total : 1) * 4;
  if ((e = L->sell.alloc(cells * sizeof(int32_t)))) return e;
  k_fill_i32<<<1024, kB, 0, st>>>(L->sell.as<int32_t>(), cells, n);  // padding index n reads spin 0
  if (wkind == 2) {
    if ((e = L->sell_w.alloc(cells * sizeof(int32_t)))) return e;
    k_fill_i32<<<1024, kB, 0, st>>>(L->sell_w.as<int32_t>(), cells, 0);
  } else {
    L->sell_w.reset();
  }
  if (wkind == 0)
    k_sell_fill<0><<<blocks(n), kB, 0, st>>>(g.off, g.col, g.w, L->order.as<int32_t>(), L->sell_off.as<int32_t>(), n,
                                             L->sell.as<int32_t>(), nullptr);
  else if (wkind == 1)
    k_sell_fill<1><<<blocks(n), kB, 0, st>>>(g.off, g.col, g.w, L->order.as<int32_t>(), L->sell_off.as<int32_t>(), n,
                                             L->sell.as<int32_t>(), nullptr);
  else
    k_sell_fill<2><<<blocks(n), kB, 0, st>>>(g.off, g.col, g.w, L->order.as<int32_t>(), L->sell_off.as<int32_t>(), n,
                                             L->sell.as<int32_t>(), L->sell_w.as<int32_t>());
  // the CSR in position space (K2's shared-memory copy)
  {
    DevBuf pdeg;
    if ((e = L->ppos.alloc((n > 0 ? n : 1) * sizeof(int32_t))) || (e = pdeg.alloc((n + 1) * sizeof(int32_t))) ||
        (e = L->poff.alloc((n + 1) * sizeof(int32_t))) || (e = L->pcol.alloc((2 * m > 0 ? 2 * m : 1) * sizeof(int32_t))))
      return e;
    k_pos_deg<<<blocks(n + 1), kB, 0, st>>>(L->order.as<int32_t>(), g.off, n, L->ppos.as<int32_t>(),
                                            pdeg.as<int32_t>());
    if ((e = exclusive_scan(pdeg.as<int32_t>(), L->poff.as<int32_t>(), n + 1, st))) return e;
    k_pos_fill<<<blocks(n), kB, 0, st>>>(L->order.as<int32_t>(), g.off, g.col, wkind == 1 ? g.w : nullptr,
                                         L->ppos.as<int32_t>(), L->poff.as<int32_t>(), n, L->pcol.as<int32_t>());
    if ((e = cudaGetLastError())) return e;
  }
  // canonical edge list (u < v, row order): count, scan, fill
  DevBuf ucnt, eoff;
  if ((e = ucnt.alloc((n + 1) * sizeof(int32_t))) || (e = eoff.alloc((n + 1) * sizeof(int32_t)))) return e;
  k_up_count<<<blocks(n + 1), kB, 0, st>>>(g.off, g.col, n, ucnt.as<int32_t>());
  if ((e = exclusive_scan(ucnt.as<int32_t>(), eoff.as<int32_t>(), n + 1, st))) return e;
  if ((e = L->edges.alloc((m > 0 ? m : 1) * sizeof(int2)))) return e;
  if (m == 0) k_fill_i32<<<1, 32, 0, st>>>(L->edges.as<int32_t>(), 2, 0);
  if (wkind != 0) {
    if ((e = L->edge_w.alloc((m > 0 ? m : 1) * sizeof(int32_t)))) return e;
  } else {
    L->edge_w.reset();
  }
  k_edges_fill<<<blocks(n), kB, 0, st>>>(g.off, g.col, wkind != 0 ? g.w : nullptr, eoff.as<int32_t>(), n,
                                         L->edges.as<int2>(), wkind != 0 ? L->edge_w.as<int32_t>() : nullptr);
  if ((e = cudaGetLastError())) return e;
  return cudaStreamSynchronize(st);
}

// K4 layout: the SELL rows with every neighbour replaced by its position in
// the visit order (pos[order[p]] = p), so that chunk c's spins are bits
// 32c..32c+31 of one word and a neighbour's spin is bit (q & 31) of word
// q >> 5. Padding entries point at position 32 * chunks (a word that stays
// zero); bit 31 keeps the -1 weight of +-1 graphs.
__global__ void k_inverse(const int32_t* order, const int32_t* off, int n, int32_t* pos, int32_t* pdeg) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) {
    const int v = order[p];
    pos[v] = p;
    pdeg[p] = off[v + 1] - off[v];
  }
}

__global__ void k_psell(const int32_t* sell, long long cells, const int32_t* pos, int n, int zpos, int32_t* psell) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < cells;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int32_t x = sell[i];
    const int v = x & 0x7fffffff;
    psell[i] = v >= n ? zpos : (pos[v] | (x & static_cast<int32_t>(0x80000000u)));
  }
}

// Forward window masks: bit l of fwd[v] = bit l of win[v + 1 + l] (vertex
// v + 1 + l has v as a +1 / -1 neighbour at distance l + 1), so one uniform load
// of the changed vertex's word gives the whole next window's corrections.
__global__ void k_fwd_masks(const uint32_t* __restrict__ wpos, const uint32_t* __restrict__ wneg, int n,
                            uint32_t* __restrict__ fpos, uint32_t* __restrict__ fneg) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  uint32_t p = 0u, q = 0u;
  for (int l = 0; l < 32 && v + 1 + l < n; l++) {
    p |= ((wpos[v + 1 + l] >> l) & 1u) << l;
    q |= ((wneg[v + 1 + l] >> l) & 1u) << l;
  }
  fpos[v] = p;
  fneg[v] = q;
}

cudaError_t build_pipe_layout(const DevCsr& g, int win, PipeLayout* L, cudaStream_t st) {
  const int n = g.n;
  cudaError_t e;
  if ((e = L->win_pos.alloc(n * sizeof(uint32_t))) || (e = L->win_neg.alloc(n * sizeof(uint32_t)))) return e;
  k_win_masks<<<blocks(n), kB, 0, st>>>(g.off, g.col, g.w, n, win, L->win_pos.as<uint32_t>(),
                                        L->win_neg.as<uint32_t>());
  if ((e = cudaGetLastError())) return e;
  if ((e = L->fwd_pos.alloc(n * sizeof(uint32_t))) || (e = L->fwd_neg.alloc(n * sizeof(uint32_t)))) return e;
  k_fwd_masks<<<blocks(n), kB, 0, st>>>(L->win_pos.as<uint32_t>(), L->win_neg.as<uint32_t>(), n,
                                        L->fwd_pos.as<uint32_t>(), L->fwd_neg.as<uint32_t>());
  if ((e = cudaGetLastError())) return e;
  // k1_window rows
  const int chunks = (n + 31) / 32;
  DevBuf wcnt;
  if ((e = wcnt.alloc((chunks + 1) * sizeof(int32_t))) || (e = L->wsell_off.alloc((chunks + 1) * sizeof(int32_t))))
    return e;
  k_wchunk_rows<<<blocks(chunks + 1), kB, 0, st>>>(g.off, n, chunks, wcnt.as<int32_t>());
  if ((e = exclusive_scan(wcnt.as<int32_t>(), L->wsell_off.as<int32_t>(), chunks + 1, st))) return e;
  int rows = 0;
  if ((e = cudaMemcpy(&rows, L->wsell_off.as<int32_t>() + chunks, sizeof rows, cudaMemcpyDeviceToHost))) return e;
  const long long cells = static_cast<long long>(rows > 0 ? rows : 1) * 32;
  if ((e = L->wsell.alloc(cells * sizeof(int32_t)))) return e;
  k_fill_i32<<<1024, kB, 0, st>>>(L->wsell.as<int32_t>(), cells, n);
  k_wsell_fill<<<blocks(n), kB, 0, st>>>(g.off, g.col, g.w, L->wsell_off.as<int32_t>(), n, L->wsell.as<int32_t>());
  if ((e = cudaGetLastError())) return e;
  return cudaStreamSynchronize(st);
}

// position-space canonical edges (K4 finishing kernel's cut): edge i of the
// u < v list as (min position | -1 weight in bit 31, max position), keyed
// for a sort by the larger position
__global__ void k_pedge_keys(const int2* edges, long long m, const int32_t* pos, int32_t* key, int32_t* idx) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int2 e = edges[i];
    key[i] = max(pos[e.x], pos[e.y]);
    idx[i] = static_cast<int32_t>(i);
  }
}
__global__ void k_pedge_fill(const int2* edges, const int32_t* ew, long long m, const int32_t* pos,
                             const int32_t* idx, int wkind, int2* pedges, int32_t* pw) {
  for (long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; j < m;
       j += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = idx[j];
    const int2 e = edges[i];
    const int a = pos[e.x], b = pos[e.y];
    const int w = ew ? ew[i] : 1;
    pedges[j] = make_int2(min(a, b) | (wkind == 1 && w < 0 ? static_cast<int>(0x80000000u) : 0), max(a, b));
    if (pw) pw[j] = w;
  }
}

cudaError_t build_part_layout(const DevCsr& g, const ThruLayout& T, long long m, int wkind, DevBuf& psell,
                              DevBuf& pdeg, DevBuf& pedges, DevBuf& pedge_w, cudaStream_t st) {
  cudaError_t e;
  const int n = g.n;
  DevBuf pos;
  if ((e = pos.alloc((n > 0 ? n : 1) * sizeof(int32_t)))) return e;
  if ((e = pdeg.alloc((n > 0 ? n : 1) * sizeof(int32_t)))) return e;
  const long long cells = (T.slots > 0 ? T.slots : 1) * 4;
  if ((e = psell.alloc(cells * sizeof(int32_t)))) return e;
  k_inverse<<<blocks(n), kB, 0, st>>>(T.order.as<int32_t>(), g.off, n, pos.as<int32_t>(), pdeg.as<int32_t>());
  k_psell<<<1184, kB, 0, st>>>(T.sell.as<int32_t>(), cells, pos.as<int32_t>(), n, 32 * ((n + 31) / 32),
                               psell.as<int32_t>());
  // edges sorted by their larger position: those between main vertices form
  // a prefix for any tail length
  const long long mm = m > 0 ? m : 1;
  DevBuf key, key_s, idx, idx_s;
  if ((e = key.alloc(mm * 4)) || (e = key_s.alloc(mm * 4)) || (e = idx.alloc(mm * 4)) || (e = idx_s.alloc(mm * 4)) ||
      (e = pedges.alloc(mm * sizeof(int2))))
    return e;
  if (wkind == 2) {
    if ((e = pedge_w.alloc(mm * 4))) return e;
  } else {
    pedge_w.reset();
  }
  if (m > 0) {
    k_pedge_keys<<<1184, kB, 0, st>>>(T.edges.as<int2>(), m, pos.as<int32_t>(), key.as<int32_t>(), idx.as<int32_t>());
    size_t bytes = 0;
    int bits = 1;
    while (bits < 31 && (1LL << bits) <= n) bits++;
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.as<int32_t>(), key_s.as<int32_t>(), idx.as<int32_t>(),
                                             idx_s.as<int32_t>(), static_cast<int>(m), 0, bits, st)))
      return e;
    DevBuf tmp;
    if ((e = tmp.alloc(bytes))) return e;
    if ((e = cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.as<int32_t>(), key_s.as<int32_t>(), idx.as<int32_t>(),
                                             idx_s.as<int32_t>(), static_cast<int>(m), 0, bits, st)))
      return e;
    k_pedge_fill<<<1184, kB, 0, st>>>(T.edges.as<int2>(), wkind != 0 ? T.edge_w.as<int32_t>() : nullptr, m,
                                      pos.as<int32_t>(), idx_s.as<int32_t>(), wkind, pedges.as<int2>(),
                                      wkind == 2 ? pedge_w.as<int32_t>() : nullptr);
    if ((e = cudaGetLastError())) return e;
    if ((e = cudaStreamSynchronize(st))) return e;  // (tmp is released on return)
  }
  if ((e = cudaGetLastError())) return e;
  return cudaStreamSynchronize(st);
}

// edges of a position-sorted list with larger position < lim (one thread: a
// binary search)
__global__ void k_count_below(const int2* pedges, long long m, int lim, long long* out) {
  long long lo = 0, hi = m;
  while (lo < hi) {
    const long long mid = (lo + hi) / 2;
    if (pedges[mid].y < lim)
      lo = mid + 1;
    else
      hi = mid;
  }
  *out = lo;
}

cudaError_t part_edges_below(const DevBuf& pedges, long long m, int lim, long long* count) {
  DevBuf d;
  cudaError_t e;
  if ((e = d.alloc(sizeof(long long)))) return e;
  k_count_below<<<1, 1>>>(pedges.as<int2>(), m, lim, d.as<long long>());
  if ((e = cudaGetLastError())) return e;
  return cudaMemcpy(count, d.p, sizeof(long long), cudaMemcpyDeviceToHost);
}

cudaError_t build_eval_layout(const DevCsr& g, int64_t m, int wkind, EvalLayout* L, cudaStream_t st) {
  const int n = g.n;
  const bool split = wkind == 1, weights = wkind == 2;
  L->m = m;
  L->narrow = n <= 65536;
  DevBuf cpos, cneg, opos, oneg;
  cudaError_t e;
  if ((e = cpos.alloc((n + 1) * sizeof(int32_t))) || (e = cneg.alloc((n + 1) * sizeof(int32_t))) ||
      (e = opos.alloc((n + 1) * sizeof(int32_t))) || (e = oneg.alloc((n + 1) * sizeof(int32_t))))
    return e;
  k_eval_count<<<blocks(n + 1), kB, 0, st>>>(g.off, g.col, g.w, n, split, cpos.as<int32_t>(), cneg.as<int32_t>());
  if ((e = exclusive_scan(cpos.as<int32_t>(), opos.as<int32_t>(), n + 1, st))) return e;
  if ((e = exclusive_scan(cneg.as<int32_t>(), oneg.as<int32_t>(), n + 1, st))) return e;
  int32_t mp = 0;
  if ((e = cudaMemcpy(&mp, opos.as<int32_t>() + n, sizeof mp, cudaMemcpyDeviceToHost))) return e;
  L->mpos = mp;
  const size_t cells = m > 0 ? static_cast<size_t>(m) : 1;
  if ((e = L->edges.alloc(cells * (L->narrow ? sizeof(uint32_t) : sizeof(int2))))) return e;
  if (weights) {
    if ((e = L->w.alloc(cells * sizeof(int32_t)))) return e;
  } else {
    L->w.reset();
  }
  if (L->narrow)
    k_eval_fill<true><<<blocks(n), kB, 0, st>>>(g.off, g.col, g.w, n, split, weights, opos.as<int32_t>(),
                                                oneg.as<int32_t>(), L->mpos, L->edges.p, L->w.as<int32_t>());
  else
    k_eval_fill<false><<<blocks(n), kB, 0, st>>>(g.off, g.col, g.w, n, split, weights, opos.as<int32_t>(),
                                                 oneg.as<int32_t>(), L->mpos, L->edges.p, L->w.as<int32_t>());
  if ((e = cudaGetLastError())) return e;
  return cudaStreamSynchronize(st);
}

cudaError_t build_block_rows(const DevCsr& g, DevBuf& rows, cudaStream_t st) {
  cudaError_t e;
  if ((e = rows.alloc((g.n > 0 ? g.n : 1) * sizeof(uint4)))) return e;
  k_block_rows<<<blocks(g.n), kB, 0, st>>>(g.off, g.col, g.w, g.n, rows.as<uint4>());
  if ((e = cudaGetLastError())) return e;
  return cudaStreamSynchronize(st);
}

}  // namespace gdi
