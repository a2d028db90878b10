// K2 — throughput GDI sweep for the reference's pooled (racy) mode (sm_100a).
//
// Contract: reference proj/src/anneal.cpp:203-225 with workers > 1 and
// SPEC.md "annealer / Concurrency Model": within a sweep every vertex is
// visited exactly once, concurrently and in any interleaving, reading the
// current (possibly not yet updated) neighbour spins; every spin change is
// folded into the shared balance counter G which each visit reads live
// (visit_node, anneal.cpp:86-128); a barrier ends the sweep, records the
// exact trace (cut, balance, counter; anneal.cpp:165-187) and decays pf.
// Results are not bit-reproducible (neither are the reference's); quality is
// checked statistically against the exact mode (tests/test_gpu_throughput.py).
//
// Why one warp per replica. A first version let 128 threads of a CTA visit
// concurrently against one shared counter: every thread saw nearly the same
// stale G, all over-corrected together and the balance oscillated (the
// paper's "biphasic oscillation"; imbalance ~240 on G22).
// Here a warp owns a replica and visits its vertices in chunks of 32 (one
// per lane): the 32 decisions are made as if the lanes ran in order, i.e.
// lane l sees G plus the spin changes of lanes < l. That sequential
// counter is obtained by a fixed-point iteration on an exclusive warp prefix
// sum of the deltas (lane 0 is right after one round, lanes <= k after k+1;
// spin changes are rare, so it converges in 1-3 rounds). Only the
// neighbour-spin reads inside a chunk stay racy, as the contract allows.
//
// Layout: spins int8 in shared memory (n bytes per replica, 4 replicas per
// CTA). Vertices are visited in a degree-binned order (sorted by degree,
// built once per graph) and their rows are stored SELL-32 over that order:
// chunk c holds the rows of order[32c..32c+31] interleaved so that the k-th
// int4 (4 neighbour indices) of all 32 lanes is one contiguous 512-byte,
// fully coalesced load, and degree binning keeps the zero-padding small.
// +-1 weights ride in the sign bit of the index. The layout is shared by all
// replicas through L1/L2. Draws: Philox4x32-10 keyed by the replica seed with
// counter (sweep, vertex): out[0..1] = 64-bit unit draw, bit 31 of out[2] =
// tie coin. Barrier: exact cut over the canonical edge list (coalesced) +
// spin sum for the trace and the counter-integrity value.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "device_rng.cuh"
#include "kernels.cuh"
#include "launch.hpp"
#include "sweep_common.cuh"

namespace gdi {

namespace {

constexpr int kWarps = 4;  // replicas per CTA (one warp each)

// WK: 0 unit weights, 1 +-1 weights (sign bit of the SELL index), 2 general.
template <int WK>
__device__ __forceinline__ int contrib(const int8_t* s, int idx, int w) {
  if (WK == 1) return idx < 0 ? -s[idx & 0x7fffffff] : s[idx];
  if (WK == 2) return w * s[idx];
  return s[idx];
}

// One chunk's spin-independent inputs plus its racy field: gathered one
// chunk ahead of its decision (see k2_sweep).
struct ChunkIn {
  int v, own, f;
  bool live, coin, flip;
};

template <int WK, int KMAX>
__device__ __forceinline__ ChunkIn gather_chunk(const ThruArgs& a, const int8_t* s, int base, int sweep, uint32_t k0,
                                                uint32_t k1, unsigned long long tm, bool en, int lane) {
  ChunkIn c{0, 0, 0, false, false, false};
  const int idx = base + lane;
  c.live = idx < a.g.n;
  if (!c.live) return c;
  c.v = __ldg(a.order + idx);
  const int c0 = __ldg(a.sell_off + (base >> 5)), c1 = __ldg(a.sell_off + (base >> 5) + 1);
  const int groups = (c1 - c0) >> 5;
  // issue every row load first (one coalesced 512 B warp load per group)
  int4 g4[KMAX], w4[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; k++) {
    if (k < groups) {
      g4[k] = __ldg(a.sell + c0 + k * 32 + lane);
      if (WK == 2) w4[k] = __ldg(a.sell_w + c0 + k * 32 + lane);
    }
  }
  const Philox4 x = philox4x32_10(static_cast<uint32_t>(sweep), static_cast<uint32_t>(c.v), 0u, 0u, k0, k1);
  c.coin = (x.z >> 31) != 0;
  c.flip = en && ((static_cast<uint64_t>(x.x) << 32) | x.y) <= tm;
  c.own = s[c.v];
  int f = 0;
#pragma unroll
  for (int k = 0; k < KMAX; k++) {
    if (k < groups) {
      const int4 q = g4[k];
      const int4 w = WK == 2 ? w4[k] : make_int4(1, 1, 1, 1);
      f += contrib<WK>(s, q.x, w.x) + contrib<WK>(s, q.y, w.y) + contrib<WK>(s, q.z, w.z) + contrib<WK>(s, q.w, w.w);
    }
  }
  for (int k = KMAX; k < groups; k++) {  // rows longer than the bucket
    const int4 q = __ldg(a.sell + c0 + k * 32 + lane);
    const int4 w = WK == 2 ? __ldg(a.sell_w + c0 + k * 32 + lane) : make_int4(1, 1, 1, 1);
    f += contrib<WK>(s, q.x, w.x) + contrib<WK>(s, q.y, w.y) + contrib<WK>(s, q.z, w.z) + contrib<WK>(s, q.w, w.w);
  }
  c.f = f;
  return c;
}

// STD: the reference's literal `standard` strategy (anneal.cpp:97-101): every
// visit re-reads all n spins (the "full traversal" the paper's GDI removes,
// PAPER.md Alg. 2 vs Alg. 3). Each lane sums the replica's spins itself for
// its own visit (O(n) work per visit, as on the reference's threads); the sum
// equals the live counter here, so the decisions are those of `gdi` and only
// the cost differs (acceptance criterion 6 measures exactly that ratio).
template <int WK, int KMAX, bool STD>
__global__ void __launch_bounds__(32 * kWarps) k2_sweep(const ThruArgs a) {
  extern __shared__ __align__(16) int8_t smem[];
  const int n = a.g.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x * kWarps + warp;
  if (r >= a.replicas) return;  // whole warp exits; no block-level sync below
  int8_t* s = smem + static_cast<size_t>(warp) * a.n_pad;
  const uint64_t seed = a.seeds[r];
  const size_t rs = static_cast<size_t>(r);
  const int2* __restrict__ edges = a.edges;
  const int32_t* __restrict__ ew = a.edge_w;

  // init (anneal.cpp:148-155): stream-0 coins; the serial stream is walked
  // by every lane, lane i%32 stores spin i
  int G = 0;
  {
    Xoshiro r0 = Xoshiro::stream(seed, 0);
    for (int i = 0; i < n; i++) {
      const int v = (r0.next() >> 63) ? 1 : -1;
      G += v;
      if ((i & 31) == lane) s[i] = static_cast<int8_t>(v);
    }
    for (int i = n + lane; i < a.n_pad; i += 32) s[i] = 0;  // SELL padding index n reads 0
  }
  __syncwarp();
  if (a.snaps != nullptr)
    for (int i = lane; i < n; i += 32) a.snaps[rs * (a.sweeps + 1) * n + i] = s[i];
  if (lane == 0 && a.stamps != nullptr) a.stamps[rs * (a.sweeps + 1)] = globaltimer_ns();
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  const int a4 = a.a4, bb = a.b;

  for (int sweep = 0; sweep < a.sweeps; sweep++) {
    const unsigned long long tm = a.tmask[sweep];
    const bool en = a.thr[sweep] >= 0;
    // Software pipeline over chunks: chunk c+1 is gathered (row loads, spin
    // reads, draws) before chunk c's spins are written. Those reads are racy
    // exactly as the contract allows (another worker may read a neighbour
    // before this one's write lands); the counter stays sequential.
    ChunkIn cur = gather_chunk<WK, KMAX>(a, s, 0, sweep, k0, k1, tm, en, lane);
    for (int base = 0; base < n; base += 32) {
      ChunkIn nxt{0, 0, 0, false, false, false};
      if (base + 32 < n) nxt = gather_chunk<WK, KMAX>(a, s, base + 32, sweep, k0, k1, tm, en, lane);
      // sequentially consistent counter inside the chunk (see header)
      if (STD) {  // full traversal per visit
        __syncwarp();  // the previous chunk's spin writes are visible to every lane
        int tot = 0;
#pragma unroll 4
        for (int j = 0; j < n; j++) tot += s[j];
        G = cur.live ? tot : G;
        G = __shfl_sync(0xffffffffu, G, 0);  // every lane summed the same spins
      }
      const int base_diff = -a4 * cur.own - bb * cur.f;  // diff = a4 (G + excl) + base_diff
      int fin = cur.live ? decide(a4 * G + base_diff, cur.coin, cur.flip) : 0;
      int d = cur.live ? fin - cur.own : 0;
      if (__any_sync(0xffffffffu, d != 0)) {
        const unsigned below = (1u << lane) - 1u;  // lanes < this lane
        for (int round = 0; round < 33; round++) {
          // d is -2, 0 or +2: the exclusive prefix is two masked popcounts
          const unsigned up = __ballot_sync(0xffffffffu, d > 0), dn = __ballot_sync(0xffffffffu, d < 0);
          const int excl = 2 * (__popc(up & below) - __popc(dn & below));
          const int fin2 = cur.live ? decide(a4 * (G + excl) + base_diff, cur.coin, cur.flip) : 0;
          if (__all_sync(0xffffffffu, fin2 == fin)) break;
          fin = fin2;
          d = cur.live ? fin - cur.own : 0;
        }
      }
      if (cur.live && d != 0) s[cur.v] = static_cast<int8_t>(fin);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      G += d;
      cur = nxt;
    }
    __syncwarp();
    // record_barrier: exact cut (each edge once, coalesced over the
    // canonical edge list) + spin sum
    long long cut = 0;
    int sum = 0;
    for (int u = lane; u < n; u += 32) sum += s[u];
    for (long long e = lane; e < a.m; e += 32) {
      const int2 uv = __ldg(edges + e);
      if (s[uv.x] != s[uv.y]) cut += WK == 0 ? 1 : __ldg(ew + e);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cut += __shfl_xor_sync(0xffffffffu, cut, o);
      sum += __shfl_xor_sync(0xffffffffu, sum, o);
    }
    if (lane == 0) {
      if (a.trace != nullptr) a.trace[rs * a.sweeps + sweep] = DevTrace{cut, sum, G};
      if (a.stamps != nullptr) a.stamps[rs * (a.sweeps + 1) + sweep + 1] = globaltimer_ns();
      if (sweep + 1 == a.sweeps) a.final_out[rs] = DevTrace{cut, sum, G};
    }
    if (a.snaps != nullptr)
      for (int i = lane; i < n; i += 32) a.snaps[(rs * (a.sweeps + 1) + sweep + 1) * n + i] = s[i];
  }
  for (int i = lane; i < n; i += 32) a.spins_out[rs * n + i] = s[i];
}

// K2 with incremental fields (chosen when 4 replicas' spins + int32 fields fit
// in shared memory): every vertex's field is kept exact in shared memory, so
// a visit reads own spin and field (two loads) instead of gathering its row.
// Each chunk's few spin changes are then applied in lane order: the exact cut
// moves by -(d/2) * field (the field as of that change), and the change is
// scattered into the neighbours' fields. The decisions inside a chunk read
// the fields as of the chunk start (racy within the chunk, as K2 always was;
// the counter stays sequentially consistent); the per-sweep cut needs no
// edge-list pass.
struct IncfIn {
  int v, own, f;
  bool live, coin, flip;
};

// FT: field storage, the narrowest type holding max_i sum_j |w_ij| (int8 for
// every G-set config: 2 bytes per vertex per replica with the spin).
template <int WK, typename FT>
__global__ void __launch_bounds__(32 * kWarps) k2_incf(const ThruArgs a) {
  extern __shared__ __align__(16) int8_t smem[];
  const int n = a.g.n, n_pad = a.n_pad;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x * kWarps + warp;
  if (r >= a.replicas) return;
  int8_t* s = smem + static_cast<size_t>(warp) * n_pad;
  FT* fld = reinterpret_cast<FT*>(smem + static_cast<size_t>(kWarps) * n_pad) + static_cast<size_t>(warp) * n_pad;
  const int32_t* __restrict__ off = a.g.off;
  const int32_t* __restrict__ col = a.g.col;
  const int32_t* __restrict__ wgt = a.g.w;
  const uint64_t seed = a.seeds[r];
  const size_t rs = static_cast<size_t>(r);
  const unsigned FULL = 0xffffffffu;

  int G = 0;
  {
    Xoshiro r0 = Xoshiro::stream(seed, 0);  // anneal.cpp:148-155
    for (int i = 0; i < n; i++) {
      const int v = (r0.next() >> 63) ? 1 : -1;
      G += v;
      if ((i & 31) == lane) s[i] = static_cast<int8_t>(v);
    }
  }
  __syncwarp();
  long long cut = 0;
  for (int v = lane; v < n; v += 32) {
    int f = 0;
    const int sv = s[v];
    for (int e = __ldg(off + v); e < __ldg(off + v + 1); e++) {
      const int u = __ldg(col + e);
      const int w = WK == 0 ? 1 : __ldg(wgt + e);
      f += w * s[u];
      if (u > v && s[u] != sv) cut += w;
    }
    fld[v] = static_cast<FT>(f);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cut += __shfl_xor_sync(FULL, cut, o);
  __syncwarp();
  if (a.snaps != nullptr)
    for (int i = lane; i < n; i += 32) a.snaps[rs * (a.sweeps + 1) * n + i] = s[i];
  if (lane == 0 && a.stamps != nullptr) a.stamps[rs * (a.sweeps + 1)] = globaltimer_ns();
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  const int a4 = a.a4, bb = a.b;
  const unsigned below = (1u << lane) - 1u;

  for (int sweep = 0; sweep < a.sweeps; sweep++) {
    const unsigned long long tm = a.tmask[sweep];
    const bool en = a.thr[sweep] >= 0;
    long long dcut = 0;
    // software pipeline: chunk c+1's own spins, fields and draws are read
    // before chunk c is decided and applied (a racy read one chunk ahead, as
    // the row-gathering K2 does); the cut uses the fields as of each change
    auto load = [&](int b) -> IncfIn {
      IncfIn c;
      const int idx = b + lane;
      c.live = idx < n;
      c.v = c.live ? __ldg(a.order + idx) : 0;
      c.own = c.live ? s[c.v] : 0;
      c.f = c.live ? fld[c.v] : 0;
      const Philox4 x = philox4x32_10(static_cast<uint32_t>(sweep), static_cast<uint32_t>(c.v), 0u, 0u, k0, k1);
      c.coin = (x.z >> 31) != 0;
      c.flip = en && ((static_cast<uint64_t>(x.x) << 32) | x.y) <= tm;
      return c;
    };
    IncfIn cur = load(0);
    for (int base = 0; base < n; base += 32) {
      const IncfIn nx = base + 32 < n ? load(base + 32) : IncfIn{0, 0, 0, false, false, false};
      const bool live = cur.live, coin = cur.coin, flip = cur.flip;
      const int v = cur.v, own = cur.own, f = cur.f;
      cur = nx;
      const int base_diff = -a4 * own - bb * f;
      int fin = live ? decide(a4 * G + base_diff, coin, flip) : 0;
      int d = live ? fin - own : 0;
      unsigned up = __ballot_sync(FULL, d > 0), dn = __ballot_sync(FULL, d < 0);
      if ((up | dn) != 0u) {
        for (int round = 0; round < 33; round++) {
          const int excl = 2 * (__popc(up & below) - __popc(dn & below));
          const int fin2 = live ? decide(a4 * (G + excl) + base_diff, coin, flip) : 0;
          if (__all_sync(FULL, fin2 == fin)) break;
          fin = fin2;
          d = live ? fin - own : 0;
          up = __ballot_sync(FULL, d > 0);
          dn = __ballot_sync(FULL, d < 0);
        }
        G += 2 * (__popc(up) - __popc(dn));
        // apply the changes in lane order: exact cut, spin, field scatter
        for (unsigned chg = up | dn; chg != 0u; chg &= chg - 1u) {
          const int j = __ffs(chg) - 1;
          const int vj = __shfl_sync(FULL, v, j), dj = __shfl_sync(FULL, d, j);
          dcut -= static_cast<long long>(dj >> 1) * fld[vj];
          if (lane == 0) s[vj] = static_cast<int8_t>(s[vj] + dj);
          const int e1 = __ldg(off + vj + 1);
          for (int e = __ldg(off + vj) + lane; e < e1; e += 32) {
            const int u = __ldg(col + e);  // a row has no repeated neighbour: no two lanes hit one field
            fld[u] = static_cast<FT>(fld[u] + (WK == 0 ? dj : __ldg(wgt + e) * dj));
          }
          __syncwarp();
        }
      }
    }
    cut += dcut;
    // record_barrier: spin sum (the counter-integrity check) + the exact cut
    int sum = 0;
    for (int u = lane; u < n; u += 32) sum += s[u];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
    if (lane == 0) {
      if (a.trace != nullptr) a.trace[rs * a.sweeps + sweep] = DevTrace{cut, sum, G};
      if (a.stamps != nullptr) a.stamps[rs * (a.sweeps + 1) + sweep + 1] = globaltimer_ns();
      if (sweep + 1 == a.sweeps) a.final_out[rs] = DevTrace{cut, sum, G};
    }
    if (a.snaps != nullptr)
      for (int i = lane; i < n; i += 32) a.snaps[(rs * (a.sweeps + 1) + sweep + 1) * n + i] = s[i];
  }
  for (int i = lane; i < n; i += 32) a.spins_out[rs * n + i] = s[i];
}

// K2 chains: several warps per replica (the racy pooled mode's concurrency
// inside one replica, anneal.cpp:203-225). A CTA holds RPC replicas x P
// chains (one warp each); a replica's spins (int8) and exact fields (biased,
// packed in 32-bit words so a change scatters with word atomics: no carry
// crosses into a neighbour's lane since |field| <= max degree < bias) live in
// shared memory with the visit order and (when it fits) the CSR with 16-bit
// columns. Chain j of a replica visits every P-th segment of kSeg chunks of
// the degree-binned order against its own counter, started from its share of the
// replica's exact imbalance (decoupled balance, as K4); after a per-replica
// barrier, chain 0 decides the last T chunks (lowest degrees) in order
// against the exact counter, so sweeps end balanced. A visit reads own spin
// and field (racy against the other chains' concurrent scatters, as the
// contract allows); the 32 decisions of a chunk see the counter in lane order
// (two evaluations, else the exact threshold scan). The exact cut at the
// barrier comes from the exact fields: sum_u s_u f_u = 2 sum_e w_e s_u s_v, so
// cut = (W - sum_u s_u f_u / 2) / 2 (evaluate.cpp:10-18), an O(n) reduction.
template <int FB>
__device__ __forceinline__ int fget(const unsigned char* fld, int v) {
  if (FB == 1) return static_cast<int>(fld[v]) - 128;
  if (FB == 2) return static_cast<int>(reinterpret_cast<const uint16_t*>(fld)[v]) - 32768;
  return reinterpret_cast<const int*>(fld)[v];
}
template <int FB>
__device__ __forceinline__ void fset(unsigned char* fld, int v, int f) {
  if (FB == 1)
    fld[v] = static_cast<unsigned char>(f + 128);
  else if (FB == 2)
    reinterpret_cast<uint16_t*>(fld)[v] = static_cast<uint16_t>(f + 32768);
  else
    reinterpret_cast<int*>(fld)[v] = f;
}
template <int FB>
__device__ __forceinline__ void fadd(unsigned char* fld, int v, int d) {
  unsigned* w = reinterpret_cast<unsigned*>(fld);
  if (FB == 1)
    atomicAdd(w + (v >> 2), static_cast<unsigned>(d) << ((v & 3) * 8));
  else if (FB == 2)
    atomicAdd(w + (v >> 1), static_cast<unsigned>(d) << ((v & 1) * 16));
  else
    atomicAdd(reinterpret_cast<int*>(fld) + v, d);
}
__device__ __forceinline__ void bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int WK, int FB, bool CS>
__global__ void __launch_bounds__(1024, 1) k2_chains(const ThruArgs a, const ChainCfg cf) {
  extern __shared__ __align__(16) unsigned char csm[];
  __shared__ int red_d[32], rep_G[16];
  __shared__ __align__(16) int2 scan_buf[32][32];  // in-order scan scratch per warp (warp_seq_decide)
  __shared__ __align__(16) int scan_g[32][32];
  __shared__ long long red_sf[32], red_s[32];
  __shared__ long long Wtot;
  const int n = a.g.n, P = cf.chains;
  const int nck = (n + 31) >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = warp / P, j = warp - slot * P;
  const int r = blockIdx.x * cf.rpc + slot;
  const unsigned FULL = 0xffffffffu;
  int32_t* order = reinterpret_cast<int32_t*>(csm + cf.off_order);
  int32_t* offs = reinterpret_cast<int32_t*>(csm + cf.off_offs);
  uint16_t* cols = reinterpret_cast<uint16_t*>(csm + cf.off_cols);

  // ---- prologue (whole CTA): visit order, CSR, total edge weight W
  long long wpart = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) order[i] = __ldg(a.order + i);
  if (CS) {
    // the shared-memory CSR in position space (row p = vertex order[p],
    // neighbours as positions): a chunk's lane p reads its own spin, field
    // and row directly, without the order[] indirection
    for (int i = threadIdx.x; i <= n; i += blockDim.x) offs[i] = __ldg(a.poff + i);
    const int nnz = __ldg(a.poff + n);
    for (int e = threadIdx.x; e < nnz; e += blockDim.x) {
      const int c = __ldg(a.pcol + e);
      const bool neg = WK == 1 && c < 0;
      cols[e] = static_cast<uint16_t>(neg ? ((c & 0x7fffffff) | 0x8000) : c);
      wpart += neg ? -1 : 1;
    }
  } else {
    const int nnz = __ldg(a.g.off + n);
    for (int e = threadIdx.x; e < nnz; e += blockDim.x) wpart += WK == 0 ? 1 : __ldg(a.g.w + e);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wpart += __shfl_xor_sync(FULL, wpart, o);
  if (threadIdx.x == 0) Wtot = 0;
  __syncthreads();
  if (lane == 0 && wpart != 0) atomicAdd(reinterpret_cast<unsigned long long*>(&Wtot), static_cast<unsigned long long>(wpart));
  __syncthreads();
  if (slot >= cf.rpc || r >= a.replicas) return;  // only per-replica barriers below
  const long long W2 = Wtot;  // = 2 * total weight (every edge twice in the CSR)

  auto row = [&](int v, int& e0, int& e1) {
    if (CS) {
      e0 = offs[v];
      e1 = offs[v + 1];
    } else {
      e0 = __ldg(a.g.off + v);
      e1 = __ldg(a.g.off + v + 1);
    }
  };
  // neighbour u and weight of CSR entry e
  auto entry = [&](int e, int& u, int& w) {
    if (CS) {
      const int c = cols[e];
      u = WK == 1 ? (c & 0x7fff) : c;
      w = WK == 1 && (c & 0x8000) ? -1 : 1;
    } else {
      u = __ldg(a.g.col + e);
      w = WK == 0 ? 1 : __ldg(a.g.w + e);
    }
  };

  unsigned char* rep = csm + cf.off_rep + slot * cf.rep_bytes;
  int8_t* s = reinterpret_cast<int8_t*>(rep);
  unsigned char* fld = rep + cf.n_pad4;
  const int bid = 1 + slot, bthreads = 32 * P;
  const size_t rs = static_cast<size_t>(r);
  const uint64_t seed = a.seeds[r];
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  const int a4 = a.a4, bb = a.b;

  // ---- init (anneal.cpp:148-155): the serial stream-0 coins (chain 0), fields
  if (j == 0) {
    Xoshiro r0 = Xoshiro::stream(seed, 0);
    int G = 0;
    for (int i = 0; i < n; i++) {
      const int v = (r0.next() >> 63) ? 1 : -1;
      G += v;
      if ((i & 31) == lane) s[CS ? __ldg(a.ppos + i) : i] = static_cast<int8_t>(v);  // (position space when CS)
    }
    if (lane == 0) rep_G[slot] = G;
  }
  bar_sync(bid, bthreads);
  for (int v = j * 32 + lane; v < n; v += bthreads) {
    int e0, e1, f = 0;
    row(v, e0, e1);
    for (int e = e0; e < e1; e++) {
      int u, w;
      entry(e, u, w);
      f += w * s[u];
    }
    fset<FB>(fld, v, f);
  }
  bar_sync(bid, bthreads);
  if (a.snaps != nullptr)
    for (int i = j * 32 + lane; i < n; i += bthreads) a.snaps[rs * (a.sweeps + 1) * n + (CS ? order[i] : i)] = s[i];
  if (j == 0 && lane == 0 && a.stamps != nullptr) a.stamps[rs * (a.sweeps + 1)] = globaltimer_ns();

  // one chunk: visits against counter G (lane order), spin stores and the
  // scatter of every change into its neighbours' fields
  // draws: one Philox call per four chunks (kept for the chain's next three)
  uint64_t spare = 0, spare2 = 0;
  int spare_c = -1;
  auto chunk = [&](int c, int& G, int sweep, unsigned long long tm, bool en) {
    const int p = c * 32 + lane;
    const bool live = p < n;
    const int v = live ? (CS ? p : order[p]) : 0;
    const int own = live ? s[v] : -1, f = live ? fget<FB>(fld, v) : 0;
    // one Philox4x32-10 call per four chunks (4b .. 4b + 3; counter (sweep,
    // 32b + lane, 2, 0), key = the replica seed), 32 bits per visit: coin =
    // bit 0, a 31-bit uniform against the flip threshold's top 31 bits
    // (tm >> 33: resolution 2^-31, against flip probabilities >= 1.7e-6 at
    // the end of the default schedule). Pairs of 64-bit uniforms took 6% more
    // time (G22 14.73 vs 13.80 ms), same quality.
    if ((c >> 2) != spare_c) {
      const Philox4 x = philox4x32_10(static_cast<uint32_t>(sweep), static_cast<uint32_t>(c >> 2) * 32u + lane, 2u, 0u,
                                      k0, k1);
      spare = (static_cast<uint64_t>(x.y) << 32) | x.x;
      spare2 = (static_cast<uint64_t>(x.w) << 32) | x.z;
      spare_c = c >> 2;
    }
    const uint64_t pr = (c & 2) ? spare2 : spare;
    const unsigned w32 = (c & 1) ? static_cast<unsigned>(pr >> 32) : static_cast<unsigned>(pr);
    const bool coin = (w32 & 1u) != 0, flip = en && (w32 >> 1) <= static_cast<unsigned>(tm >> 33);

    const int base = -a4 * own - bb * f;
    int fin = live ? decide(a4 * G + base, coin, flip) : own;
    unsigned up = __ballot_sync(FULL, fin > own), dn = __ballot_sync(FULL, fin < own);
    if ((up | dn) == 0u) return;
    const unsigned below = (1u << lane) - 1u;
    const int fin2 = live ? decide(a4 * (G + 2 * (__popc(up & below) - __popc(dn & below))) + base, coin, flip) : own;
    if (__all_sync(FULL, fin2 == fin)) {
      G += 2 * (__popc(up) - __popc(dn));
    } else {
      fin = warp_seq_decide(own, f, live, coin, flip, G, a4, bb, lane, scan_buf[warp], scan_g[warp]);
      up = __ballot_sync(FULL, fin > own);
      dn = __ballot_sync(FULL, fin < own);
    }
    if (fin != own) s[v] = static_cast<int8_t>(fin);
    if (cf.lane_rows && __popc(up | dn) >= 2) {
      // short rows, several changes: every changed lane walks its own row
      if (live && fin != own) {
        int e0, e1;
        row(v, e0, e1);
        const int dl = fin > own ? 2 : -2;
#pragma unroll 1
        for (int e = e0; e < e1; e++) {
          int u, w;
          entry(e, u, w);
          fadd<FB>(fld, u, w * dl);
        }
      }
      return;
    }
    for (unsigned chg = up | dn; chg != 0u; chg &= chg - 1u) {
      const int l = __ffs(chg) - 1;
      const int vl = __shfl_sync(FULL, v, l), dl = ((up >> l) & 1u) ? 2 : -2;
      int e0, e1;
      row(vl, e0, e1);
      for (int e = e0 + lane; e < e1; e += 32) {
        int u, w;
        entry(e, u, w);
        fadd<FB>(fld, u, w * dl);
      }
    }
  };

  // the chain with the fewest main chunks decides the tail (sweep-invariant)
  int jt = 0;
  {
    const int nmain0 = nck - cf.tail, nseg = (nmain0 + cf.seg - 1) / cf.seg, L = nmain0 - (nseg - 1) * cf.seg;
    int best = 1 << 30;
    for (int q = 0; q < P; q++) {
      const int cnt = (q < nseg ? (nseg - q + P - 1) / P : 0) * cf.seg - (q == (nseg - 1) % P ? cf.seg - L : 0);
      if (cnt <= best) {
        best = cnt;
        jt = q;
      }
    }
  }
  for (int sweep = 0; sweep < a.sweeps; sweep++) {
    const unsigned long long tm = a.tmask[sweep];
    const bool en = a.thr[sweep] >= 0;
    // this chain's share of the replica's imbalance (units of 2, remainder
    // rotated over the chains; see k4_partition.cu). (Every chain reading the
    // replica's live counter instead, the other chains' changes published per
    // chunk, oscillated: G22 cut 9745 vs 6726, never balanced, even with two
    // chains: each chain corrects the whole imbalance at once.)
    const int Gs = rep_G[slot];
    const int par = Gs & 1, Gh = (Gs - par) / 2;
    int q = Gh / P, rem = Gh - q * P;
    if (rem < 0) {
      rem += P;
      q -= 1;
    }
    const int rot = (j + P - sweep % P) % P;
    const int share = 2 * (q + (rot < rem ? 1 : 0)) + (rot == P - 1 ? par : 0);
    int G = share;
    spare_c = -1;  // (draws are per sweep)
    // chain j visits the segments j, j + P, ... of kSeg consecutive chunks,
    // each in order: concurrent chains are kSeg chunks apart (round-robin
    // single chunks made adjacent lattice sites concurrent: torus(100,20) best
    // cut 84 vs 44 sequential), and every chain still spans the whole degree
    // range (contiguous blocks gave chain 0 only the stiffest, highest-degree
    // vertices, whose share of the imbalance it could not correct: 57% of
    // runs balanced on a hub graph vs 86% sequential)
    // the tail: the last T chunks (a quarter of the graph in the final sweep
    // balanced no more runs of a hub graph: 81% either way, 86% sequential)
    const int T = cf.tail, nmain = nck - T;
    const int kSeg = cf.seg;
#pragma unroll 1
    for (int s0 = j * kSeg; s0 < nmain; s0 += P * kSeg) {
      const int c1 = min(nmain, s0 + kSeg);
#pragma unroll 1
      for (int c = s0; c < c1; c++) chunk(c, G, sweep, tm, en);
    }
    if (lane == 0) red_d[warp] = G - share;
    bar_sync(bid, bthreads);
    // the tail, in order against the replica's exact counter, by the chain
    // with the fewest main chunks (G22: per-chain main chunks
    // 16/16/16/12, the 3-chunk tail by chain 3 instead of 0: 19.8 -> 18.5 ms;
    // dealing the last round's segments in reverse instead, so that chain 0
    // had the short one, was as fast but ended fewer hub-graph runs balanced)
    if (j == jt) {
      int dsum = lane < P ? red_d[slot * P + lane] : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(FULL, dsum, o);
      int Gt = Gs + dsum;
#pragma unroll 1
      for (int c = nmain; c < nck; c++) chunk(c, Gt, sweep, tm, en);
      if (lane == 0) rep_G[slot] = Gt;
    }
    bar_sync(bid, bthreads);
    // record_barrier: spin sum and the exact cut from the exact fields
    long long sf = 0, ss = 0;
    int v0 = 0;
    if (FB == 1 && a.snaps == nullptr) {
      // four vertices per step: int8 spins x biased byte fields by dp4a
      // (sum s (f + 128) - 128 sum s)
      const int n4 = n >> 2;
      int sfi = 0, ssi = 0;
      for (int q = j * 32 + lane; q < n4; q += bthreads) {
        const int s4 = reinterpret_cast<const int*>(s)[q];
        const unsigned f4 = reinterpret_cast<const unsigned*>(fld)[q];
        int d, e;
        asm("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(s4), "r"(0x01010101), "r"(0));
        asm("dp4a.s32.u32 %0, %1, %2, %3;" : "=r"(e) : "r"(s4), "r"(f4), "r"(0));  // signed spins x unsigned bytes
        ssi += d;
        sfi += e - 128 * d;
      }
      sf = sfi;
      ss = ssi;
      v0 = 4 * n4;
    }
    for (int v = v0 + j * 32 + lane; v < n; v += bthreads) {
      const int sv = s[v];
      sf += sv * fget<FB>(fld, v);
      ss += sv;
      if (a.snaps != nullptr) a.snaps[(rs * (a.sweeps + 1) + sweep + 1) * n + (CS ? order[v] : v)] = static_cast<int8_t>(sv);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sf += __shfl_xor_sync(FULL, sf, o);
      ss += __shfl_xor_sync(FULL, ss, o);
    }
    if (lane == 0) {
      red_sf[warp] = sf;
      red_s[warp] = ss;
    }
    bar_sync(bid, bthreads);
    if (j == 0 && lane == 0) {
      long long SF = 0, S = 0;
      for (int k = 0; k < P; k++) {
        SF += red_sf[slot * P + k];
        S += red_s[slot * P + k];
      }
      const long long cut = (W2 / 2 - SF / 2) / 2;
      const DevTrace rec{cut, S, rep_G[slot]};
      if (a.trace != nullptr) a.trace[rs * a.sweeps + sweep] = rec;
      if (a.stamps != nullptr) a.stamps[rs * (a.sweeps + 1) + sweep + 1] = globaltimer_ns();
      if (sweep + 1 == a.sweeps) a.final_out[rs] = rec;
    }
  }
  for (int i = j * 32 + lane; i < n; i += bthreads) a.spins_out[rs * n + (CS ? order[i] : i)] = s[i];
}

template <int WK, int FB>
const void* chains_fn(bool cs) {
  return cs ? reinterpret_cast<const void*>(&k2_chains<WK, FB, true>)
            : reinterpret_cast<const void*>(&k2_chains<WK, FB, false>);
}
template <int WK>
const void* chains_fn(int fb, bool cs) {
  return fb == 1 ? chains_fn<WK, 1>(cs) : fb == 2 ? chains_fn<WK, 2>(cs) : chains_fn<WK, 4>(cs);
}

template <typename FT>
const void* incf_fn(int wkind) {
  return wkind == 0   ? reinterpret_cast<const void*>(&k2_incf<0, FT>)
         : wkind == 1 ? reinterpret_cast<const void*>(&k2_incf<1, FT>)
                      : reinterpret_cast<const void*>(&k2_incf<2, FT>);
}

template <int WK, bool STD>
const void* k2_fn(int kmax) {
  switch (kmax) {
    case 1: return reinterpret_cast<const void*>(&k2_sweep<WK, 1, STD>);
    case 2: return reinterpret_cast<const void*>(&k2_sweep<WK, 2, STD>);
    case 4: return reinterpret_cast<const void*>(&k2_sweep<WK, 4, STD>);
    case 8: return reinterpret_cast<const void*>(&k2_sweep<WK, 8, STD>);
    default:  // (weighted rows carry a weight array: 16 groups of both spilled, so 8 + the loop)
      if constexpr (WK == 2)
        return reinterpret_cast<const void*>(&k2_sweep<WK, 8, STD>);
      else
        return reinterpret_cast<const void*>(&k2_sweep<WK, 16, STD>);
  }
}

}  // namespace

namespace {

// k2_chains shared-memory layout and shape; false when it does not fit.
bool chains_layout(const GraphStats& st, int wkind, int32_t replicas, int fb, ChainCfg* c, bool* cs) {
  const int n = st.n;
  const long long nnz = 2 * st.m;
  const int nck = (n + 31) / 32;
  int rpc = (replicas + 147) / 148;
  rpc = rpc < 1 ? 1 : rpc > 15 ? 15 : rpc;  // (named barriers 1..15, one per replica)
  // chains per replica: up to 4, fewer on small graphs, where concurrent
  // chains' last-moment flips (each balanced against its own share) leave a
  // residual imbalance that the few tail vertices cannot absorb (G1, n = 800:
  // 77% of runs balanced with 4 chains, 94% in the exact mode)
  int P = 32 / rpc;
  P = P > 4 ? 4 : P < 1 ? 1 : P;
  P = std::min(P, std::max(1, n / 500));
  if (const char* e = std::getenv("GDI_K2_CHAINS")) P = std::max(1, std::min(std::atoi(e), 32 / rpc));
  // one tail chunk: the other chains wait at the named barrier while it is
  // decided (G22: 3 chunks -> 1: 15.5 -> 14.8 ms; the runs that end balanced
  // are the same: G22 99.8%, G55 100%, hub graph 0.81 vs 0.80 over 2048 runs;
  // no tail at all: hub graph 0.68)
  int T = 1;
  if (const char* e = std::getenv("GDI_K2_TAIL")) T = std::max(0, std::min(std::atoi(e), nck - 1));
  int seg = 8;
  if (const char* e = std::getenv("GDI_K2_SEG")) seg = std::max(1, std::atoi(e));
  c->seg = seg;
  int lane_maxdeg = 16;
  if (const char* e = std::getenv("GDI_K2_LANE_MAXDEG")) lane_maxdeg = std::atoi(e);  // A/B
  c->lane_rows = st.max_degree <= lane_maxdeg;
  if (nck - T < P) P = std::max(1, nck - T);
  auto r16 = [](long long x) { return (x + 15) & ~15LL; };
  const long long n_pad4 = r16(n + 4);
  const long long rep = r16(n_pad4 + static_cast<long long>(fb) * n_pad4);
  const long long order = r16(4LL * n);
  const long long offs = r16(4LL * (n + 1)), cols = r16(2 * nnz);
  const long long cap = 227 * 1024 - 2048;  // (static shared memory)
  const bool cs_ok = wkind != 2 && n <= (wkind == 1 ? 32767 : 65535);
  long long total = order + offs + cols + rpc * rep;
  *cs = cs_ok && total <= cap;
  if (!*cs) total = order + rpc * rep;
  if (total > cap) return false;
  c->rpc = rpc;
  c->chains = P;
  c->tail = T;
  c->off_order = 0;
  c->off_offs = static_cast<int32_t>(order);
  c->off_cols = static_cast<int32_t>(order + offs);
  c->off_rep = static_cast<int32_t>(*cs ? order + offs + cols : order);
  c->rep_bytes = static_cast<int32_t>(rep);
  c->n_pad4 = static_cast<int32_t>(n_pad4);
  c->smem = static_cast<int32_t>(total);
  return true;
}

}  // namespace

int thru_plan(const GraphStats& st, int wkind, int32_t replicas, int64_t a4, int64_t b, bool standard,
              ThruPlan* plan) {
  // 32-bit decision arithmetic must be exact (same bound as k1_window)
  long long x = a4 < 0 ? -a4 : a4, y = b < 0 ? -b : b;
  while (y) {
    const long long t = x % y;
    x = y;
    y = t;
  }
  const long long ra = a4 / x, rb = b / x;
  const double bound = static_cast<double>(ra) * (2.0 * st.n + 1) + static_cast<double>(rb) * (st.max_abs_field + 1);
  if (bound >= 2147483647.0) return -1;
  const int n_pad = (st.n + 1 + 15) & ~15;  // + pad entry n
  const long long smem = static_cast<long long>(n_pad) * kWarps;
  if (smem > 200 * 1024) return -1;
  // register-resident row bucket: the int4 groups of a typical row (mean
  // degree, rounded up to 1/2/4/8/16); unused slots of the bucket are still
  // issued (predicated), so it is sized by the mean, not the longest row,
  // and longer rows loop over the remainder
  const double mean_deg = st.n > 0 ? 2.0 * static_cast<double>(st.m) / st.n : 0.0;
  const int groups = static_cast<int>((mean_deg + 3.999) / 4);
  const int kmax = groups <= 1 ? 1 : groups <= 2 ? 2 : groups <= 4 ? 4 : groups <= 8 ? 8 : 16;
  // incremental fields when 4 replicas' spins (1 B) + fields (fb B) fit
  const char* force = std::getenv("GDI_FORCE_KERNEL");
  const int fb = st.max_abs_field <= 127 ? 1 : st.max_abs_field <= 32767 ? 2 : 4;
  const bool incf =
      !standard && (1LL + fb) * n_pad * kWarps <= 200 * 1024 && !(force && std::string(force) == "k2_gather");
  ChainCfg cc{};
  bool cs = false;
  plan->chains = false;
  const bool chains = !standard && !(force && (std::string(force) == "k2_gather" || std::string(force) == "k2_incf")) &&
                      chains_layout(st, wkind, replicas, fb, &cc, &cs);
  if (chains) {
    plan->fn = wkind == 0 ? chains_fn<0>(fb, cs) : wkind == 1 ? chains_fn<1>(fb, cs) : chains_fn<2>(fb, cs);
    plan->chains = true;
    plan->cfg = cc;
    plan->block = 32 * cc.rpc * cc.chains;
    plan->grid = (replicas + cc.rpc - 1) / cc.rpc;
    plan->n_pad = n_pad;
    plan->a4 = static_cast<int32_t>(ra);
    plan->b = static_cast<int32_t>(rb);
    static const char* cn[3] = {"k2_chains<unit>", "k2_chains<pm1>", "k2_chains<weighted>"};
    plan->name = cn[wkind];
    plan->smem = cc.smem;
    return 0;
  }
  if (standard)
    plan->fn = wkind == 0 ? k2_fn<0, true>(kmax) : wkind == 1 ? k2_fn<1, true>(kmax) : k2_fn<2, true>(kmax);
  else if (incf)
    plan->fn = fb == 1 ? incf_fn<int8_t>(wkind) : fb == 2 ? incf_fn<int16_t>(wkind) : incf_fn<int>(wkind);
  else
    plan->fn = wkind == 0 ? k2_fn<0, false>(kmax) : wkind == 1 ? k2_fn<1, false>(kmax) : k2_fn<2, false>(kmax);
  plan->block = 32 * kWarps;
  plan->grid = (replicas + kWarps - 1) / kWarps;
  plan->n_pad = n_pad;
  plan->a4 = static_cast<int32_t>(ra);
  plan->b = static_cast<int32_t>(rb);
  static const char* names[3][3] = {{"k2_sweep<unit>", "k2_sweep<pm1>", "k2_sweep<weighted>"},
                                     {"k2_sweep<unit,standard>", "k2_sweep<pm1,standard>", "k2_sweep<weighted,standard>"},
                                     {"k2_sweep<unit,incf>", "k2_sweep<pm1,incf>", "k2_sweep<weighted,incf>"}};
  plan->name = names[standard ? 1 : incf ? 2 : 0][wkind];
  plan->smem = static_cast<int>((incf ? 1LL + fb : 1LL) * n_pad * kWarps);
  return 0;
}

cudaError_t thru_launch(const ThruPlan& plan, const ThruArgs& args, cudaStream_t stream) {
  cudaError_t err = allow_max_smem(plan.fn);
  if (err != cudaSuccess) return err;
  ThruArgs a = args;
  a.a4 = plan.a4;
  a.b = plan.b;
  a.n_pad = plan.n_pad;
  if (plan.chains) {
    ChainCfg c = plan.cfg;
    void* pc[] = {&a, &c};
    return cudaLaunchKernel(plan.fn, dim3(plan.grid), dim3(plan.block), pc, plan.smem, stream);
  }
  void* params[] = {&a};
  return cudaLaunchKernel(plan.fn, dim3(plan.grid), dim3(plan.block), params, plan.smem, stream);
}

}  // namespace gdi
