// K4 — vertex-partitioned throughput sweep for large graphs (sm_100a).
//
// Contract: the reference's pooled racy mode (proj/src/anneal.cpp:203-225,
// SPEC.md "annealer / Concurrency Model") for graphs whose spins do not fit
// in one CTA's shared memory — BASELINE configs[4], the 1M-vertex rudy graph
// — with one or a few replicas, so the parallelism has to come from the
// vertices of one replica rather than from independent replicas (K2).
//
// Chains. The chunks (32 vertices, SELL-32 rows over the degree-binned
// order, the same layout as K2) are dealt round-robin to P chains; a chain
// is one warp (P = all resident warps / replicas). A chain visits its chunks
// in order with its counter in a register, and inside a chunk the 32
// decisions see the counter as if made in order (K2's fixed-point ballot
// prefix). Neighbour spins are read through L2 while other chains write them
// (racy reads, as the contract allows). A first version chained the 16
// warps of a CTA through a shared-memory token: the ~700-cycle handoff per
// chunk, not the memory system, bounded it (116 us per 1M-vertex sweep).
//
// Decoupled global balance. A single counter read live by ~10^4 concurrent
// visitors over-corrects (all see the same stale imbalance and all flip
// towards the minority: the "biphasic oscillation" of PAPER.md:632-633; K2's
// first version showed it). Here chain J starts each sweep from its share of
// the exact global imbalance G at the last barrier (G/P in units of 2,
// remainder spread over a rotating set of chains, so the shares sum to G) and then
// counts only its own spin changes. Every chain drives its own counter to
// zero, so together they remove exactly G per sweep instead of P times G,
// and each chain absorbs its own random flips. The last T chunks of the
// order (its lowest-degree vertices) form a tail that the last CTA to finish
// decides against the exact global counter, so a sweep ends balanced as the
// sequential algorithm does rather than with the sum of P chain residuals.
// With P = 1 this is the exact sequential counter.
//
// Barrier (record_barrier, anneal.cpp:165-187): k4_pack bit-packs the spins
// (and sums them), k4_cut streams the canonical edge list against the
// 1 bit/vertex copy (L1-resident: 125 KB for 1M vertices) and the last block
// writes the trace record, checks nothing is lost (counter = G + chain
// deltas) and rolls the counter. Kernel boundaries are the sweep barriers;
// the session replays the 1 + 3M launches as one CUDA graph.
//
// Multi-GPU (vertex partitioning): the chain numbering is
// global (chain0, world_chains), so a device runs a contiguous block of the
// chains; between sweeps the owned chunks' spins are exchanged and the
// deltas summed (host side), and the edge list is sliced per device.
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "device_rng.cuh"
#include "kernels.cuh"
#include "launch.hpp"
#include "sweep_common.cuh"

namespace gdi {

namespace {

constexpr int kNW = 16;  // warps per CTA
#ifndef K4_DEFER
#define K4_DEFER 1
#endif
// chunks per chain deferred to the CTA tail: warp 0 decides the CTA's 16 *
// kDefer tail chunks in order while the other warps wait, ~30% of an M1 sweep
// with 2 (1.74 -> 1.53 ms per 20 sweeps with 1, balance unchanged; 0 leaves
// sweeps imbalanced)
constexpr int kDefer = K4_DEFER;
constexpr int kTailMax = 32;  // global tail chunks (>= kDefer * kNW: shares stage[])
constexpr int kPackBlock = 256;
constexpr int kCutBlock = 512;

// Racy neighbour read through L2 (other chains write concurrently; L1 would
// keep a stale line for the whole sweep). WK as in K2.
template <int WK>
__device__ __forceinline__ int nb(const int8_t* s, int idx, int w) {
  if (WK == 1) {
    const int v = __ldcg(s + (idx & 0x7fffffff));
    return idx < 0 ? -v : v;
  }
  const int v = __ldcg(s + idx);
  return WK == 2 ? w * v : v;
}

struct ChunkIn {
  int v, own, f;
  bool live, coin, flip;
};

template <int WK, int KMAX>
__device__ __forceinline__ ChunkIn gather(const PartArgs& a, const int8_t* s, int c, int sweep, uint32_t k0,
                                          uint32_t k1, unsigned long long tm, bool en, int lane) {
  ChunkIn ci{0, 0, 0, false, false, false};
  const int idx = c * 32 + lane;
  ci.live = idx < a.g.n;
  if (!ci.live) return ci;
  ci.v = __ldg(a.order + idx);
  const int c0 = __ldg(a.sell_off + c), c1 = __ldg(a.sell_off + c + 1);
  const int groups = (c1 - c0) >> 5;
  int4 g4[KMAX], w4[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; k++)
    if (k < groups) {
      g4[k] = __ldg(a.sell + c0 + k * 32 + lane);
      if (WK == 2) w4[k] = __ldg(a.sell_w + c0 + k * 32 + lane);
    }
  const Philox4 x = philox4x32_10(static_cast<uint32_t>(sweep), static_cast<uint32_t>(ci.v), 0u, 0u, k0, k1);
  ci.coin = (x.z >> 31) != 0;
  ci.flip = en && ((static_cast<uint64_t>(x.x) << 32) | x.y) <= tm;
  ci.own = __ldcg(s + ci.v);
  int f = 0;
#pragma unroll
  for (int k = 0; k < KMAX; k++)
    if (k < groups) {
      const int4 q = g4[k];
      const int4 w = WK == 2 ? w4[k] : make_int4(1, 1, 1, 1);
      f += nb<WK>(s, q.x, w.x) + nb<WK>(s, q.y, w.y) + nb<WK>(s, q.z, w.z) + nb<WK>(s, q.w, w.w);
    }
  for (int k = KMAX; k < groups; k++) {
    const int4 q = __ldg(a.sell + c0 + k * 32 + lane);
    const int4 w = WK == 2 ? __ldg(a.sell_w + c0 + k * 32 + lane) : make_int4(1, 1, 1, 1);
    f += nb<WK>(s, q.x, w.x) + nb<WK>(s, q.y, w.y) + nb<WK>(s, q.z, w.z) + nb<WK>(s, q.w, w.w);
  }
  ci.f = f;
  return ci;
}

// The 32 decisions of one chunk against counter G (sequentially consistent
// inside the chunk); writes the changed spins and advances G.
__device__ __forceinline__ void decide_chunk(const ChunkIn& cur, int& G, int8_t* s, int a4, int bb, int lane,
                                             const PartArgs* peers = nullptr) {
  const unsigned below = (1u << lane) - 1u;
  const int base_diff = -a4 * cur.own - bb * cur.f;
  int fin = cur.live ? decide(a4 * G + base_diff, cur.coin, cur.flip) : 0;
  int d = cur.live ? fin - cur.own : 0;
  unsigned up = __ballot_sync(0xffffffffu, d > 0), dn = __ballot_sync(0xffffffffu, d < 0);
  if ((up | dn) != 0u) {
    for (int round = 0; round < 33; round++) {
      const int excl = 2 * (__popc(up & below) - __popc(dn & below));
      const int fin2 = cur.live ? decide(a4 * (G + excl) + base_diff, cur.coin, cur.flip) : 0;
      if (__all_sync(0xffffffffu, fin2 == fin)) break;
      fin = fin2;
      d = cur.live ? fin - cur.own : 0;
      up = __ballot_sync(0xffffffffu, d > 0);
      dn = __ballot_sync(0xffffffffu, d < 0);
    }
    if (cur.live && d != 0) {
      s[cur.v] = static_cast<int8_t>(fin);
      if (peers != nullptr)  // fused exchange: the change lands in every rank's copy
        for (int q = 0; q < peers->npeer; q++) peers->peer[q][cur.v] = static_cast<int8_t>(fin);
    }
  }
  G += 2 * (__popc(up) - __popc(dn));
}

// Initial spins (one Philox draw per vertex: the throughput mode is not
// bit-exact, so the serial stream-0 walk of anneal.cpp:148-155 is not needed)
// and the exact initial counter.
__global__ void __launch_bounds__(256) k4_init(const PartArgs a, int ns) {
  const int r = blockIdx.y, v = blockIdx.x * 256 + threadIdx.x, n = a.g.n;
  const uint64_t seed = a.seeds[r];
  int sp = 0;
  if (v < n) {
    const Philox4 x = philox4x32_10(0xffffffffu, static_cast<uint32_t>(v), 1u, 0u, static_cast<uint32_t>(seed),
                                    static_cast<uint32_t>(seed >> 32));
    sp = (x.x >> 31) ? 1 : -1;
    if (a.snaps != nullptr) a.snaps[static_cast<size_t>(r) * (a.sweeps + 1) * n + v] = static_cast<int8_t>(sp);
  }
  if (v < ns) a.spins[static_cast<size_t>(r) * ns + v] = static_cast<int8_t>(sp);  // pad (index n) = 0
  int t = sp;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __shared__ int red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    int b = 0;
    for (int w = 0; w < 8; w++) b += red[w];
    if (b != 0) atomicAdd(reinterpret_cast<unsigned long long*>(a.gsum + r), static_cast<unsigned long long>(b));
    if (blockIdx.x == 0 && a.stamps != nullptr) a.stamps[static_cast<size_t>(r) * (a.sweeps + 1)] = globaltimer_ns();
  }
}

template <int WK, int KMAX>
__global__ void __launch_bounds__(32 * kNW, KMAX >= 4 ? 1 : 2) k4_sweep(const PartArgs a, int ns) {
  __shared__ int cta_delta, cta_share, last, tail_g;
  __shared__ ChunkIn stage[kTailMax][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const int J = a.chain0 + (blockIdx.x * kNW + warp) * a.chain_stride, P = a.world_chains;
  const int n = a.g.n, nck = (n + 31) >> 5, T = (a.debug & 4) ? 0 : a.tail, nmain = nck - T;
  const int K = J < nmain ? (nmain - J + P - 1) / P : 0;
  int8_t* s = a.spins + static_cast<size_t>(r) * ns;
  const int sweep = a.sweep;
  const uint64_t seed = a.seeds[r];
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  const unsigned long long tm = a.tmask[sweep];
  const bool en = a.thr[sweep] >= 0;
  const int a4 = a.a4, bb = a.b;

  // this chain's share of the global imbalance at the last barrier, in
  // units of 2 (a spin change moves a counter by 2: a chain handed +-1 would
  // take it for balanced and keep it, so an imbalance spread as +-1 shares is
  // only half corrected); the parity bit goes to one rotating chain
  const long long Gs = a.gsum[r];
  const long long par = Gs & 1, Gh = (Gs - par) / 2;
  long long q = Gh / P, rem = Gh - q * P;
  if (rem < 0) {
    rem += P;
    q -= 1;
  }
  const int rot = static_cast<int>((J + P - sweep % P) % P);
  const int share = static_cast<int>(2 * (q + (rot < rem ? 1 : 0)) + (rot == P - 1 ? par : 0));
  if (threadIdx.x == 0) {
    cta_delta = 0;
    cta_share = 0;
  }
  __syncthreads();

  int G = share;
  // every chunk but the chain's last kDefer: those go to the CTA tail below
#pragma unroll 1
  for (int k = 0; k + kDefer < K; k++) {
    const ChunkIn cur = gather<WK, KMAX>(a, s, J + k * P, sweep, k0, k1, tm, en, lane);
    decide_chunk(cur, G, s, a4, bb, lane, a.npeer > 0 ? &a : nullptr);
  }
  // CTA tail: the 16 * kDefer deferred chunks (low-degree end of the order)
  // are decided in order by warp 0 against the CTA's exact counter (sum of
  // its chains' counters), so a CTA leaves a residual of at most a spin or
  // two instead of the sum of 16 chain residuals
#pragma unroll
  for (int d = 0; d < kDefer; d++) {
    const int k = K - kDefer + d;
    stage[d * kNW + warp][lane] =
        k >= 0 ? gather<WK, KMAX>(a, s, J + k * P, sweep, k0, k1, tm, en, lane) : ChunkIn{0, 0, 0, false, false, false};
  }
  if (lane == 0) {
    atomicAdd(&cta_delta, G - share);
    atomicAdd(&cta_share, share);
  }
  __syncthreads();
  if (warp == 0) {
    const int gc0 = cta_share + cta_delta;
    int Gc = gc0;
    for (int t = 0; t < kDefer * kNW; t++) decide_chunk(stage[t][lane], Gc, s, a4, bb, lane, a.npeer > 0 ? &a : nullptr);
    if (lane == 0) cta_delta += Gc - gc0;
    if ((a.debug & 8) && lane == 0 && a.watchdog != nullptr && sweep + 1 == a.sweeps) {
      atomicAdd(a.watchdog + 6, Gc != 0 ? 1 : 0);
      atomicAdd(a.watchdog + 7, gc0 < 0 ? -gc0 : gc0);
      atomicAdd(a.watchdog + 1, Gc < 0 ? -Gc : Gc);
    }
  }
  __threadfence();  // this CTA's spin writes before the ticket (the tail reads them)
  __syncthreads();  // (also: the CTA tail is done with stage[])
  if (threadIdx.x == 0) {
    if (cta_delta != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.gdelta + r), static_cast<unsigned long long>(cta_delta));
    last = 0;
    if (T > 0 && a.tail_ticket) {
      __threadfence();
      last = atomicAdd(a.finished + r, 1u) == gridDim.x - 1;
      if (last) {
        __threadfence();
        tail_g = static_cast<int>(a.gsum[r] + static_cast<long long>(atomicAdd(
                                                  reinterpret_cast<unsigned long long*>(a.gdelta + r), 0ull)));
        a.finished[r] = 0u;
      }
    }
  }
  __syncthreads();
  if (!last) return;
  // tail: gathered by all warps (every other chain is done), decided in
  // order by warp 0 against the exact counter
  for (int t = warp; t < T; t += kNW) stage[t][lane] = gather<WK, KMAX>(a, s, nmain + t, sweep, k0, k1, tm, en, lane);
  __syncthreads();
  if (warp != 0) return;
  const int g0 = tail_g;
  int Gt = g0;
  for (int t = 0; t < T; t++) decide_chunk(stage[t][lane], Gt, s, a4, bb, lane);
  if ((a.debug & 8) && lane == 0 && a.watchdog != nullptr && sweep + 1 == a.sweeps) {
    a.watchdog[2] = g0;
    a.watchdog[3] = Gt;
    a.watchdog[4] = T;
    a.watchdog[5] = nmain;
  }
  if (lane == 0 && Gt != g0)
    atomicAdd(reinterpret_cast<unsigned long long*>(a.gdelta + r), static_cast<unsigned long long>(Gt - g0));
}

// Barrier part 1: bit-pack the spins (bit l of word w = vertex 32w + l is
// +1), sum them, copy snapshots / final spins.
__global__ void __launch_bounds__(kPackBlock) k4_pack(const PartArgs a, int ns, int8_t* spins_out) {
  const int r = blockIdx.y, n = a.g.n, sweep = a.sweep;
  const int lane = threadIdx.x & 31;
  const int8_t* s = a.spins + static_cast<size_t>(r) * ns;
  const int nw = (n + 31) >> 5;
  const bool last_sweep = sweep + 1 == a.sweeps;
  int8_t* snap = a.snaps != nullptr ? a.snaps + (static_cast<size_t>(r) * (a.sweeps + 1) + sweep + 1) * n : nullptr;
  int sum = 0;
  const int warps = gridDim.x * (kPackBlock / 32);
  for (int w = blockIdx.x * (kPackBlock / 32) + (threadIdx.x >> 5); w < nw; w += warps) {
    const int v = 32 * w + lane;
    const int8_t x = v < n ? __ldcg(s + v) : static_cast<int8_t>(0);
    sum += x;
    const unsigned bits = __ballot_sync(0xffffffffu, x > 0);
    if (lane == 0) a.bits[static_cast<size_t>(r) * nw + w] = bits;
    if (v < n) {
      if (snap != nullptr) snap[v] = x;
      if (last_sweep) spins_out[static_cast<size_t>(r) * n + v] = x;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  __shared__ int red[kPackBlock / 32];
  if (lane == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kPackBlock / 32; w++) t += red[w];
    if (t != 0) atomicAdd(a.acc + 2 * r + 1, static_cast<unsigned long long>(static_cast<long long>(t)));
  }
}

// Barrier part 2: exact cut over this device's edge slice against the packed
// spins; the last block writes the trace record and rolls the counter.
template <int WK>
__global__ void __launch_bounds__(kCutBlock) k4_cut(const PartArgs a) {
  const int r = blockIdx.y, n = a.g.n, sweep = a.sweep;
  const uint32_t* __restrict__ bits = a.bits + static_cast<size_t>(r) * ((n + 31) >> 5);
  const long long tid = static_cast<long long>(blockIdx.x) * kCutBlock + threadIdx.x;
  const long long stride = static_cast<long long>(gridDim.x) * kCutBlock;
  long long cut = 0;
  // four edges per thread in flight (the loop was latency-serial: edge load,
  // then the two bit loads, per iteration)
  long long e = a.e_begin + tid;
  for (; e + 3 * stride < a.e_end; e += 4 * stride) {
    int2 uv[4];
#pragma unroll
    for (int q = 0; q < 4; q++) uv[q] = __ldg(a.edges + e + q * stride);
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint32_t x =
          (__ldg(bits + (uv[q].x >> 5)) >> (uv[q].x & 31)) ^ (__ldg(bits + (uv[q].y >> 5)) >> (uv[q].y & 31));
      if (x & 1u) cut += WK == 0 ? 1 : __ldg(a.edge_w + e + q * stride);
    }
  }
  for (; e < a.e_end; e += stride) {
    const int2 uv = __ldg(a.edges + e);
    const uint32_t x = (__ldg(bits + (uv.x >> 5)) >> (uv.x & 31)) ^ (__ldg(bits + (uv.y >> 5)) >> (uv.y & 31));
    if (x & 1u) cut += WK == 0 ? 1 : __ldg(a.edge_w + e);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cut += __shfl_xor_sync(0xffffffffu, cut, o);
  __shared__ long long red[kCutBlock / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cut;
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long c = 0;
  for (int w = 0; w < kCutBlock / 32; w++) c += red[w];
  if (c != 0) atomicAdd(a.acc + 2 * r, static_cast<unsigned long long>(c));
  __threadfence();
  if (atomicAdd(a.done + r, 1u) != gridDim.x - 1) return;
  __threadfence();
  const long long cv = static_cast<long long>(atomicAdd(a.acc + 2 * r, 0ull));
  const long long sv = static_cast<long long>(atomicAdd(a.acc + 2 * r + 1, 0ull));
  const long long counter = a.gsum[r] + a.gdelta[r];
  const DevTrace rec{cv, sv, counter};
  if (a.trace != nullptr) a.trace[static_cast<size_t>(r) * a.sweeps + sweep] = rec;
  if (a.stamps != nullptr) a.stamps[static_cast<size_t>(r) * (a.sweeps + 1) + sweep + 1] = globaltimer_ns();
  if (sweep + 1 == a.sweeps) a.final_out[r] = rec;
  a.gsum[r] = counter;
  a.gdelta[r] = 0;
  a.acc[2 * r] = 0ull;
  a.acc[2 * r + 1] = 0ull;
  a.done[r] = 0u;
}

// Vertex-partition exchange (rank r of W ranks owns chunks c = r (mod W)).
// Send buffer: [int64 counter delta of this sweep][uint32 word i = spins of
// chunk r + i*W, bit l = lane l's vertex is +1]. Every rank receives all W
// buffers (stride bytes apart), rewrites the other ranks' vertices in its own
// spin copy and sets the sweep's total delta for the barrier.
__global__ void __launch_bounds__(256) k4_xpack(const PartArgs a, int ns, unsigned char* send) {
  const int n = a.g.n, nck = (n + 31) >> 5, W = a.world, rk = a.rank;
  const int lane = threadIdx.x & 31;
  const int8_t* s = a.spins;
  uint32_t* words = reinterpret_cast<uint32_t*>(send + 8);
  const int nmain = nck - a.tail;  // tail chunks are recomputed identically on every rank
  const int nw = a.npeer > 0 ? 0 : nmain > rk ? (nmain - rk + W - 1) / W : 0;  // peer mode: deltas only
  for (int i = blockIdx.x * 8 + (threadIdx.x >> 5); i < nw; i += gridDim.x * 8) {
    const int idx = (rk + i * W) * 32 + lane;
    const int8_t x = idx < n ? __ldcg(s + __ldg(a.order + idx)) : static_cast<int8_t>(-1);
    const unsigned b = __ballot_sync(0xffffffffu, x > 0);
    if (lane == 0) words[i] = b;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<long long*>(send) = a.gdelta[0];
}

__global__ void __launch_bounds__(256) k4_xunpack(const PartArgs a, int ns, const unsigned char* recv,
                                                  long long stride) {
  const int n = a.g.n, nck = (n + 31) >> 5, W = a.world, rk = a.rank;
  const int lane = threadIdx.x & 31;
  int8_t* s = a.spins;
  const int nmain = a.npeer > 0 ? 0 : nck - a.tail;  // peer mode: the spins arrived during the sweep
  for (int c = blockIdx.x * 8 + (threadIdx.x >> 5); c < nmain; c += gridDim.x * 8) {
    const int q = c % W;
    if (q == rk) continue;
    const uint32_t w = reinterpret_cast<const uint32_t*>(recv + q * stride + 8)[c / W];
    const int idx = c * 32 + lane;
    if (idx < n) s[__ldg(a.order + idx)] = ((w >> lane) & 1u) ? 1 : -1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    long long d = 0;
    for (int q = 0; q < W; q++) d += *reinterpret_cast<const long long*>(recv + q * stride);
    a.gdelta[0] = d;  // the barrier folds it into the counter
  }
}

// Global tail for ranks > 1: after the exchange every rank holds the same
// spins and the exact counter, so each runs the tail chunks itself (same
// gathers, same Philox draws, one warp deciding in order) and the ranks stay
// identical without a second exchange.
template <int WK, int KMAX>
__global__ void __launch_bounds__(32 * kNW) k4_gtail(const PartArgs a, int ns) {
  __shared__ ChunkIn stage[kTailMax][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = a.g.n, nck = (n + 31) >> 5, T = a.tail, nmain = nck - T;
  const int r = blockIdx.y, sweep = a.sweep;
  int8_t* s = a.spins + static_cast<size_t>(r) * ns;
  const uint64_t seed = a.seeds[r];
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  const unsigned long long tm = a.tmask[sweep];
  const bool en = a.thr[sweep] >= 0;
  for (int t = warp; t < T; t += kNW) stage[t][lane] = gather<WK, KMAX>(a, s, nmain + t, sweep, k0, k1, tm, en, lane);
  __syncthreads();
  if (warp != 0) return;
  const int g0 = static_cast<int>(a.gsum[r] + a.gdelta[r]);
  int Gt = g0;
  for (int t = 0; t < T; t++) decide_chunk(stage[t][lane], Gt, s, a.a4, a.b, lane);
  if (lane == 0) a.gdelta[r] += Gt - g0;
}

template <int WK>
const void* gtail_fn(int kmax) {
  switch (kmax) {
    case 1: return reinterpret_cast<const void*>(&k4_gtail<WK, 1>);
    case 2: return reinterpret_cast<const void*>(&k4_gtail<WK, 2>);
    default: return reinterpret_cast<const void*>(&k4_gtail<WK, 4>);
  }
}

template <int WK>
const void* sweep_fn(int kmax) {
  switch (kmax) {
    case 1: return reinterpret_cast<const void*>(&k4_sweep<WK, 1>);
    case 2: return reinterpret_cast<const void*>(&k4_sweep<WK, 2>);
    default: return reinterpret_cast<const void*>(&k4_sweep<WK, 4>);
  }
}

}  // namespace

int part_plan(const GraphStats& st, int wkind, int32_t replicas, int64_t a4, int64_t b, PartPlan* plan) {
  long long x = a4 < 0 ? -a4 : a4, y = b < 0 ? -b : b;
  while (y) {
    const long long t = x % y;
    x = y;
    y = t;
  }
  const long long ra = a4 / x, rb = b / x;
  const double bound = static_cast<double>(ra) * (2.0 * st.n + 1) + static_cast<double>(rb) * (st.max_abs_field + 1);
  if (bound >= 2147483647.0) return -1;
  if (st.n < 1) return -1;
  // register row bucket sized by the mean degree (as K2); longer rows loop
  const double mean_deg = 2.0 * static_cast<double>(st.m) / st.n;
  const int groups = static_cast<int>((mean_deg + 3.999) / 4);
  const int kmax = groups <= 1 ? 1 : groups <= 2 ? 2 : 4;
  // chains = warps: fill the resident slots across the replicas (CTAs of 16
  // warps, 1 or 2 per SM by __launch_bounds__), at least 4 chunks per chain
  const int nck = (st.n + 31) / 32;
  const int ctas_per_sm = kmax >= 4 ? 1 : 2;
  const int R = replicas > 0 ? replicas : 1;
  int ctas = ctas_per_sm * 148 / R;
  const int max_ctas = nck / (4 * kNW);
  ctas = ctas < max_ctas ? ctas : max_ctas;
  plan->ctas = ctas < 1 ? 1 : ctas;
  plan->chains = plan->ctas * kNW;
  // tail chunks run by the last CTA against the exact counter (see k4_sweep)
  // one device: 8 chunks. The chains' residual after the CTA tails is a few
  // spins; a 32-chunk tail balanced no better (M1 and a 100k graph, 4 seeds:
  // final imbalance 0 either way) and cost a fifth of the M1 sweep (the last
  // CTA decides its chunks in order against a counter that cascades through
  // them). Partitioned over ranks the residuals of every rank's chains add
  // up: 8 chunks left a fused W=4 run imbalanced, so 32 there.
  constexpr int kTailDefault = 8;
  plan->tail = nck / 8 < kTailDefault ? nck / 8 : kTailDefault;
  plan->tail_multi = nck / 8 < kTailMax ? nck / 8 : kTailMax;
  if (const char* e = std::getenv("GDI_K4_TAIL")) {  // tuning experiments
    const int t = std::atoi(e);
    plan->tail = plan->tail_multi = t < 0 ? 0 : t > kTailMax ? kTailMax : t > nck / 8 ? nck / 8 : t;
  }
  plan->sweep_fn = wkind == 0 ? sweep_fn<0>(kmax) : wkind == 1 ? sweep_fn<1>(kmax) : sweep_fn<2>(kmax);
  plan->gtail_fn = wkind == 0 ? gtail_fn<0>(kmax) : wkind == 1 ? gtail_fn<1>(kmax) : gtail_fn<2>(kmax);
  plan->cut_fn = wkind == 0   ? reinterpret_cast<const void*>(&k4_cut<0>)
                 : wkind == 1 ? reinterpret_cast<const void*>(&k4_cut<1>)
                              : reinterpret_cast<const void*>(&k4_cut<2>);
  plan->block = 32 * kNW;
  long long cg = (st.m + kCutBlock * 8 - 1) / (kCutBlock * 8);
  plan->cut_grid = static_cast<int>(cg < 1 ? 1 : cg > 2 * 148 ? 2 * 148 : cg);
  long long pg = ((st.n + 31) / 32 + 7) / 8;
  plan->pack_grid = static_cast<int>(pg < 1 ? 1 : pg > 4 * 148 ? 4 * 148 : pg);
  plan->a4 = static_cast<int32_t>(ra);
  plan->b = static_cast<int32_t>(rb);
  plan->name = wkind == 0 ? "k4_sweep<unit>" : wkind == 1 ? "k4_sweep<pm1>" : "k4_sweep<weighted>";
  return 0;
}

int part_launch_count(const PartPlan&, int32_t sweeps) { return 1 + 3 * sweeps; }

int part_stride(int n) { return (n + 1 + 15) & ~15; }

namespace {

PartArgs prepared(const PartPlan& plan, const PartArgs& args) {
  PartArgs a = args;
  a.a4 = plan.a4;
  a.b = plan.b;
  a.tail = a.world == 1 ? plan.tail : plan.tail_multi;
  a.tail_ticket = a.world == 1 ? 1 : 0;  // ranks > 1: k4_gtail after the exchange
  const char* dbg = std::getenv("GDI_K4_DEBUG");
  a.debug = dbg ? std::atoi(dbg) : 0;
  return a;
}

}  // namespace

cudaError_t part_init_launch(const PartPlan& plan, const PartArgs& args, cudaStream_t stream) {
  PartArgs a = prepared(plan, args);
  const int ns = part_stride(a.g.n);
  const int R = a.replicas;
  cudaError_t err;
  if ((err = cudaMemsetAsync(a.gsum, 0, R * sizeof(long long), stream))) return err;
  if ((err = cudaMemsetAsync(a.gdelta, 0, R * sizeof(long long), stream))) return err;
  if ((err = cudaMemsetAsync(a.acc, 0, 2 * R * sizeof(unsigned long long), stream))) return err;
  if ((err = cudaMemsetAsync(a.done, 0, R * sizeof(unsigned int), stream))) return err;
  if ((err = cudaMemsetAsync(a.finished, 0, R * sizeof(unsigned int), stream))) return err;
  k4_init<<<dim3((ns + 255) / 256, R), 256, 0, stream>>>(a, ns);
  return cudaGetLastError();
}

cudaError_t part_sweep_launch(const PartPlan& plan, const PartArgs& args, int sweep, cudaStream_t stream) {
  PartArgs a = prepared(plan, args);
  a.sweep = sweep;
  int ns = part_stride(a.g.n);
  void* p1[] = {&a, &ns};
  return cudaLaunchKernel(plan.sweep_fn, dim3(plan.ctas, a.replicas), dim3(plan.block), p1, 0, stream);
}

cudaError_t part_barrier_launch(const PartPlan& plan, const PartArgs& args, int sweep, int8_t* spins_out,
                                cudaStream_t stream) {
  PartArgs a = prepared(plan, args);
  a.sweep = sweep;
  const int ns = part_stride(a.g.n);
  k4_pack<<<dim3(plan.pack_grid, a.replicas), kPackBlock, 0, stream>>>(a, ns, spins_out);
  cudaError_t err = cudaGetLastError();
  if (err) return err;
  void* p3[] = {&a};
  return cudaLaunchKernel(plan.cut_fn, dim3(plan.cut_grid, a.replicas), dim3(kCutBlock), p3, 0, stream);
}

cudaError_t part_xpack_launch(const PartPlan& plan, const PartArgs& args, void* send, cudaStream_t stream) {
  PartArgs a = prepared(plan, args);
  const int nck = (a.g.n + 31) / 32;
  const int nw = (nck - a.rank + a.world - 1) / a.world;
  k4_xpack<<<(nw + 7) / 8 > 0 ? ((nw + 7) / 8 < 1184 ? (nw + 7) / 8 : 1184) : 1, 256, 0, stream>>>(
      a, part_stride(a.g.n), static_cast<unsigned char*>(send));
  return cudaGetLastError();
}

cudaError_t part_xunpack_launch(const PartPlan& plan, const PartArgs& args, const void* recv, long long stride,
                                int sweep, cudaStream_t stream) {
  PartArgs a = prepared(plan, args);
  a.sweep = sweep;
  int ns = part_stride(a.g.n);
  const int nck = (a.g.n + 31) / 32;
  k4_xunpack<<<(nck + 7) / 8 < 1184 ? (nck + 7) / 8 : 1184, 256, 0, stream>>>(
      a, ns, static_cast<const unsigned char*>(recv), stride);
  cudaError_t err = cudaGetLastError();
  if (err || a.tail == 0 || a.tail_ticket) return err;
  void* p[] = {&a, &ns};
  return cudaLaunchKernel(plan.gtail_fn, dim3(1, a.replicas), dim3(plan.block), p, 0, stream);
}

long long part_exchange_bytes(int n, int world, bool peer) {
  if (peer) return 16;  // counter delta only
  const int nck = (n + 31) / 32;
  const long long words = (nck + world - 1) / world;  // rank 0 owns the most
  return (8 + 4 * words + 15) & ~15LL;
}

cudaError_t part_launch(const PartPlan& plan, const PartArgs& args, int8_t* spins_out, cudaStream_t stream) {
  cudaError_t err = part_init_launch(plan, args, stream);
  if (err) return err;
  for (int sw = 0; sw < args.sweeps; sw++) {
    if ((err = part_sweep_launch(plan, args, sw, stream))) return err;
    if ((err = part_barrier_launch(plan, args, sw, spins_out, stream))) return err;
  }
  return cudaSuccess;
}

}  // namespace gdi
