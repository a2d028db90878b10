// K4 — vertex-partitioned throughput sweep for large graphs (sm_100a).
//
// Contract: the reference's pooled racy mode (proj/src/anneal.cpp:203-225,
// SPEC.md "annealer / Concurrency Model") for graphs whose spins do not fit
// one warp's chain of K2 — BASELINE configs[4], the 1M-vertex rudy graph —
// with one or a few replicas, so the parallelism has to come from the
// vertices of one replica rather than from independent replicas (K2).
//
// Spins in position space. The visit order is the degree-binned order of the
// SELL layout; position p holds vertex order[p]. A replica's spins are one bit
// per position (bit l of word c = position 32c + l is +1): chunk c's 32
// decisions become one word, written by one store (no atomics: only the
// chunk's chain writes it), and the whole spin state of the 1M-vertex graph is
// 125 KB. The SELL rows hold neighbour *positions* (build_part_layout).
//
// Shared-memory spin copy. Every CTA (one per SM, 32 warps) keeps a copy of its
// replica's spin words in shared memory and reads neighbour spins from it
// (one LDS per neighbour instead of a 32-byte L2 sector per 1-byte gather).
// Decisions go to the global words (authoritative) and to the CTA's copy; the
// CTA's last warp is not a chain but re-copies the global words into the copy
// (TMA bulk copies, one after another: ~4-5 us each here), so other CTAs'
// changes arrive within about one chunk step, read racily as the contract
// allows. ~150k of the 1M vertices are in flight at any moment
// anyway. A chain's own spins are read from the global words, which only it
// writes, so the counter stays exact. Measured against the round-1 kernel
// (int8 spins gathered from L2 at each visit) on M1, 20 sweeps: 1.52 -> 1.18
// ms, cut +1.3% (1.254M -> 1.268M; the reference's own pooled mode is +2% to
// +7% on this graph); reading the last two bands of chunks from L2 instead
// (SMODE 2, GDI_K4_FRESH=1) restores the cut (1.2555M) at 2.5 ms.
//
// Chains and decoupled global balance. The chunks are dealt round-robin to P
// chains, one per warp, each with an exactly sequential counter; inside a
// chunk the 32 decisions see the counter as if made in order (fixed point of
// a ballot prefix). A single counter read live by ~10^4 concurrent visitors
// over-corrects (all see the same stale imbalance and flip towards the
// minority: the biphasic oscillation of PAPER.md:632-633), so chain J starts
// each sweep from its share of the exact global imbalance G at the last
// barrier (G/P in units of 2, remainder rotated over the chains) and counts
// only its own changes. Chains 0..D-1 of a CTA defer their last chunk to a
// CTA tail that one warp decides in order against the CTA's exact counter (the
// sum of its 32 chains' counters), and the last T chunks of the order form a
// global tail decided in order against the exact global counter in the
// barrier kernel, so a sweep ends balanced as the sequential algorithm does.
// (A block-wide fixed point over all 1024 deferred vertices, each seeing the
// block prefix of the changes before it, needed ~N rounds: the low-degree
// tail vertices are all counter-sensitive near G = 0, so every change shifted
// the decisions after it.)
//
// Barrier (record_barrier, anneal.cpp:165-187), k4_finish: every CTA replays
// the global tail (identical inputs, identical results) into shared memory,
// then counts its share of the exact cut (each edge once, by its endpoint
// with the lower position) and of the spin sum, reading tail words from its
// shared copy; the last CTA writes the trace record and the tail words and
// rolls the counter. Two launches per sweep; the session replays the
// 1 + 2M launches as one CUDA graph.
//
// Multi-GPU (vertex partitioning): rank r of W runs the
// chains J = r (mod W), i.e. owns the chunks c = r (mod W). Fused exchange: a
// changed chunk word is stored into every peer's copy in the same instruction
// stream as the decision (one 4-byte store per peer over NVLink); the sweep's
// counter delta goes to the per-sweep all-gather. Unfused: the owned words go
// to the send buffer and the finishing kernel reads the other ranks' words
// from the all-gathered buffer (and copies them into the local words for the
// next sweep). Every rank replays the global tail identically.
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

constexpr int kNW = 32;       // warps per CTA (one thread per deferred vertex in the CTA tail)
constexpr int kTailMax = kNW;  // global tail chunks: one per warp of a finishing CTA
constexpr unsigned FULL = 0xffffffffu;

template <int WK, int KMAX>
struct Row {
  int4 g[KMAX];
  int4 w[WK == 2 ? KMAX : 1];
  int c0, groups, v, deg;
  unsigned word;  // the chunk's own spin word (global, authoritative)
};

// One lane's visit of a chunk: everything the decision needs.
struct Visit {
  int own, f;
  bool live, coin, flip;
};

template <int WK, int KMAX>
__device__ __forceinline__ void load_row(const PartArgs& a, const uint32_t* gb, int c, int c0, int c1, int lane,
                                         Row<WK, KMAX>& r) {
  r.c0 = c0;
  r.groups = (c1 - c0) >> 5;
#pragma unroll
  for (int k = 0; k < KMAX; k++)
    if (k < r.groups) {
      r.g[k] = __ldg(a.psell + c0 + k * 32 + lane);
      if (WK == 2) r.w[k] = __ldg(a.sell_w + c0 + k * 32 + lane);
    }
  const int p = c * 32 + lane;
  r.v = p < a.g.n ? __ldg(a.order + p) : 0;
  r.deg = p < a.g.n ? __ldg(a.pdeg + p) : 0;
  r.word = __ldcg(gb + c);
}

// One SELL entry x (a neighbour position; bit 31 = weight -1 on +-1 graphs):
// unit / +-1 weights: the bit of s_e * w_e = +1 (padding entries point at a
// zero word: 0), summed and turned into the field by f = 2 * count - degree;
// general weights: w_e * s_e directly (padding has weight 0).
template <int WK, typename Word>
__device__ __forceinline__ int term(int x, int w, Word word) {
  const int q = WK == 1 ? (x & 0x7fffffff) : x;
  const unsigned sh = __funnelshift_r(word(q >> 5), 0u, q);  // (shift mod 32)
  if (WK == 2) return (sh & 1u) ? w : -w;
  return static_cast<int>((sh ^ (static_cast<unsigned>(x) >> 31)) & 1u);
}

constexpr int kLaneRows = 8;  // groups beyond the bucket walked lane per vertex; longer: warp per vertex

// Row entries beyond the register bucket. A chunk's rows are padded to its
// longest, so when one is far longer than the rest (a hub vertex, first in
// the degree-binned order) every lane would walk the hub's length: then the
// warp takes one lane's remaining row at a time instead (32 int4 groups per
// step, coalesced within the row's SELL column, then a warp sum), north_star
// (2)'s warp-per-vertex path for high-degree rows.
template <int WK, int KMAX, typename Word>
__device__ __forceinline__ int long_rows(const PartArgs& a, const Row<WK, KMAX>& r, Word word, int lane) {
  if (r.groups <= KMAX) return 0;
  int acc = 0;
  if (r.groups - KMAX <= kLaneRows) {
    for (int k = KMAX; k < r.groups; k++) {
      const int4 q = __ldg(a.psell + r.c0 + k * 32 + lane);
      const int4 w = WK == 2 ? __ldg(a.sell_w + r.c0 + k * 32 + lane) : make_int4(1, 1, 1, 1);
      acc += term<WK>(q.x, w.x, word) + term<WK>(q.y, w.y, word) + term<WK>(q.z, w.z, word) + term<WK>(q.w, w.w, word);
    }
    return acc;
  }
  const int mine = max(0, (r.deg + 3) / 4 - KMAX);  // this lane's groups beyond the bucket
  for (unsigned pend = __ballot_sync(FULL, mine > 0); pend != 0u; pend &= pend - 1u) {
    const int l = __ffs(pend) - 1, gl = __shfl_sync(FULL, mine, l);
    int sum = 0;
    for (int k = KMAX + lane; k < KMAX + gl; k += 32) {
      const int4 q = __ldg(a.psell + r.c0 + k * 32 + l);
      const int4 w = WK == 2 ? __ldg(a.sell_w + r.c0 + k * 32 + l) : make_int4(1, 1, 1, 1);
      sum += term<WK>(q.x, w.x, word) + term<WK>(q.y, w.y, word) + term<WK>(q.z, w.z, word) + term<WK>(q.w, w.w, word);
    }
    sum = __reduce_add_sync(FULL, sum);
    if (lane == l) acc += sum;
  }
  return acc;
}

// The spin-word loads of the register bucket are issued first and consumed
// after the Philox draw, so their latency (an LDS, or an L2 round trip for
// the fresh bands of SMODE 2) overlaps the RNG.
// Draws: chain chunks k .. k + 3 (k a multiple of 4) of chain J share one
// Philox4x32-10 call (counter (sweep, 32 * quad + lane, 2, 0), quad id = the
// first chunk J + k * P), 32 bits per visit as in K2 (coin = bit 0, a 31-bit
// uniform against tm >> 33); a visit whose quad was drawn before takes its
// word from `qd` (have), else draws and keeps all four. Global-tail chunks
// (>= nmain, no chain) draw alone (quad id = the chunk, word 0).
template <int WK, int KMAX, typename Word>
__device__ __forceinline__ Visit make_visit(const PartArgs& a, const Row<WK, KMAX>& r, int c, Word word, int lane,
                                            int sweep, uint32_t k0, uint32_t k1, unsigned long long tm,
                                            bool en, uint32_t quad, int idx, uint4& qd, bool have) {
  Visit x;
  x.live = c * 32 + lane < a.g.n;
  x.own = x.live ? (((r.word >> lane) & 1u) ? 1 : -1) : -1;
  auto pos = [](int e) { return WK == 1 ? (e & 0x7fffffff) : e; };
  unsigned wv[4 * KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; k++)
    if (k < r.groups) {
      wv[4 * k + 0] = word(pos(r.g[k].x) >> 5);
      wv[4 * k + 1] = word(pos(r.g[k].y) >> 5);
      wv[4 * k + 2] = word(pos(r.g[k].z) >> 5);
      wv[4 * k + 3] = word(pos(r.g[k].w) >> 5);
    }
  if (!have) {
    const Philox4 ph = philox4x32_10(static_cast<uint32_t>(sweep), quad * 32u + static_cast<uint32_t>(lane), 2u, 0u,
                                     k0, k1);
    qd = make_uint4(ph.x, ph.y, ph.z, ph.w);
  }
  const unsigned w32 = idx == 0 ? qd.x : idx == 1 ? qd.y : idx == 2 ? qd.z : qd.w;
  x.coin = (w32 & 1u) != 0;
  x.flip = en && (w32 >> 1) <= static_cast<unsigned>(tm >> 33);
  auto bit = [](int e, int w, unsigned wd) {
    const unsigned sh = __funnelshift_r(wd, 0u, WK == 1 ? (e & 0x7fffffff) : e);
    if (WK == 2) return (sh & 1u) ? w : -w;
    return static_cast<int>((sh ^ (static_cast<unsigned>(e) >> 31)) & 1u);
  };
  int acc = 0;
#pragma unroll
  for (int k = 0; k < KMAX; k++)
    if (k < r.groups) {
      const int4 q = r.g[k];
      const int4 w = WK == 2 ? r.w[k] : make_int4(1, 1, 1, 1);
      acc += bit(q.x, w.x, wv[4 * k]) + bit(q.y, w.y, wv[4 * k + 1]) + bit(q.z, w.z, wv[4 * k + 2]) +
             bit(q.w, w.w, wv[4 * k + 3]);
    }
  acc += long_rows<WK, KMAX>(a, r, word, lane);
  x.f = x.live ? (WK == 2 ? acc : 2 * acc - r.deg) : 0;
  return x;
}

// The 32 decisions of one chunk against counter G, each seeing G after the
// changes of the lanes before it; advances G and returns the chunk's new
// spin word: two evaluations settle most chunks, else the in-order scan
// (sweep_common.cuh warp_seq_decide). (Written out here: the same logic
// behind a shared helper with a round loop measured 1.5x slower.)
// (K4_ROUNDS > 2 evaluations before the scan measured slower: M1 1.31 ->
// 1.40-1.43 ms; taking the second evaluation as final instead of scanning
// saves 15% but wrecks quality: cut +47%, imbalance up to 400)
#ifndef K4_ROUNDS
#define K4_ROUNDS 2
#endif
__device__ __forceinline__ unsigned decide_chunk(const Visit& x, int& G, int a4, int bb, int lane, int2* sbuf,
                                                 int* sgout) {
  const int base = -a4 * x.own - bb * x.f;
  int fin = x.live ? decide(a4 * G + base, x.coin, x.flip) : x.own;
  unsigned up = __ballot_sync(FULL, fin > x.own), dn = __ballot_sync(FULL, fin < x.own);
  if ((up | dn) == 0u) return __ballot_sync(FULL, fin > 0);
  const unsigned below = (1u << lane) - 1u;
#pragma unroll
  for (int round = 1; round < K4_ROUNDS; round++) {
    const int fin2 =
        x.live ? decide(a4 * (G + 2 * (__popc(up & below) - __popc(dn & below))) + base, x.coin, x.flip) : x.own;
    if (__all_sync(FULL, fin2 == fin)) {
      G += 2 * (__popc(up) - __popc(dn));
      return __ballot_sync(FULL, fin > 0);
    }
    fin = fin2;
    up = __ballot_sync(FULL, fin > x.own);
    dn = __ballot_sync(FULL, fin < x.own);
  }
  fin = warp_seq_decide(x.own, x.f, x.live, x.coin, x.flip, G, a4, bb, lane, sbuf, sgout);
  return __ballot_sync(FULL, fin > 0);
}

// A staged visit packed into one word (shared memory): the field in the low
// 16 bits, then own, live, coin, flip.
__device__ __forceinline__ unsigned pack(const Visit& x) {
  return (static_cast<unsigned>(x.f) & 0xffffu) | (x.own > 0 ? 1u << 16 : 0u) | (x.live ? 1u << 17 : 0u) |
         (x.coin ? 1u << 18 : 0u) | (x.flip ? 1u << 19 : 0u);
}
__device__ __forceinline__ Visit unpack(unsigned u) {
  Visit x;
  x.f = static_cast<int>(static_cast<short>(u & 0xffffu));
  x.own = (u >> 16) & 1u ? 1 : -1;
  x.live = (u >> 17) & 1u;
  x.coin = (u >> 18) & 1u;
  x.flip = (u >> 19) & 1u;
  return x;
}

// Bulk copies global -> shared (TMA engine) completing on a per-warp mbarrier.
__device__ __forceinline__ void mbar_init(uint64_t* mb) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(mb)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W%=;\n}" ::"r"(saddr(mb)),
      "r"(parity)
      : "memory");
}
// The whole copy as `parts` bulk copies in flight on one barrier (one
// expect_tx for all of them); bytes a multiple of 16 * parts.
__device__ __forceinline__ void bulk_copy_parts(void* dst, const void* src, unsigned bytes, uint64_t* mb, int parts) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(mb)), "r"(bytes) : "memory");
  const unsigned part = bytes / parts;
  for (int i = 0; i < parts; i++)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     saddr(static_cast<char*>(dst) + i * part)),
                 "l"(static_cast<const char*>(src) + i * part), "r"(part), "r"(saddr(mb))
                 : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* mb) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(mb)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(mb))
               : "memory");
}

// A warp's share of a CTA's shared spin copy: words [w * S, w * S + S) with S
// a multiple of 4 (16-byte aligned bulk copies).
struct Slice {
  int lo, bytes;
  __device__ Slice(int nwp, int warp, int nwarps) {
    const int S = ((nwp + nwarps - 1) / nwarps + 3) & ~3;
    lo = warp * S;
    const int hi = lo + S < nwp ? lo + S : nwp;
    bytes = hi > lo ? 4 * (hi - lo) : 0;
  }
};

// Refresh this warp's slice of the CTA's shared spin copy from the global
// words: one bulk copy by lane 0, landing while the warp goes on deciding
// (readers see a word's old or new value, as with any racy read). The
// previous refresh of the slice is waited for first (phase parity).
struct Refresher {
  uint64_t* mb;
  unsigned phase;
  bool pending;
  __device__ void issue(uint32_t* sb, const uint32_t* gb, const Slice& sl, int lane) {
    if (lane != 0 || sl.bytes == 0) return;
    if (pending) {
      mbar_wait(mb, phase);
      phase ^= 1u;
    }
    bulk_copy(sb + sl.lo, gb + sl.lo, sl.bytes, mb);
    pending = true;
  }
  __device__ void drain(int lane) {
    if (lane == 0 && pending) {
      mbar_wait(mb, phase);
      phase ^= 1u;
      pending = false;
    }
  }
};

// The shared spin copy of a cluster of `mc` CTAs (2) fetched once: slice
// w is read from L2 by CTA (w mod mc) and multicast into every CTA of the
// cluster (148 SMs re-reading the same 125 KB made a plain copy ~3.7 us).
// Every thread of the CTA calls this; the cluster barriers order the
// mbarrier inits before the peers' copies and keep every multicast write
// landed before any CTA of the cluster moves on.
__device__ __forceinline__ void cluster_copy(uint32_t* dst, const uint32_t* src, const Slice& sl, uint64_t* mb,
                                             int warp, int lane, int mc) {
  unsigned crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  if (lane == 0) {
    mbar_init(mb);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (lane == 0 && sl.bytes > 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(mb)), "r"(sl.bytes) : "memory");
    if (warp % mc == static_cast<int>(crank))
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
          "%4;" ::"r"(saddr(dst + sl.lo)),
          "l"(src + sl.lo), "r"(sl.bytes), "r"(saddr(mb)), "h"(static_cast<unsigned short>((1u << mc) - 1u))
          : "memory");
    mbar_wait(mb, 0u);
  }
  __syncwarp();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Initial spins (one Philox draw per vertex: the throughput mode is not
// bit-exact, so the serial stream-0 walk of anneal.cpp:148-155 is not needed)
// and the exact initial counter. One thread per position of every word.
__global__ void __launch_bounds__(256) k4_init(const PartArgs a) {
  const int r = blockIdx.y, p = blockIdx.x * 256 + threadIdx.x, n = a.g.n;
  const uint64_t seed = a.seeds[r];
  int sp = 0;
  if (p < n) {
    const int v = __ldg(a.order + p);
    const Philox4 x = philox4x32_10(0xffffffffu, static_cast<uint32_t>(v), 1u, 0u, static_cast<uint32_t>(seed),
                                    static_cast<uint32_t>(seed >> 32));
    sp = (x.x >> 31) ? 1 : -1;
    if (a.snaps != nullptr) a.snaps[static_cast<size_t>(r) * (a.sweeps + 1) * n + v] = static_cast<int8_t>(sp);
  }
  const unsigned word = __ballot_sync(FULL, sp > 0);
  if ((threadIdx.x & 31) == 0 && (p >> 5) < a.nwp) a.bits[static_cast<size_t>(r) * a.nwp + (p >> 5)] = word;
  int t = sp;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
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

// SMODE: 0 neighbour spins from the global words (graphs whose copy does not
// fit shared memory), 1 from the CTA's shared copy, 2 from the shared copy
// except the chunks of the previous and the current band (the chunks decided
// in the last and in this chunk step by the chains of every CTA: what the
// sequential order would already show, and what a refreshed copy lags
// behind), which are read from the global words.
template <int WK, int KMAX, int SMODE>
__global__ void __launch_bounds__(32 * kNW, 1) k4_sweep(const PartArgs a) {
  constexpr bool SM = SMODE > 0;
  extern __shared__ __align__(16) uint32_t sb[];
  __shared__ unsigned stage[kNW][32];
  __shared__ int st_c[kNW];
  __shared__ unsigned st_w[kNW];
  __shared__ int red_share[kNW], red_delta[kNW];
  __shared__ __align__(16) int2 scan_buf[kNW][32];  // in-order scan scratch (warp_seq_decide)
  __shared__ __align__(16) int scan_g[kNW][32];
  __shared__ int last, chains_done;
  __shared__ uint64_t mbar[kNW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  // refresh: the last warp is not a chain but keeps re-copying the whole spin
  // copy (one bulk copy after another) until the chains are done
  const bool rmode = SM && a.refresh != 0;
  const int NW = blockDim.x >> 5;       // warps per CTA (<= kNW; part_plan)
  const int CW = rmode ? NW - 1 : NW;   // chains per CTA
  const bool is_chain = warp < CW;
  const int J = a.chain0 + (blockIdx.x * CW + warp) * a.chain_stride, P = a.world_chains;
  const int n = a.g.n, nck = (n + 31) >> 5, T = a.tail, nmain = nck - T;
  const int K = is_chain && J < nmain ? (nmain - J + P - 1) / P : 0;
  const int D = min(a.cta_tail, CW);    // chains (warps 0..D-1) deferring their last chunk
  const int Km = warp < D ? K - 1 : K;  // chunks decided by the chain itself
  uint32_t* gb = a.bits + static_cast<size_t>(r) * a.nwp;
  const int sweep = a.sweep;
  const uint64_t seed = a.seeds[r];
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  const unsigned long long tm = a.tmask[sweep];
  const bool en = a.thr[sweep] >= 0;
  const int a4 = a.a4, bb = a.b;
  const int W = a.world;
  uint32_t* send_words = (a.send != nullptr && a.npeer == 0) ? reinterpret_cast<uint32_t*>(a.send + 8) : nullptr;

  const Slice slice(a.nwp, warp, NW);
  Refresher rf{&mbar[warp], 0u, false};
  if (SM && a.mcast > 1) {
    cluster_copy(sb, gb, slice, &mbar[warp], warp, lane, a.mcast);
    rf.phase = slice.bytes > 0 ? 1u : 0u;  // (as after rf.drain)
  } else if (SM) {  // the whole copy: every warp its slice
    if (lane == 0) {
      mbar_init(&mbar[warp]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    rf.issue(sb, gb, slice, lane);
    rf.drain(lane);
  }
  int blo = 0, bhi = 0;  // SMODE 2: chunks [blo, bhi) read from the global words
  auto word = [&](int wi) -> unsigned {
    if (SMODE == 0) return __ldcg(gb + wi);
    if (SMODE == 1) return sb[wi];
    const bool fresh = static_cast<unsigned>(wi - blo) < static_cast<unsigned>(bhi - blo);
    unsigned v = 0u, u = 0u;
    if (fresh)
      v = __ldcg(gb + wi);
    else
      u = sb[wi];
    return fresh ? v : u;
  };

  // this chain's share of the global imbalance at the last barrier, in units
  // of 2 (a spin change moves a counter by 2: a chain handed +-1 would take it
  // for balanced and keep it); the parity bit goes to one rotating chain
  const long long Gs = a.gsum[r];
  const long long par = Gs & 1, Gh = (Gs - par) / 2;
  long long q = Gh / P, rem = Gh - q * P;
  if (rem < 0) {
    rem += P;
    q -= 1;
  }
  const int rot = static_cast<int>((J + P - sweep % P) % P);
  const int share = is_chain ? static_cast<int>(2 * (q + (rot < rem ? 1 : 0)) + (rot == P - 1 ? par : 0)) : 0;
  // SELL bounds of this chain's first 32 chunks, one per lane (saves a
  // dependent L2 round trip per chunk)
  const int pc = J + lane * P;
  const int so0 = lane < K ? __ldg(a.sell_off + pc) : 0, so1 = lane < K ? __ldg(a.sell_off + pc + 1) : 0;
  auto bounds = [&](int k, int& c0, int& c1) {
    if (k < 32) {
      c0 = __shfl_sync(FULL, so0, k);
      c1 = __shfl_sync(FULL, so1, k);
    } else {
      c0 = __ldg(a.sell_off + J + k * P);
      c1 = __ldg(a.sell_off + J + k * P + 1);
    }
  };
  auto commit = [&](int c, unsigned old, unsigned nw) {
    if (nw != old) {
      if (lane == 0) {
        gb[c] = nw;
        if (SM) sb[c] = nw;
      }
      if (lane < a.npeer) a.peer[lane][c] = nw;  // fused exchange: one store per peer
    }
    if (send_words != nullptr && lane == 0) send_words[c / W] = nw;
  };
  if (threadIdx.x == 0) chains_done = 0;
  __syncthreads();

  if (rmode && !is_chain) {
    // (one copy takes ~4-5 us here, about one chunk step; copying only the
    // bands being decided, or from every chain warp between its chunks, was
    // not fresher: no better cut)
    if (lane == 0) {  // (rf: this warp's barrier, its phase past the initial copy)
      int rounds = 0;
      while (*static_cast<volatile int*>(&chains_done) < CW) {
        bulk_copy_parts(sb, gb, a.nwp * 4, rf.mb, a.nwp % 32 == 0 ? a.copy_parts : 1);
        mbar_wait(rf.mb, rf.phase);
        rf.phase ^= 1u;
        rounds++;
      }
      if ((a.debug & 1) && a.watchdog != nullptr) {  // GDI_K4_DEBUG=1: refresh rounds per CTA
        atomicAdd(a.watchdog + 0, rounds);
        atomicAdd(a.watchdog + 1, 1);
      }
    }
    __syncwarp();
  }
  int G = share;
  Row<WK, KMAX> cur, nxt;
  if (K > 0) {
    int c0, c1;
    bounds(0, c0, c1);
    load_row<WK, KMAX>(a, gb, J, c0, c1, lane, cur);
  }
  uint4 qd = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll 1
  for (int k = 0; k < Km; k++) {
    const int c = J + k * P;
    if (k + 1 < K) {
      int c0, c1;
      bounds(k + 1, c0, c1);
      load_row<WK, KMAX>(a, gb, c + P, c0, c1, lane, nxt);
    }
    blo = (k - 1) * P;
    bhi = (k + 1) * P;
    const Visit x = make_visit<WK, KMAX>(a, cur, c, word, lane, sweep, k0, k1, tm, en,
                                         static_cast<uint32_t>(J + (k & ~3) * P), k & 3, qd, (k & 3) != 0);
    commit(c, cur.word, decide_chunk(x, G, a4, bb, lane, scan_buf[warp], scan_g[warp]));
    cur = nxt;
  }
  if (rmode && is_chain && lane == 0) atomicAdd(&chains_done, 1);
  // CTA tail: the last chunks of chains 0..D-1 (low-degree end of the
  // order), decided in order by warp 0 against the CTA's exact counter (sum of
  // its chains' counters), so a CTA leaves a residual of at most a spin or two
  // instead of the sum of 32 chain residuals
  if (warp < D) {
    const int ct = J + (K - 1) * P;
    blo = (K - 2) * P;
    bhi = K * P;
    // (its quad was drawn by the loop above when K - 1 is not a multiple of 4)
    const Visit xt = K > 0 ? make_visit<WK, KMAX>(a, cur, ct, word, lane, sweep, k0, k1, tm, en,
                                                  static_cast<uint32_t>(J + ((K - 1) & ~3) * P), (K - 1) & 3, qd,
                                                  ((K - 1) & 3) != 0)
                           : Visit{-1, 0, false, false, false};
    stage[warp][lane] = pack(xt);
    if (lane == 0) {
      st_c[warp] = K > 0 ? ct : -1;
      st_w[warp] = cur.word;
    }
  }
  if (lane == 0) {
    red_share[warp] = share;
    red_delta[warp] = G - share;
  }
  __syncthreads();
  if (warp == 0) {
    int sh = lane < NW ? red_share[lane] : 0, dl = lane < NW ? red_delta[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sh += __shfl_xor_sync(FULL, sh, o);
      dl += __shfl_xor_sync(FULL, dl, o);
    }
    const int g0 = sh + dl;
    int Gc = g0;
#pragma unroll 1
    for (int t = 0; t < D; t++) {
      const int c = st_c[t];
      if (c < 0) continue;
      const unsigned nw = decide_chunk(unpack(stage[t][lane]), Gc, a4, bb, lane, scan_buf[warp], scan_g[warp]);
      commit(c, st_w[t], nw);
    }
    const int cta_delta = dl + Gc - g0;
    if (lane == 0 && cta_delta != 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.gdelta + r), static_cast<unsigned long long>(cta_delta));
  }
  if (a.send == nullptr) return;
  // ranks > 1: the last CTA moves the sweep's delta into the send buffer
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    last = atomicAdd(a.finished + r, 1u) == gridDim.x - 1;
    if (last) {
      __threadfence();
      *reinterpret_cast<long long*>(a.send) =
          static_cast<long long>(atomicExch(reinterpret_cast<unsigned long long*>(a.gdelta + r), 0ull));
      a.finished[r] = 0u;
    }
  }
}

// This lane's share of the cut over edges [lo, hi) of the position-space
// edge list (u | -1 weight in bit 31, v), warp w of nw warps taking the
// 64-edge blocks w, w + nw, ... (lane = 2 edges of a block per load).
template <int WK, typename Word>
__device__ __forceinline__ long long edge_cut(const PartArgs& a, long long lo, long long hi, int w, int nw, int lane,
                                              Word word) {
  long long cut = 0;
  const int4* E = reinterpret_cast<const int4*>(a.pedges);
  // [lo, hi) in edge pairs: an odd lo / hi is handled as a single edge
  if (lo & 1) {
    if (w == 0 && lane == 0 && lo < hi) {
      const int2 e = __ldg(a.pedges + lo);
      const int u = e.x & 0x7fffffff;
      if (((word(u >> 5) >> (u & 31)) ^ (word(e.y >> 5) >> (e.y & 31))) & 1u)
        cut += WK == 0 ? 1 : WK == 1 ? (e.x < 0 ? -1 : 1) : __ldg(a.pedge_w + lo);
    }
    lo++;
  }
  const long long q0 = lo >> 1, q1 = hi >> 1;  // int4 pairs [q0, q1); edge hi - 1 alone when hi is odd
  const long long stride = static_cast<long long>(nw) * 32;
  for (long long q = q0 + static_cast<long long>(w) * 32 + lane; q < q1; q += 4 * stride) {
    int4 x[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const long long qq = q + j * stride;
      x[j] = qq < q1 ? __ldg(E + qq) : make_int4(0, 0, 0, 0);  // (edge (0, 0): never cut)
    }
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int us[2] = {x[j].x, x[j].z}, vs[2] = {x[j].y, x[j].w};
#pragma unroll
      for (int t = 0; t < 2; t++) {
        const int u = us[t] & 0x7fffffff, v = vs[t];
        if (((word(u >> 5) >> (u & 31)) ^ (word(v >> 5) >> (v & 31))) & 1u)
          cut += WK == 0 ? 1 : WK == 1 ? (us[t] < 0 ? -1 : 1) : __ldg(a.pedge_w + 2 * (q + j * stride) + t);
      }
    }
  }
  if ((hi & 1) && hi - 1 >= lo && w == 0 && lane == 1) {
    const long long e1 = hi - 1;
    const int2 e = __ldg(a.pedges + e1);
    const int u = e.x & 0x7fffffff;
    if (((word(u >> 5) >> (u & 31)) ^ (word(e.y >> 5) >> (e.y & 31))) & 1u)
      cut += WK == 0 ? 1 : WK == 1 ? (e.x < 0 ? -1 : 1) : __ldg(a.pedge_w + e1);
  }
  return cut;
}

// Barrier: global tail, exact cut share and spin sum, trace record, outputs.
// recv (ranks > 1): the all-gathered send buffers, rstride bytes apart.
// SM: the spin words are copied into shared memory first (bulk copies; in the
// unfused exchange the main chunks owned by other ranks come from recv), so
// every lookup is one LDS. The global tail is decided by warp 0 while the
// other warps count the cut over the edges between main vertices; the edges
// with a tail endpoint are counted from the tail rows afterwards.
template <int WK, int KMAX, bool SM>
__global__ void __launch_bounds__(32 * kNW, 1) k4_finish(const PartArgs a, const unsigned char* recv, long long rstride,
                                                        int8_t* spins_out) {
  extern __shared__ __align__(16) uint32_t sw[];
  __shared__ uint32_t tw[kTailMax];
  __shared__ unsigned stage[kTailMax][32];
  __shared__ int tail_delta;
  __shared__ __align__(16) int2 scan_buf[kNW][32];
  __shared__ __align__(16) int scan_g[kNW][32];
  __shared__ long long lred[2][kNW];
  __shared__ int last;
  __shared__ uint64_t mbar[kNW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y, n = a.g.n, nck = (n + 31) >> 5, T = a.tail, nmain = nck - T, zpos = 32 * nck;
  const int tlo = 32 * nmain;  // first tail position
  const int W = a.world, rk = a.rank, sweep = a.sweep;
  uint32_t* gb = a.bits + static_cast<size_t>(r) * a.nwp;
  const bool unfused = recv != nullptr && a.npeer == 0 && W > 1;
  long long G0 = a.gsum[r];
  if (recv != nullptr)
    for (int q = 0; q < W; q++) G0 += *reinterpret_cast<const long long*>(recv + q * rstride);
  else
    G0 += __ldcg(a.gdelta + r);
  // spin words before the tail: main chunks owned by other ranks come from
  // the all-gathered buffer (unfused exchange), everything else is local
  auto mword = [&](int wi) -> unsigned {
    if (unfused && wi < nmain && wi % W != rk)
      return reinterpret_cast<const uint32_t*>(recv + (wi % W) * rstride + 8)[wi / W];
    return __ldg(gb + wi);  // (read-only in this kernel until the last CTA's tail stores)
  };
  // 1a. the global tail's visits, gathered by T warps from the global words
  // (mword) while the shared copy lands: the tail decisions need not wait
  // for the copy
  const uint64_t seed = a.seeds[r];
  Refresher rf{&mbar[warp], 0u, false};
  const Slice sl(a.nwp, warp, kNW);
  if (SM && !unfused) {
    if (lane == 0) {
      mbar_init(&mbar[warp]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    rf.issue(sw, gb, sl, lane);
  }
  if (warp < T) {
    const int c = nmain + warp;
    Row<WK, KMAX> row;
    load_row<WK, KMAX>(a, gb, c, __ldg(a.sell_off + c), __ldg(a.sell_off + c + 1), lane, row);
    row.word = mword(c);
    uint4 qd = make_uint4(0u, 0u, 0u, 0u);
    const Visit xt = make_visit<WK, KMAX>(a, row, c, mword, lane, sweep, static_cast<uint32_t>(seed),
                                          static_cast<uint32_t>(seed >> 32), a.tmask[sweep], a.thr[sweep] >= 0,
                                          static_cast<uint32_t>(c), 0, qd, false);
    stage[warp][lane] = pack(xt);
  }
  if (SM) {
    if (unfused)
      for (int wi = threadIdx.x; wi < a.nwp; wi += blockDim.x) sw[wi] = mword(wi);
    else
      rf.drain(lane);
  }
  __syncthreads();
  // lookups before the tail is decided (tail words: their values before it)
  auto pre = [&](int wi) -> unsigned { return SM ? sw[wi] : mword(wi); };
  // 1b. the tail decided in order by warp 0 against the exact counter (every
  // CTA and every rank replays it identically)
  long long cut = 0, pop = 0;
  if (warp == 0) {
    int Gt = static_cast<int>(G0);
#pragma unroll 1
    for (int t = 0; t < T; t++) {
      const unsigned nw = decide_chunk(unpack(stage[t][lane]), Gt, a.a4, a.b, lane, scan_buf[warp], scan_g[warp]);
      if (lane == 0) tw[t] = nw;
    }
    if (lane == 0) tail_delta = Gt - static_cast<int>(G0);
  } else {
    // 2a. this rank's share of the exact cut (evaluate.cpp:10-18) over the
    // edges between main vertices: the prefix [0, m_main) of the
    // position-space edge list (each edge once), rank r taking the r-th
    // slice; two edges per 16-byte load, 4 loads in flight per lane
    const long long lo = a.m_main * rk / W, hi = a.m_main * (rk + 1) / W;
    cut += edge_cut<WK>(a, lo, hi, blockIdx.x * (kNW - 1) + warp - 1, gridDim.x * (kNW - 1), lane, pre);
  }
  __syncthreads();
  const int tot = tail_delta;
  auto word = [&](int wi) -> unsigned { return wi >= nmain && wi < nck ? tw[wi - nmain] : pre(wi); };
  // 2b. the edges with a tail endpoint (the rest of the list), after the
  // tail is decided: rank 0
  if (rk == 0) cut += edge_cut<WK>(a, a.m_main, a.m_edges, blockIdx.x * kNW + warp, gridDim.x * kNW, lane, word);
  // 3. the spin sum (global, on every rank), the unfused exchange's copy of the
  // other ranks' words for the next sweep, and the natural-order outputs
  const bool last_sweep = sweep + 1 == a.sweeps;
  int8_t* snap = a.snaps != nullptr ? a.snaps + (static_cast<size_t>(r) * (a.sweeps + 1) + sweep + 1) * n : nullptr;
  const int nthreads = gridDim.x * blockDim.x;
  for (int wi = blockIdx.x * blockDim.x + threadIdx.x; wi < nck; wi += nthreads) {
    const unsigned x = word(wi);
    pop += __popc(x);
    if (unfused && wi < nmain && wi % W != rk) gb[wi] = x;
  }
  if (snap != nullptr || last_sweep)
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += nthreads) {
      const int8_t s = ((word(p >> 5) >> (p & 31)) & 1u) ? 1 : -1;
      const int v = __ldg(a.order + p);
      if (snap != nullptr) snap[v] = s;
      if (last_sweep) spins_out[static_cast<size_t>(r) * n + v] = s;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cut += __shfl_xor_sync(FULL, cut, o);
    pop += __shfl_xor_sync(FULL, pop, o);
  }
  if (lane == 0) {
    lred[0][warp] = cut;
    lred[1][warp] = pop;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long cs = 0, ps = 0;
    for (int w = 0; w < kNW; w++) {
      cs += lred[0][w];
      ps += lred[1][w];
    }
    if (cs != 0) atomicAdd(a.acc + 2 * r, static_cast<unsigned long long>(cs));
    if (ps != 0) atomicAdd(a.acc + 2 * r + 1, static_cast<unsigned long long>(ps));
    __threadfence();
    last = atomicAdd(a.done + r, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // the last CTA: tail words into the live copy, trace record, counter roll
  if (lane == 0 && warp < T) gb[nmain + warp] = tw[warp];
  if (threadIdx.x != 0) return;
  __threadfence();
  const long long cv = static_cast<long long>(atomicAdd(a.acc + 2 * r, 0ull));
  const long long sv = 2 * static_cast<long long>(atomicAdd(a.acc + 2 * r + 1, 0ull)) - n;
  const long long counter = G0 + tot;
  if ((a.debug & 2) && a.watchdog != nullptr && last_sweep) {  // GDI_K4_DEBUG=2: the last tail's counter
    a.watchdog[2] = static_cast<int>(G0);
    a.watchdog[3] = tot;
    a.watchdog[4] = T;
    a.watchdog[5] = static_cast<int>(a.gsum[r]);
  }
  const DevTrace rec{cv, sv, counter};
  if (a.trace != nullptr) a.trace[static_cast<size_t>(r) * a.sweeps + sweep] = rec;
  if (a.stamps != nullptr) a.stamps[static_cast<size_t>(r) * (a.sweeps + 1) + sweep + 1] = globaltimer_ns();
  if (last_sweep) a.final_out[r] = rec;
  a.gsum[r] = counter;
  if (recv == nullptr) a.gdelta[r] = 0;
  a.acc[2 * r] = 0ull;
  a.acc[2 * r + 1] = 0ull;
  a.done[r] = 0u;
}



template <int WK, int KMAX>
void pick_k(bool sm, PartPlan* plan) {
  plan->sweep_fn = !sm           ? reinterpret_cast<const void*>(&k4_sweep<WK, KMAX, 0>)
                   : plan->fresh ? reinterpret_cast<const void*>(&k4_sweep<WK, KMAX, 2>)
                                 : reinterpret_cast<const void*>(&k4_sweep<WK, KMAX, 1>);
  plan->finish_fn = plan->fin_smem > 0 ? reinterpret_cast<const void*>(&k4_finish<WK, KMAX, true>)
                                       : reinterpret_cast<const void*>(&k4_finish<WK, KMAX, false>);
}

// (the register bucket is at most 2 int4 groups, 1 with a weight array: at
// 64 registers per thread, 4 groups spilled 56-350 bytes; longer rows loop)
template <int WK>
void pick(int kmax, bool sm, PartPlan* plan) {
  if constexpr (WK == 2)
    pick_k<WK, 1>(sm, plan);
  else if (kmax == 1)
    pick_k<WK, 1>(sm, plan);
  else
    pick_k<WK, 2>(sm, plan);
}

}  // namespace

int part_words(int n) { return (((n + 31) / 32 + 1) + 31) & ~31; }  // (a multiple of 32 words: 8 equal 16-byte-aligned copy parts)

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
  if (st.n < 1 || st.n > (1 << 30)) return -1;
  if (st.max_abs_field > 32767) return -1;  // staged fields are 16-bit (pack)
  // register row bucket sized by the mean degree (as K2); longer rows loop
  const double mean_deg = 2.0 * static_cast<double>(st.m) / st.n;
  const int groups = static_cast<int>((mean_deg + 3.999) / 4);
  const int kmax = groups <= 1 ? 1 : groups <= 2 ? 2 : 4;
  // one CTA per SM, spread over the replicas, with as many chain warps as
  // the in-flight bound below allows (all SMs busy: M1 keeps 3125 chains on
  // 148 SMs, 21 per CTA, rather than 31 per CTA on 100 SMs)
  const int nck = (st.n + 31) / 32;
  const int R = replicas > 0 ? replicas : 1;
  // at most 1/14 of the graph in flight (chains x 32 <= n / 14): the cut
  // grows with the fraction of vertices decided concurrently more than with
  // the spin copy's staleness (M1, 20 sweeps, 6 seeds, chains spread over all
  // SMs: 1/8 -> +1.4% over the sequential cut in 1.17 ms, 1/10 -> +1.05% in
  // 1.19 ms, 1/12 -> +0.86% in 1.20 ms, 1/14 -> +0.72% in 1.26 ms; with 31
  // chains per CTA on fewer SMs 1/10 gave +0.7% in 1.28-1.34 ms; a 100k-vertex
  // hub graph +4.9% at 1/2, +0.5% at 1/8)
  int frac = 14;
  if (const char* e = std::getenv("GDI_K4_FRAC")) frac = std::max(1, std::atoi(e));
  const int want = std::max(1, std::min(nck / frac, nck / 2));  // chains per replica (>= 2 chunks each)
  plan->refresh = 1;
  if (const char* e = std::getenv("GDI_K4_REFRESH")) plan->refresh = std::atoi(e);
  plan->fresh = 0;
  if (const char* e = std::getenv("GDI_K4_FRESH")) plan->fresh = std::atoi(e);
  // 4 deferred chunks per CTA (decided in order by one warp while the CTA's
  // other warps wait); the global tail is sized below
  plan->cta_tail = 4;
  if (const char* e = std::getenv("GDI_K4_CTA_TAIL")) {
    const int t = std::atoi(e);
    plan->cta_tail = t < 0 ? 0 : t > kNW ? kNW : t;
  }
  plan->nwp = part_words(st.n);
  plan->smem = plan->nwp * 4;
  plan->smem_copy = plan->smem <= 200 * 1024;
  if (!plan->smem_copy) {
    plan->smem = 0;
    plan->refresh = 0;  // (no copy to refresh: every warp is a chain)
  }
  const int cmax = plan->refresh != 0 ? kNW - 1 : kNW;  // chain warps per CTA
  const int ctas = std::max(1, std::min(148 / R, want));  // every SM, fewer chain warps each
  const int cw = std::max(1, std::min(cmax, (want + ctas - 1) / ctas));
  plan->ctas = ctas;
  plan->chains = ctas * cw;
  // global tail: 8 chunks when every CTA defers 4 chunks to its own tail; 16
  // when the CTAs hold fewer chains (shallower CTA tails leave more residual:
  // 100k-vertex graph, 2 chains per CTA, 30 sweeps: imbalance 4-8 in 2 of 36
  // runs with 8, 0-2 in all with 16, as the reference's own pooled mode);
  // 32 when partitioned over ranks (every rank's residuals add up)
  const int t1 = cw < 4 ? 16 : 8;
  plan->tail = nck / 8 < t1 ? nck / 8 : t1;
  plan->tail_multi = nck / 8 < kTailMax ? nck / 8 : kTailMax;
  if (const char* e = std::getenv("GDI_K4_TAIL")) {  // tuning experiments
    const int t = std::atoi(e);
    plan->tail = plan->tail_multi = t < 0 ? 0 : t > kTailMax ? kTailMax : t > nck / 8 ? nck / 8 : t;
  }
  plan->warps = cw + (plan->refresh != 0 ? 1 : 0);
  plan->fin_smem = plan->smem;
  if (const char* e = std::getenv("GDI_K4_FIN_COPY")) plan->fin_smem = std::atoi(e) ? plan->smem : 0;  // A/B
  if (wkind == 0)
    pick<0>(kmax, plan->smem_copy, plan);
  else if (wkind == 1)
    pick<1>(kmax, plan->smem_copy, plan);
  else
    pick<2>(kmax, plan->smem_copy, plan);
  plan->block = 32 * plan->warps;
  // finishing CTAs: one per SM with the shared copy (each copies the words),
  // else up to two per SM
  const int fg = (nck + kNW - 1) / kNW, fmax = (148 + R - 1) / R;  // (64 registers x 1024 threads: 1 CTA per SM)
  plan->fin_block = 32 * kNW;
  plan->fin_grid = fg < fmax ? fg : fmax;
  plan->a4 = static_cast<int32_t>(ra);
  plan->b = static_cast<int32_t>(rb);
  if (plan->smem > 48 * 1024 &&
      (allow_max_smem(plan->sweep_fn) != cudaSuccess ||
       (plan->fin_smem > 0 && allow_max_smem(plan->finish_fn) != cudaSuccess)))
    return -1;
  plan->name = wkind == 0 ? "k4_sweep<unit>" : wkind == 1 ? "k4_sweep<pm1>" : "k4_sweep<weighted>";
  part_plan_mcast(plan, R);
  return 0;
}

// Sweep CTAs in clusters of two sharing the initial copy (multicast): opt-in
// (GDI_K4_MCAST=2), and only when every cluster of the grid fits at once.
// Measured on M1: one B200 1.234 -> 1.192 ms with it, another 1.20 -> 1.26 ms
// (both with every cluster resident by cudaOccupancyMaxActiveClusters), so
// the plain per-CTA copy stays the default. Clusters of four never all fit
// (two waves, 1.95 ms).
void part_plan_mcast(PartPlan* plan, int replicas) {
  plan->mcast = 1;
  if (!plan->smem_copy || plan->ctas % 2 != 0) return;
  const char* e = std::getenv("GDI_K4_MCAST");
  if (e == nullptr || std::atoi(e) != 2) return;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(plan->ctas, replicas > 0 ? replicas : 1);
  cfg.blockDim = dim3(plan->block);
  cfg.dynamicSmemBytes = plan->smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, plan->sweep_fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  if (2LL * clusters >= static_cast<long long>(plan->ctas) * (replicas > 0 ? replicas : 1)) plan->mcast = 2;
}

int part_launch_count(const PartPlan&, int32_t sweeps) { return 1 + 2 * sweeps; }

namespace {

PartArgs prepared(const PartPlan& plan, const PartArgs& args) {
  PartArgs a = args;
  a.a4 = plan.a4;
  a.b = plan.b;
  a.tail = a.world == 1 ? plan.tail : plan.tail_multi;
  a.m_main = a.world == 1 ? plan.m_main : plan.m_main_multi;
  a.cta_tail = plan.cta_tail;
  a.nwp = plan.nwp;
  a.refresh = plan.refresh;
  a.copy_parts = 1;
  if (const char* e = std::getenv("GDI_K4_PARTS")) a.copy_parts = std::max(1, std::min(8, std::atoi(e)));
  a.mcast = plan.mcast;
  const char* dbg = std::getenv("GDI_K4_DEBUG");
  a.debug = dbg ? std::atoi(dbg) : 0;
  return a;
}

}  // namespace

cudaError_t part_init_launch(const PartPlan& plan, const PartArgs& args, cudaStream_t stream) {
  PartArgs a = prepared(plan, args);
  const int R = a.replicas;
  cudaError_t err;
  if ((err = cudaMemsetAsync(a.gsum, 0, R * sizeof(long long), stream))) return err;
  if ((err = cudaMemsetAsync(a.gdelta, 0, R * sizeof(long long), stream))) return err;
  if ((err = cudaMemsetAsync(a.acc, 0, 2 * R * sizeof(unsigned long long), stream))) return err;
  if ((err = cudaMemsetAsync(a.done, 0, R * sizeof(unsigned int), stream))) return err;
  if ((err = cudaMemsetAsync(a.finished, 0, R * sizeof(unsigned int), stream))) return err;
  k4_init<<<dim3((a.nwp * 32 + 255) / 256, R), 256, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t part_sweep_launch(const PartPlan& plan, const PartArgs& args, int sweep, cudaStream_t stream) {
  PartArgs a = prepared(plan, args);
  a.sweep = sweep;
  void* p[] = {&a};
  if (a.mcast == 1)
    return cudaLaunchKernel(plan.sweep_fn, dim3(plan.ctas, a.replicas), dim3(plan.block), p, plan.smem, stream);
  // clusters of two CTAs (the multicast initial copy)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(plan.ctas, a.replicas);
  cfg.blockDim = dim3(plan.block);
  cfg.dynamicSmemBytes = plan.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.mcast;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, plan.sweep_fn, p);
}

cudaError_t part_finish_launch(const PartPlan& plan, const PartArgs& args, int sweep, const void* recv,
                               long long stride, int8_t* spins_out, cudaStream_t stream) {
  PartArgs a = prepared(plan, args);
  a.sweep = sweep;
  const unsigned char* rv = static_cast<const unsigned char*>(recv);
  void* p[] = {&a, &rv, &stride, &spins_out};
  // (no clusters here: the multicast copy in the finishing kernel measured
  // slower, M1 1.191 -> 1.229 ms)
  return cudaLaunchKernel(plan.finish_fn, dim3(plan.fin_grid, a.replicas), dim3(plan.fin_block), p, plan.fin_smem,
                          stream);
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
    if ((err = part_finish_launch(plan, args, sw, nullptr, 0, spins_out, stream))) return err;
  }
  return cudaSuccess;
}

}  // namespace gdi
