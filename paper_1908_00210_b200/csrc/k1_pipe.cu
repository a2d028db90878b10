// K1 v2 — bit-exact GDI sweep, warp-specialised pipeline (sm_100a).
//
// Same contract as k1_exact.cu (bit-identical to the reference's
// single-worker anneal, reference proj/src/anneal.cpp:132-231), restructured
// so the serial per-replica chain carries only a few ALU ops per visit.
//
// Warp roles inside one CTA (RC <= 32 replicas, lane = replica):
//  * spin words: words[v] (bit l = replica l is +1) in shared memory,
//    written by the decider with one __ballot_sync per visit.
//  * gatherers (NG warps): for global visit U = sweep*n + i they compute the
//    neighbour field of vertex i for every replica EXCLUDING the L=32
//    vertices visited immediately before U ((i-1)..(i-L) mod n). Every other
//    neighbour's latest visit is <= U-L-1, so its word is final once the
//    decider has published progress P >= U-L, and no later write can happen
//    before U. The spin-independent split of each adjacency row into "far"
//    entries and a 32-bit "window" mask is precomputed once per graph
//    (gdi_graph_create). A gatherer puts one far neighbour per lane (one
//    coalesced index load, one shared-memory word load per lane), then one
//    ballot + popc per replica turns the words into per-replica counts.
//  * producer (1 warp): runs each replica's xoshiro256++ stream 1
//    (rng.hpp:23-33) ahead of the decider into a per-lane shared-memory ring.
//  * decider (warp 0): adds the window part exactly from a 32-bit history H
//    of its own last decisions (field = f_far + 2 popc(H & mask+) -
//    2 popc(H & mask-), constants folded into f_far) and applies the
//    reference decision (anneal.cpp:94-127) in 32-bit arithmetic on
//    (4A, B) / gcd(4A, B) (same sign, same ties; selected only when the
//    reduced |4A|(n+3) + |B|(max_i sum_j |w_ij| + 2) < 2^31). Splitting off
//    the newest history bit gives
//        diff_t = W_t + fin_{t-1} * V_t,   fin_t = ((diff_t < 0) ^ flip_t) ? +1 : -1
//    with W_t, V_t, flip_t independent of fin_{t-1}.
//  * draws: a visit consumes one draw, preceded by a coin draw on an exact
//    tie (anneal.cpp:106-121). Within a chunk of visits each lane may absorb
//    one tie (its later visits shift by one draw, handled with selects); a
//    second tie of the same (active) lane in a chunk is rare and triggers an
//    exact out-of-line replay of the batch. The flip test is the exact
//    integer form x <= floor(pf*2^53)*2^11 + 2047.
//  * sync: gatherer -> decider per-batch sequence numbers; decider ->
//    gatherers progress P; producer <-> decider per-lane ring positions; all
//    release/acquire at CTA scope on shared memory. Every polling loop has a
//    watchdog that aborts the CTA (reported as an error) instead of hanging.
//
// The hot loops are kept small on purpose: warp specialisation runs three
// different loops on one SM, and a first version with fully unrolled
// gatherers spent 40% of the decider's stall samples on instruction-cache
// misses (profiles/).
//
// Restricted to |w| == 1 graphs (unit or +-1), n >= 2L, sweeps*n < 2^31;
// everything else runs k1_exact.cu. Exact incremental cut for the trace as
// in k1_exact.cu (per-sweep int32 delta: |delta| <= 2m < 2^31).
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "device_rng.cuh"
#include "kernels.cuh"
#include "launch.hpp"
#include "sweep_common.cuh"

namespace gdi {

namespace {

constexpr int kWin = 32;      // window L (history bits)
constexpr int kBatch = 8;     // visits per queue batch (B)
constexpr int kChunk = 4;     // decider visits unrolled per inner iteration
constexpr int kQB = 8;        // queue depth in batches (QB*B > L + B)
constexpr int kNW = 8;        // warps per CTA
// Warp w runs on SM sub-partition w % 4. The decider is bound by its own
// SMSP's ALU/FMA issue rate (measured: a busy co-resident warp slows it by
// half), so warp 4 - its SMSP partner - only helps with the prologue and
// then retires; the producer and the gatherers share SMSPs 1-3.
constexpr int kIdle = 4;      // SMSP 0 partner of the decider: retires after init
constexpr int kProducer = 1;  // RNG producer
constexpr int kNG = kNW - 3;  // gatherer warps (2, 3, 5, 6, 7)
constexpr int kRing = 64;     // draws buffered per lane (power of two, >= 4B)
constexpr long long kWatchdog = 1LL << 26;

// Shared-memory layout (byte offsets from the dynamic smem base).
struct Layout {
  int ring, q, qm, part, ready, genpos, cons, progress, done, abort, total;
  __host__ __device__ static Layout make(int n_words) {
    Layout L;
    L.ring = ((n_words * 4) + 15) & ~15;
    L.q = L.ring + 8 * kRing * 32;
    L.qm = L.q + 8 * kQB * kBatch * 32;
    L.part = L.qm + 8 * kQB * kBatch;
    L.ready = L.part + 8 * kNW * 32;
    L.genpos = L.ready + 4 * kQB;
    L.cons = L.genpos + 4 * 32;
    L.progress = L.cons + 4 * 32;
    L.done = L.progress + 4;
    L.abort = L.done + 4;
    L.total = L.abort + 8;
    return L;
  }
};

// Decider state between visits. H = history used by the previous visit
// (bit k-1 = spin of the visit k before it), fin/own = that visit's final and
// prior spin, AG = a*G before that visit's change was applied (a = reduced
// 4A), pos = first unconsumed draw.
struct DState {
  uint32_t H;
  int fin, own, AG, dcut, pos;
};

struct Sweep {  // per-sweep bookkeeping handled at a barrier
  long long cut;
  int sweep, i;
  unsigned long long tm;
  bool en;
};

struct ReplayIO {
  DState st;
  Sweep sw;
};

// Safety net: record why a polling loop gave up and raise the abort flag.
__device__ __noinline__ void watchdog(const PipeArgs& a, unsigned abort_s, int where, long long x, long long y) {
  st_release(abort_s, 1);
  if (a.watchdog != nullptr && atomicCAS(a.watchdog, 0, where) == 0) {
    a.watchdog[1] = static_cast<int>(blockIdx.x);
    a.watchdog[2] = static_cast<int>(threadIdx.x);
    a.watchdog[3] = static_cast<int>(x);
    a.watchdog[4] = static_cast<int>(y);
  }
}

__device__ __forceinline__ uint64_t ring_at(const uint64_t* ring, int pos, int lane) {
  return ring[(pos & (kRing - 1)) * 32 + lane];
}

// record_barrier (anneal.cpp:165-187): exact cut, spin sum, counter.
__device__ __noinline__ void record_barrier(const PipeArgs& a, const uint32_t* words, Sweep& sw, int dcut, int G,
                                            int lane, bool active, size_t rs) {
  const int n = a.g.n;
  sw.cut += dcut;
  if (active) {
    if (a.trace != nullptr) a.trace[rs * a.sweeps + sw.sweep] = DevTrace{sw.cut, G, G};
    if (a.stamps != nullptr) a.stamps[rs * (a.sweeps + 1) + sw.sweep + 1] = globaltimer_ns();
  }
  if (a.snaps != nullptr) {
    __syncwarp();
    if (active) {
      int8_t* dst = a.snaps + (rs * (a.sweeps + 1) + sw.sweep + 1) * n;
      for (int v = 0; v < n; v++) dst[v] = ((words[v] >> lane) & 1u) ? 1 : -1;
    }
  }
  if (++sw.sweep < a.sweeps) {
    sw.tm = a.tmask[sw.sweep];
    sw.en = a.thr[sw.sweep] >= 0;
  }
}

// Exact replay of one batch (rare): per-visit draw accounting straight from
// the ring, queue entries re-read from the (still valid) slot.
template <bool SIGNED>
__device__ __noinline__ void replay_batch(const PipeArgs& a, uint32_t* words, const uint64_t* ring, const int2* qs,
                                          const uint2* ms, ReplayIO& io, int nv, int lane, bool active, size_t rs) {
  const int n = a.g.n, a4 = a.a4, bb = a.b;
  DState& st = io.st;
  Sweep& sw = io.sw;
  uint32_t hist = (st.H << 1) | static_cast<uint32_t>(st.fin > 0);
  int AG = st.AG + a4 * (st.fin - st.own);
  int pos = st.pos, fin = st.fin, own = st.own;
  for (int t = 0; t < nv; t++) {
    const int2 fo = qs[t * 32];
    const uint2 mw = ms[t];
    int p = __popc(hist & mw.x);
    if (SIGNED) p -= __popc(hist & mw.y);
    const int f = fo.x + 2 * p;
    own = fo.y;
    const int diff = AG - a4 * own - bb * f;
    int c;
    if (diff == 0) {
      c = (static_cast<long long>(ring_at(ring, pos, lane)) < 0) ? 1 : -1;
      pos++;
    } else {
      c = diff < 0 ? 1 : -1;
    }
    fin = (sw.en && ring_at(ring, pos, lane) <= sw.tm) ? -c : c;
    pos++;
    const int d = fin - own;
    AG += a4 * d;
    st.dcut -= (d >> 1) * f;
    const unsigned w = __ballot_sync(0xffffffffu, fin > 0);
    if (lane == 0) words[sw.i] = w;
    if (t + 1 < nv) hist = (hist << 1) | static_cast<uint32_t>(fin > 0);
    if (++sw.i == n) {
      sw.i = 0;
      record_barrier(a, words, sw, st.dcut, AG / a4, lane, active, rs);
      st.dcut = 0;
    }
  }
  st.H = hist;
  st.fin = fin;
  st.own = own;
  st.AG = AG - a4 * (fin - own);
  st.pos = pos;
}

// PROF: accumulate clock64 wait/work counters per role into a.prof
// (profiling builds only, GDI_PIPE_PROFILE=1; see gdi_abi.cu).
// GW: spin words in global memory (one n_words slice per CTA; graphs whose
// words do not fit in shared memory, e.g. the 1M-vertex config). Only this
// CTA reads and writes its slice, so the CTA-scope release/acquire on the
// shared-memory progress counter orders them exactly as in the smem variant
// (plain loads: no non-coherent __ldg on data written during the kernel).
template <bool SIGNED, bool UNITAB, bool PROF, bool GW>
__global__ void __launch_bounds__(32 * kNW, 1) k1_pipe(const PipeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.g.n;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int rc = a.rc;
  const int replica = blockIdx.x * rc + lane;
  const bool active = lane < rc && replica < a.replicas;
  const Layout lay = Layout::make(GW ? 0 : a.n_words);
  uint32_t* words = GW ? a.gwords + static_cast<size_t>(blockIdx.x) * a.n_words : reinterpret_cast<uint32_t*>(smem);
  uint64_t* ring = reinterpret_cast<uint64_t*>(smem + lay.ring);
  int2* q = reinterpret_cast<int2*>(smem + lay.q);
  uint2* qm = reinterpret_cast<uint2*>(smem + lay.qm);
  long long* part = reinterpret_cast<long long*>(smem + lay.part);
  int* ready = reinterpret_cast<int*>(smem + lay.ready);
  int* genpos = reinterpret_cast<int*>(smem + lay.genpos);
  int* cons = reinterpret_cast<int*>(smem + lay.cons);
  int* progress = reinterpret_cast<int*>(smem + lay.progress);
  int* done = reinterpret_cast<int*>(smem + lay.done);
  const unsigned abort_s = saddr(smem + lay.abort);
  const long long total = static_cast<long long>(a.sweeps) * n;
  const int nbatches = static_cast<int>((total + kBatch - 1) / kBatch);
  const uint64_t seed = active ? a.seeds[replica] : 0ull;

  // ---------------- init (anneal.cpp:148-155): lane = replica, stream 0
  int G = 0;  // meaningful in warp 0 (the decider) only
  if (warp == 0) {
    Xoshiro r0 = Xoshiro::stream(seed, 0);
    for (int i = 0; i < n; i++) {
      const bool up = (r0.next() >> 63) != 0;
      G += up ? 1 : -1;
      const unsigned w = __ballot_sync(0xffffffffu, up);
      if (lane == 0) words[i] = w;
    }
    if (lane == 0) {
      for (int i = n; i < a.n_words; i++) words[i] = 0u;  // index n reads 0
      *progress = 0;
      *done = 0;
      *reinterpret_cast<int*>(smem + lay.abort) = 0;
    }
    if (lane < kQB) ready[lane] = -1;
    genpos[lane] = 0;
    cons[lane] = 0;
  }
  __syncthreads();

  // exact initial cut, all warps (evaluate.cpp:10-18), per lane = replica
  long long cut = 0;
  if (!GW) {
    for (int u = warp; u < n; u += kNW) {
      const unsigned su = (words[u] >> lane) & 1u;
      const int e1 = __ldg(a.g.off + u + 1);
      for (int e = __ldg(a.g.off + u); e < e1; e++) {
        const int v = __ldg(a.g.col + e);
        if (v > u && ((words[v] >> lane) & 1u) != su) cut += SIGNED ? __ldg(a.g.w + e) : 1;
      }
    }
  } else {
    // large graphs: lane = vertex (independent loads in flight), per-replica
    // counts bit-sliced in registers, then one warp reduction per replica
    int c[32];
#pragma unroll
    for (int r = 0; r < 32; r++) c[r] = 0;
    for (int u = warp * 32 + lane; u < n; u += 32 * kNW) {
      const uint32_t wu = words[u];
      const int e1 = __ldg(a.g.off + u + 1);
      for (int e = __ldg(a.g.off + u); e < e1; e++) {
        const int v = __ldg(a.g.col + e);
        if (v <= u) continue;
        const uint32_t x = wu ^ words[v];
        const int w = SIGNED ? __ldg(a.g.w + e) : 1;
#pragma unroll
        for (int r = 0; r < 32; r++)
          if (r < rc) c[r] += ((x >> r) & 1u) ? w : 0;
      }
    }
#pragma unroll
    for (int r = 0; r < 32; r++) {
      if (r >= rc) break;
      int t = c[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == r) cut = t;
    }
  }
  part[warp * 32 + lane] = cut;
  __syncthreads();

  if (warp == 0) {
    // ============================ decider ============================
    for (int w = 1; w < kNW; w++) cut += part[w * 32 + lane];
    const size_t rs = static_cast<size_t>(replica);
    const int sweeps = a.sweeps;
    if (active && a.stamps != nullptr) a.stamps[rs * (sweeps + 1)] = globaltimer_ns();
    if (active && a.snaps != nullptr)
      for (int i = 0; i < n; i++) a.snaps[rs * (sweeps + 1) * n + i] = ((words[i] >> lane) & 1u) ? 1 : -1;
    uint32_t hist0 = 0;  // bit k-1 = spin of vertex (0 - k) mod n
    for (int k = kWin; k >= 1; k--) hist0 = (hist0 << 1) | ((words[n - k] >> lane) & 1u);

    const int a4 = a.a4, bb = a.b;
    // Decider state, all in registers (only the rare replay path copies it
    // into a local struct): see DState / Sweep for the meaning.
    uint32_t H = hist0 >> 1;  // "previous visit" = vertex n-1's initial spin, no change applied
    int fin = (hist0 & 1u) ? 1 : -1, own = fin, AG = a4 * G, dcut = 0, pos = 0;
    long long cutv = cut;
    int sweep = 0, vi = 0;
    unsigned long long tm = a.tmask[0];
    bool en = a.thr[0] >= 0;
    const unsigned ready_s = saddr(ready), progress_s = saddr(progress);
    const unsigned genpos_s = saddr(genpos + lane), cons_s = saddr(cons + lane);
    int rdy = ld_acquire(ready_s);  // prefetched ready flag of the current batch
    int gp = ld_acquire(genpos_s);  // prefetched generated-draw count
    long long p_t0 = PROF ? clock64() : 0, p_ready = 0, p_gen = 0, p_replay = 0;
    auto gsum = [&](int agv) { return UNITAB ? agv : agv / a4; };

#pragma unroll 1
    for (int b = 0; b < nbatches; b++) {
      const int slot = b % kQB;
      bool aborted = false;
      const long long p_a = PROF ? clock64() : 0;
      if (rdy != b)
        for (long long k = 0; ld_acquire(ready_s + 4 * slot) != b; k++)
          if (k > kWatchdog || ld_acquire(abort_s)) {
            watchdog(a, abort_s, 1, b, ld_acquire(ready_s + 4 * slot));
            aborted = true;
            break;
          }
      const long long p_b = PROF ? clock64() : 0;
      // draws pos .. pos+2B-1 must be available (the replay may use all)
      if (!__all_sync(0xffffffffu, gp >= pos + 2 * kBatch))
        for (long long k = 0; !__all_sync(0xffffffffu, (gp = ld_acquire(genpos_s)) >= pos + 2 * kBatch); k++)
          if (k > kWatchdog || ld_acquire(abort_s)) {
            watchdog(a, abort_s, 2, b, pos);
            aborted = true;
            break;
          }
      if (PROF) {
        const long long p_c = clock64();
        p_ready += p_b - p_a;
        p_gen += p_c - p_b;
      }
      if (aborted) break;
      // prefetch next batch's flags now; their latency hides under the chunks
      rdy = ld_acquire(ready_s + 4 * ((b + 1) % kQB));
      gp = ld_acquire(genpos_s);
      const int2* qs = q + slot * kBatch * 32 + lane;
      const uint2* ms = qm + slot * kBatch;
      const long long left = total - static_cast<long long>(b) * kBatch;
      bool replay = true;  // boundary/tail batches always take the exact path
      if (left >= kBatch && vi + kBatch <= n) {
        uint32_t H1 = H;
        int fin1 = fin, own1 = own, AG1 = AG, dcut1 = dcut, pos1 = pos;
        bool dbl = false;
#pragma unroll 1
        for (int h = 0; h < kBatch; h += kChunk) {
          int2 fo[kChunk];
          uint2 mw[kChunk];
          bool fl[kChunk + 1], cn[kChunk];
#pragma unroll
          for (int t = 0; t < kChunk; t++) {
            fo[t] = qs[(h + t) * 32];
            mw[t] = ms[h + t];
          }
#pragma unroll
          for (int k = 0; k <= kChunk; k++) {  // unit draws, flip / coin predicates
            const uint64_t d = ring_at(ring, pos1 + k, lane);
            fl[k] = en && d <= tm;
            if (k < kChunk) cn[k] = static_cast<long long>(d) < 0;
          }
          bool s = false;  // this lane already consumed one coin in this chunk
#pragma unroll
          for (int t = 0; t < kChunk; t++) {
            int S = __popc((H1 << 1) & mw[t].x);
            int e = static_cast<int>(mw[t].x & 1u);
            if (SIGNED) {
              S -= __popc((H1 << 1) & mw[t].y);
              e -= static_cast<int>(mw[t].y & 1u);
            }
            const int ownt = fo[t].y;
            int W, V;
            if (UNITAB) {
              W = AG1 - ownt - (fo[t].x + 2 * S) - own1 - e;
              V = 1 - e;
            } else {
              W = AG1 - a4 * ownt - bb * (fo[t].x + 2 * S) - a4 * own1 - bb * e;
              V = a4 - bb * e;
            }
            const bool flip = s ? fl[t + 1] : fl[t];
            const bool up_tie = cn[t] != fl[t + 1];  // coin draw t, unit draw t+1
            // serial chain: diff_t = W + fin_{t-1} V
            const int diff = W + fin1 * V;
            const bool tie = diff == 0;
            const bool up = tie ? up_tie : ((diff < 0) != flip);
            dbl |= tie && s;
            s |= tie;
            const int fnew = up ? 1 : -1;
            const int bprev = fin1 > 0 ? 1 : 0;
            const int f = fo[t].x + 2 * S + 2 * e * bprev;
            AG1 += UNITAB ? (fin1 - own1) : a4 * (fin1 - own1);
            H1 = (H1 << 1) | static_cast<uint32_t>(bprev);
            dcut1 -= ((fnew - ownt) >> 1) * f;
            fin1 = fnew;
            own1 = ownt;
            const unsigned w = __ballot_sync(0xffffffffu, up);
            if (lane == 0) words[vi + h + t] = w;
          }
          pos1 += kChunk + (s ? 1 : 0);
        }
        replay = __any_sync(0xffffffffu, dbl && active);
        if (!replay) {
          H = H1;
          fin = fin1;
          own = own1;
          AG = AG1;
          dcut = dcut1;
          pos = pos1;
          vi += kBatch;
          if (vi == n) {  // batch ended exactly on the barrier
            vi = 0;
            Sweep sw{cutv, sweep, vi, tm, en};
            record_barrier(a, words, sw, dcut, gsum(AG + (UNITAB ? 1 : a4) * (fin - own)), lane, active, rs);
            cutv = sw.cut;
            sweep = sw.sweep;
            tm = sw.tm;
            en = sw.en;
            dcut = 0;
          }
        }
      }
      if (replay) {  // rare: exact replay of the batch from the saved state
        if (PROF) p_replay++;
        ReplayIO io{DState{H, fin, own, AG, dcut, pos}, Sweep{cutv, sweep, vi, tm, en}};
        replay_batch<SIGNED>(a, words, ring, qs, ms, io, left < kBatch ? static_cast<int>(left) : kBatch, lane,
                             active, rs);
        H = io.st.H;
        fin = io.st.fin;
        own = io.st.own;
        AG = io.st.AG;
        dcut = io.st.dcut;
        pos = io.st.pos;
        cutv = io.sw.cut;
        sweep = io.sw.sweep;
        vi = io.sw.i;
        tm = io.sw.tm;
        en = io.sw.en;
      }
      // publish: the batch's spin words are final (gatherers, release) and
      // draws before pos are no longer needed (producer; the ring loads were
      // consumed by this batch's decisions, so a relaxed store suffices)
      __syncwarp();
      if (lane == 0) st_release(progress_s, (b + 1) * kBatch);
      st_relaxed(cons_s, pos);
    }
    if (lane == 0) st_release(saddr(done), 1);
    if (PROF && lane == 0 && a.prof != nullptr) {
      atomicAdd(a.prof + 0, static_cast<unsigned long long>(clock64() - p_t0));
      atomicAdd(a.prof + 1, static_cast<unsigned long long>(p_ready));
      atomicAdd(a.prof + 2, static_cast<unsigned long long>(p_gen));
      atomicAdd(a.prof + 3, static_cast<unsigned long long>(p_replay));
      atomicAdd(a.prof + 4, static_cast<unsigned long long>(nbatches));
    }
    const int Gf = gsum(AG + (UNITAB ? 1 : a4) * (fin - own));
    if (active) a.final_out[rs] = DevTrace{cutv + dcut, Gf, Gf};
  } else if (warp == kIdle) {
    // nothing: keep SMSP 0 for the decider
  } else if (warp == kProducer) {
    // ============================ producer ============================
    // Each lane runs its own replica's stream as far as its own consumer
    // allows: lanes drift apart by their individual tie counts.
    Xoshiro rng = Xoshiro::stream(seed, 1);  // anneal.cpp:191
    const unsigned genpos_s = saddr(genpos + lane), cons_s = saddr(cons + lane), done_s = saddr(done);
    int gen = 0;
    long long p_t0 = PROF ? clock64() : 0, p_wait = 0;
    long long idle = 0;  // consecutive polls without progress (watchdog)
#pragma unroll 1
    for (;;) {
      const int c = ld_acquire(cons_s);
      const bool can = gen + 8 <= c + kRing;
      if (can) {
#pragma unroll
        for (int k = 0; k < 8; k++) ring[((gen + k) & (kRing - 1)) * 32 + lane] = rng.next();
        gen += 8;
        st_release(genpos_s, gen);
      }
      if (__any_sync(0xffffffffu, can)) {
        idle = 0;
      } else {
        if (ld_acquire(done_s) || ld_acquire(abort_s)) break;
        const long long p_a = PROF ? clock64() : 0;
        __nanosleep(64);
        if (PROF) p_wait += clock64() - p_a;
        if (++idle > kWatchdog) {
          watchdog(a, abort_s, 3, gen, c);
          break;
        }
      }
    }
    if (PROF && lane == 0 && a.prof != nullptr) {
      atomicAdd(a.prof + 5, static_cast<unsigned long long>(clock64() - p_t0));
      atomicAdd(a.prof + 6, static_cast<unsigned long long>(p_wait));
    }
  } else {
    // ============================ gatherers ============================
    // lane = far neighbour of the row; per replica r: popc of a ballot.
    // All index loads of a batch are issued before waiting on progress.
    const int g = warp < kIdle ? warp - 2 : warp - 3;
    const int* __restrict__ fcol = a.far_col;
    const int4* __restrict__ meta = a.far_meta;
    const unsigned progress_s = saddr(progress), ready_s = saddr(ready);
    int i0 = static_cast<int>((static_cast<long long>(g) * kBatch) % n);
    const int stride = static_cast<int>((static_cast<long long>(kNG) * kBatch) % n);
    long long p_t0 = PROF ? clock64() : 0, p_wait = 0;
#pragma unroll 1
    for (int b = g; b < nbatches; b += kNG) {
      const long long U0 = static_cast<long long>(b) * kBatch;
      const int nv = static_cast<int>(min(static_cast<long long>(kBatch), total - U0));
      const int slot = b % kQB;
      // spin-independent prefetch: lane t < B holds row t's metadata and
      // window masks; jn[t] = far entry `lane` of row t (or n -> zero word)
      int vt = i0 + (lane & (kBatch - 1));
      vt = vt >= n ? vt - n : vt;
      const int4 mine = __ldg(meta + vt);
      const uint32_t wpos = __ldg(a.win_pos + vt);
      const uint32_t wneg = SIGNED ? __ldg(a.win_neg + vt) : 0u;
      int jn[kBatch];
#pragma unroll
      for (int t = 0; t < kBatch; t++) {
        const int off = __shfl_sync(0xffffffffu, mine.x, t);
        const int deg = __shfl_sync(0xffffffffu, mine.y + mine.z, t);
        jn[t] = lane < deg ? __ldg(fcol + off + lane) : n;
      }
      const int need = static_cast<int>(U0) + kBatch - 1 - kWin;
      const long long p_a = PROF ? clock64() : 0;
      bool aborted = false;
      if (need > 0)
        for (long long k = 0; ld_acquire(progress_s) < need; k++) {
          if (k > kWatchdog || ld_acquire(abort_s)) {
            watchdog(a, abort_s, 4, b, need);
            aborted = true;
            break;
          }
          __nanosleep(20);
        }
      if (PROF) p_wait += clock64() - p_a;
      if (aborted) break;
#pragma unroll
      for (int t = 0; t < kBatch; t++) {
        if (t < nv && (a.debug & 1)) {  // timing experiment: no field work
          q[(slot * kBatch + t) * 32 + lane] = make_int2(0, 1);
          if (lane == 0) qm[slot * kBatch + t] = make_uint2(0u, 0u);
        } else if (t < nv) {
          const int4 m = make_int4(__shfl_sync(0xffffffffu, mine.x, t), __shfl_sync(0xffffffffu, mine.y, t),
                                   __shfl_sync(0xffffffffu, mine.z, t), __shfl_sync(0xffffffffu, mine.w, t));
          const int deg = m.y + m.z;
          int cnt = 0;  // lane r < rc: count for replica r
          for (int e0 = 0; e0 < deg; e0 += 32) {
            const int j = e0 == 0 ? jn[t] : (e0 + lane < deg ? __ldg(fcol + m.x + e0 + lane) : n);
            const uint32_t wj = words[j];
            const bool neg = SIGNED && (e0 + lane >= m.y) && (e0 + lane < deg);
            const unsigned nmask = SIGNED ? __ballot_sync(0xffffffffu, neg) : 0u;
            if (rc <= 8) {
#pragma unroll
              for (int r = 0; r < 8; r++) {
                const unsigned bm = __ballot_sync(0xffffffffu, (wj >> r) & 1u);
                int v = __popc(bm);
                if (SIGNED) v -= 2 * __popc(bm & nmask);
                cnt += lane == r ? v : 0;
              }
            } else {
#pragma unroll 1
              for (int r = 0; r < rc; r++) {
                const unsigned bm = __ballot_sync(0xffffffffu, (wj >> r) & 1u);
                int v = __popc(bm);
                if (SIGNED) v -= 2 * __popc(bm & nmask);
                cnt += lane == r ? v : 0;
              }
            }
          }
          int v = i0 + t;
          v = v >= n ? v - n : v;
          const int own = ((words[v] >> lane) & 1u) ? 1 : -1;
          q[(slot * kBatch + t) * 32 + lane] = make_int2(2 * cnt - m.w, own);
          const uint32_t mp = __shfl_sync(0xffffffffu, wpos, t);
          const uint32_t mn = __shfl_sync(0xffffffffu, wneg, t);
          if (lane == 0) qm[slot * kBatch + t] = make_uint2(mp, mn);
        }
      }
      __syncwarp();
      if (lane == 0) st_release(ready_s + 4 * slot, b);
      if (ld_acquire(abort_s)) break;
      i0 += stride;
      i0 = i0 >= n ? i0 - n : i0;
    }
    if (PROF && lane == 0 && a.prof != nullptr) {
      atomicAdd(a.prof + 7, static_cast<unsigned long long>(clock64() - p_t0));
      atomicAdd(a.prof + 8, static_cast<unsigned long long>(p_wait));
    }
  }

  __syncthreads();
  // final spins, all warps: spins_out[r][v] (lane = replica)
  if (active)
    for (int v = warp; v < n; v += kNW)
      a.spins_out[static_cast<size_t>(replica) * n + v] = ((words[v] >> lane) & 1u) ? 1 : -1;
}

template <bool S, bool U>
const void* pipe_fn(bool prof, bool gw) {
  if (gw) return reinterpret_cast<const void*>(&k1_pipe<S, U, false, true>);
  return prof ? reinterpret_cast<const void*>(&k1_pipe<S, U, true, false>)
              : reinterpret_cast<const void*>(&k1_pipe<S, U, false, false>);
}

long long gcd64(long long x, long long y) {
  x = x < 0 ? -x : x;
  y = y < 0 ? -y : y;
  while (y) {
    const long long t = x % y;
    x = y;
    y = t;
  }
  return x;
}

}  // namespace

size_t pipe_smem_bytes(int n_words, int) { return Layout::make(n_words).total; }

int pipe_window() { return kWin; }

int pipe_plan(const GraphStats& st, const PipeGraph& pg, int32_t replicas, int64_t a4, int64_t b,
              int32_t sweeps, PipePlan* plan) {
  if (!pg.ok) return -1;
  if (static_cast<long long>(sweeps) * st.n >= (1LL << 31) - 64) return -1;
  if (2 * st.m >= (1LL << 31)) return -1;
  // diff = 4A (G - own) - B f: dividing both coefficients by their gcd keeps
  // the sign and the exact ties
  const long long g = gcd64(a4, b);
  const long long ra = a4 / g, rb = b / g;
  const double bound = static_cast<double>(ra) * (st.n + 3) + static_cast<double>(rb) * (st.max_abs_field + 2);
  if (bound >= 2147483647.0) return -1;
  // spin words in shared memory when they fit, else in global memory
  // (GDI_FORCE_KERNEL=pipe_gmem forces the global variant: parity tests)
  const char* force = std::getenv("GDI_FORCE_KERNEL");
  const bool gw = pipe_smem_bytes(pg.n_words, kNW) > 200 * 1024 || (force && std::string(force) == "pipe_gmem");
  const size_t smem = pipe_smem_bytes(gw ? 0 : pg.n_words, kNW);
  // replicas per CTA: spread R over the SMs (the per-replica chain is the
  // bound, so fewer lanes per CTA only adds parallel CTAs)
  int rc = (replicas + 147) / 148;
  rc = rc < 1 ? 1 : rc > 32 ? 32 : rc;
  const bool unitab = ra == 1 && rb == 1;
  const bool prof = std::getenv("GDI_PIPE_PROFILE") != nullptr;
  if (st.unit)
    plan->fn = unitab ? pipe_fn<false, true>(prof, gw) : pipe_fn<false, false>(prof, gw);
  else
    plan->fn = unitab ? pipe_fn<true, true>(prof, gw) : pipe_fn<true, false>(prof, gw);
  plan->prof = prof && !gw;
  plan->gw = gw;
  plan->rc = rc;
  plan->block = 32 * kNW;
  plan->grid = (replicas + rc - 1) / rc;
  plan->smem = static_cast<int>(smem);
  plan->a4 = static_cast<int32_t>(ra);
  plan->b = static_cast<int32_t>(rb);
  static const char* names[2][2][2] = {
      {{"k1_pipe<signed>", "k1_pipe<signed,ab=1>"}, {"k1_pipe<signed,gmem>", "k1_pipe<signed,ab=1,gmem>"}},
      {{"k1_pipe<unit>", "k1_pipe<unit,ab=1>"}, {"k1_pipe<unit,gmem>", "k1_pipe<unit,ab=1,gmem>"}}};
  plan->name = names[st.unit ? 1 : 0][gw ? 1 : 0][unitab ? 1 : 0];
  return 0;
}

cudaError_t pipe_launch(const PipePlan& plan, const PipeArgs& args, cudaStream_t stream) {
  cudaError_t err = cudaFuncSetAttribute(plan.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, plan.smem);
  if (err != cudaSuccess) return err;
  PipeArgs a = args;
  a.rc = plan.rc;
  const char* dbg = std::getenv("GDI_PIPE_DEBUG");
  a.debug = dbg ? std::atoi(dbg) : 0;
  a.a4 = plan.a4;
  a.b = plan.b;
  void* params[] = {&a};
  return cudaLaunchKernel(plan.fn, dim3(plan.grid), dim3(plan.block), params, plan.smem, stream);
}

}  // namespace gdi
