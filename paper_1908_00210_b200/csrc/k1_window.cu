// K1 v3 — bit-exact GDI sweep by speculative visit windows (sm_100a).
//
// Same contract as k1_exact.cu / k1_pipe.cu: bit-identical to the
// reference's single-worker anneal (proj/src/anneal.cpp:132-231; visit_node
// :86-128; record_barrier :165-187).
//
// Observation. In the exact sequential chain a visit only perturbs later
// visits if it changes a spin (G and a neighbour's field move) or hits an
// exact tie (one extra coin draw shifts every later draw position). Both are
// rare: on the BASELINE configs ~2% of visits (11% in the first tenth of a
// 1000-sweep anneal, 0.1% in the last; measured with the oracle). So a warp
// evaluates the next 32 visits of its replica at once (lane j = visit i0+j),
// every lane assuming no event in the lanes before it:
//   * lane j's field was gathered from the current spins, where the pending
//     lanes' vertices still hold their own (unchanged) spins;
//   * its unit draw is at pos + j (+1 for its own coin on a tie);
//   * its counter is the current G.
// A ballot finds the first lane with an event; everything up to and
// including it is exactly what the sequential chain does, so it is
// accepted: the event's spin is written, G and the draw position advance,
// and the pending lanes behind it correct their fields through the 32-bit
// window masks of the k1_pipe layout (bit k-1 of win_pos/win_neg[v]: vertex
// v-k is a +1/-1 neighbour). The window then shifts down by the accepted
// count and only the emptied lanes gather new rows. Windows never cross a
// sweep (the barrier records the exact incremental cut and the counter).
//
// Draws: one producer warp runs every replica's xoshiro256++ stream 1
// (rng.hpp:23-33; lane = replica) ahead into a per-replica shared-memory
// ring; consumers read ring[pos + lane] and ring[pos + lane + 1]. The flip
// test is the exact integer form x <= floor(pf*2^53)*2^11 + 2047, the coin is
// the sign bit. Release/acquire on shared-memory positions orders the ring;
// every polling loop has a watchdog that aborts instead of hanging.
//
// Restricted to |w| == 1 graphs with the 32-bit decision bound (k1_pipe's
// conditions); spins per replica in shared memory, or in global memory (GS)
// when they do not fit (each replica's spins are private to its warp).
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "device_rng.cuh"
#include "kernels.cuh"
#include "launch.hpp"
#include "sweep_common.cuh"

namespace gdi {

namespace {

constexpr int kRing = 256;  // draws buffered per replica (power of two, >= 34 + kGen)
#ifndef K1W_GEN
#define K1W_GEN 64
#endif
// draws per producer batch, fully unrolled: one acquire + one release per
// batch; 8 -> 16 -> 32 -> 64 measured 73.7 -> 63.8 -> 58.2 -> 54.8 ms on G22 x1024
// x1000 sweeps (128 fully unrolled thrashed the instruction cache)
constexpr int kGen = K1W_GEN;
static_assert(kRing % kGen == 0, "producer batches must not wrap the ring");
constexpr long long kWatchdog = 1LL << 28;  // polling iterations before aborting (~seconds)

// spin of SELL entry idx (bit 31 = weight -1; padding index n reads 0)
template <bool SIGNED>
__device__ __forceinline__ int nbv(const int8_t* s, int idx) {
  if (SIGNED) {
    const int v = s[idx & 0x7fffffff];
    return idx < 0 ? -v : v;
  }
  return s[idx];
}

struct WinLayout {
  int ring, genpos, cons, flags, spins, fields, total;
  __host__ __device__ static WinLayout make(int rc, int n_pad, bool gs, bool incf) {
    WinLayout L;
    L.ring = 0;
    L.genpos = L.ring + rc * kRing * 8;
    L.cons = L.genpos + 4 * 32;
    L.flags = L.cons + 4 * 32;  // [0] consumers done, [1] abort
    L.spins = L.flags + 16;
    L.fields = L.spins + (gs ? 0 : rc * n_pad);
    L.total = L.fields + (incf ? rc * n_pad * 2 : 0);
    return L;
  }
};

// INCF: every vertex's field kept exact in shared memory (int16; scattered on
// each spin change, ~2% of visits) so a window refill is two shared loads
// instead of a row gather; else rows are gathered from the natural-order
// SELL layout and pending lanes are corrected through the window masks.
template <bool SIGNED, bool UNITAB, bool GS, bool INCF>
__global__ void __launch_bounds__(512, 1) k1_window(const PipeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.g.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rc = a.rc;  // replica warps 0..rc-1, producer warps rc..rc+nprod-1
  const int n_pad = a.n_words;
  const WinLayout L = WinLayout::make(rc, n_pad, GS, INCF);
  uint64_t* ring = reinterpret_cast<uint64_t*>(smem + L.ring);
  int* genpos = reinterpret_cast<int*>(smem + L.genpos);
  int* cons = reinterpret_cast<int*>(smem + L.cons);
  int* flags = reinterpret_cast<int*>(smem + L.flags);
  const unsigned done_s = saddr(flags), abort_s = saddr(flags + 1);
  if (warp == 0) {
    genpos[lane] = 0;
    cons[lane] = 0;
    if (lane < 4) flags[lane] = 0;
  }
  __syncthreads();

  // Warp roles. rolemap 1 (default): the producer is warp 3, alone on SM
  // sub-partition 3 (warp w issues on sub-partition w % 4); consumers take the
  // warps of sub-partitions 0-2 (consumer c = warp c + c/3); the producer
  // otherwise shared its sub-partition's ALU pipe with a consumer and ran at
  // half its standalone rate. rolemap 0: consumers 0..rc-1, producers after.
  const bool rm1 = a.rolemap == 1;
  const bool producer = rm1 ? warp == 3 : warp >= rc;
  const int cw = rm1 ? (warp % 4 == 3 ? -1 : warp - warp / 4) : (producer ? -1 : warp);
  if (!producer && (cw < 0 || cw >= rc)) return;  // idle padding warp
  if (producer) {
    // ============================ producers ============================
    // producer warp p serves replicas l = p, p + np, ... (lane = l / np): a
    // stream costs ~25 instructions per draw, so one warp for all replicas
    // could not keep up with the consumers
    const int np = a.nprod, l = (rm1 ? 0 : warp - rc) + lane * np;
    const int r = blockIdx.x * rc + l;
    const bool act = l < rc && r < a.replicas;
    Xoshiro rng = Xoshiro::stream(act ? a.seeds[r] : 0ull, 1);  // anneal.cpp:191
    uint64_t* my = ring + (act ? l : 0) * kRing;
    const unsigned gp_s = saddr(genpos + (act ? l : 0)), cs_s = saddr(cons + (act ? l : 0));
    int gen = 0;
#pragma unroll 1
    for (long long spin = 0;; spin++) {
      const bool can = act && gen + kGen <= ld_acquire(cs_s) + kRing;
      if (can) {
        uint64_t* dst = my + (gen & (kRing - 1));  // batches are kGen-aligned and kGen | kRing: no wrap
#pragma unroll
        for (int k = 0; k < kGen; k++) dst[k] = rng.next();
        gen += kGen;
        st_release(gp_s, gen);
      }
      if (!__any_sync(0xffffffffu, can)) {
        // ring full: a short sleep keeps this warp's polling off the issue
        // slots the consumers need (measured: spinning, or 4 producer warps,
        // were both slower than one sleeping producer)
        if (ld_acquire(done_s) >= rc || ld_acquire(abort_s)) break;
        __nanosleep(32);
        if (spin > kWatchdog) {
          st_release(abort_s, 1);
          if (a.watchdog != nullptr) atomicCAS(a.watchdog, 0, 30);
          break;
        }
      }
    }
    return;
  }

  // ============================ replica warp ============================
  const int r = blockIdx.x * rc + cw;
  if (r >= a.replicas) {
    if (lane == 0) atomicAdd(flags, 1);
    return;
  }
  const size_t rs = static_cast<size_t>(r);
  int8_t* s = GS ? a.gspins + rs * n_pad : reinterpret_cast<int8_t*>(smem + L.spins) + cw * n_pad;
  int16_t* fld = reinterpret_cast<int16_t*>(smem + L.fields) + cw * n_pad;  // INCF only
  const int32_t* __restrict__ off = a.g.off;
  const int32_t* __restrict__ col = a.g.col;
  const int32_t* __restrict__ wgt = a.g.w;
  const int sweeps = a.sweeps;
  const unsigned FULL = 0xffffffffu;

  // init (anneal.cpp:148-155): the serial stream-0 walk, lane i%32 stores spin i
  int G = 0;
  {
    Xoshiro r0 = Xoshiro::stream(a.seeds[r], 0);
    for (int i = 0; i < n; i++) {
      const int v = (r0.next() >> 63) ? 1 : -1;
      G += v;
      if ((i & 31) == lane) s[i] = static_cast<int8_t>(v);
    }
  }
  for (int i = n + lane; i < n_pad; i += 32) s[i] = 0;  // padding index n reads spin 0
  __syncwarp();
  // exact initial cut (evaluate.cpp:10-18), lane = vertices u = lane (mod 32)
  long long cut = 0;
  for (int u = lane; u < n; u += 32) {
    const int su = s[u];
    const int e1 = __ldg(off + u + 1);
    for (int e = __ldg(off + u); e < e1; e++) {
      const int v = __ldg(col + e);
      if (v > u && s[v] != su) cut += SIGNED ? __ldg(wgt + e) : 1;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cut += __shfl_xor_sync(FULL, cut, o);
  if (INCF) {
    for (int v = lane; v < n; v += 32) {
      int acc = 0;
      const int e1 = __ldg(off + v + 1);
      for (int e = __ldg(off + v); e < e1; e++) acc += SIGNED ? __ldg(wgt + e) * s[__ldg(col + e)] : s[__ldg(col + e)];
      fld[v] = static_cast<int16_t>(acc);
    }
    __syncwarp();
  }
  if (a.snaps != nullptr)
    for (int i = lane; i < n; i += 32) a.snaps[rs * (sweeps + 1) * n + i] = s[i];
  if (lane == 0 && a.stamps != nullptr) a.stamps[rs * (sweeps + 1)] = globaltimer_ns();

  const int a4 = a.a4, bb = a.b;
  int AG = UNITAB ? G : a4 * G;  // reduced 4A * G
  int pos = 0, sweep = 0, i0 = 0, F = 0, dcut = 0;
  long long cutv = cut;
  unsigned long long tm = a.tmask[0];
  bool en = a.thr[0] >= 0;
  int own = 0, f = 0;
  uint32_t wp = 0u, wn = 0u;
  const uint64_t* myring = ring + cw * kRing;
  const unsigned gp_s = saddr(genpos + cw), cs_s = saddr(cons + cw);
  int gp = 0;
  bool aborted = false;
  const bool prof = (a.debug & 4) != 0 && a.prof != nullptr;  // GDI_PIPE_DEBUG=4: step statistics
  unsigned long long p_steps = 0, p_acc = 0, p_fill = 0, p_wait = 0, p_t0 = prof ? clock64() : 0;

#pragma unroll 1
  while (sweep < sweeps) {
    // refill the empty lanes [F, lim) of the window (vertex i0 + lane)
    const int lim = min(32, n - i0);
    const long long p_a = prof ? clock64() : 0;
    if (lane >= F && lane < lim) {
      const int v = i0 + lane;
      own = s[v];
      f = 0;
      if (INCF) {
        f = fld[v];
      } else {
        const int c = v >> 5, l = v & 31;
        const int b0 = __ldg(a.wsell_off + c), kmax = __ldg(a.wsell_off + c + 1) - b0;
        const int32_t* __restrict__ rowp = a.wsell + static_cast<size_t>(b0) * 32 + l;
        int k = 0;
        for (; k + 8 <= kmax; k += 8) {
          int u[8];
#pragma unroll
          for (int q = 0; q < 8; q++) u[q] = __ldg(rowp + (k + q) * 32);
#pragma unroll
          for (int q = 0; q < 8; q++) f += nbv<SIGNED>(s, u[q]);
        }
        for (; k < kmax; k++) f += nbv<SIGNED>(s, __ldg(rowp + k * 32));
      }
      if (!INCF) {
        wp = __ldg(a.win_pos + v);
        wn = SIGNED ? __ldg(a.win_neg + v) : 0u;
      }
    }
    F = lim;
    if (prof) p_fill += clock64() - p_a;
    // draws pos .. pos + F must be in the ring
    const long long p_w = prof ? clock64() : 0;
    if (gp < pos + F + 1 && !(a.debug & 8)) {
      for (long long k = 0; (gp = ld_acquire(gp_s)) < pos + F + 1; k++)
        if (k > kWatchdog || ld_acquire(abort_s)) {
          aborted = true;
          break;
        }
      if (aborted) break;
    }
    if (prof) p_wait += clock64() - p_w;
    const bool act = lane < F;
    const uint64_t d0 = myring[(pos + lane) & (kRing - 1)];
    const uint64_t d1 = myring[(pos + lane + 1) & (kRing - 1)];
    const int diff = UNITAB ? AG - own - f : AG - a4 * own - bb * f;
    const bool tie = diff == 0;
    const int c = diff < 0 ? 1 : diff > 0 ? -1 : (static_cast<long long>(d0) < 0 ? 1 : -1);
    const uint64_t u = tie ? d1 : d0;
    const int fin = (en && u <= tm) ? -c : c;
    const unsigned m = __ballot_sync(FULL, act && (fin != own || tie));
    int adv;
    if (m == 0u) {
      adv = F;
      pos += F;
    } else {
      const int js = __ffs(m) - 1;
      adv = js + 1;
      const int fs = __shfl_sync(FULL, fin, js), os = __shfl_sync(FULL, own, js);
      const int ts = __shfl_sync(FULL, tie ? 1 : 0, js), fj = __shfl_sync(FULL, f, js);
      pos += adv + ts;
      if (fs != os) {
        if (lane == js) s[i0 + js] = static_cast<int8_t>(fs);
        const int d = fs - os;
        AG += UNITAB ? d : a4 * d;
        dcut -= (d >> 1) * fj;
        if (INCF) {
          // scatter the change into the neighbours' fields (a row has no
          // repeated neighbour, so the lanes' updates never collide), then the
          // pending lanes reload theirs
          const int v = i0 + js;
          const int e1 = __ldg(off + v + 1);
          for (int e = __ldg(off + v) + lane; e < e1; e += 32) {
            const int u = __ldg(col + e);
            fld[u] = static_cast<int16_t>(fld[u] + (SIGNED ? __ldg(wgt + e) * d : d));
          }
          __syncwarp();
          if (lane > js && lane < F) f = fld[i0 + lane];
        } else {
          const int k = lane - js;  // pending lanes behind the event: field correction
          if (k >= 1) {
            if ((wp >> (k - 1)) & 1u) f += d;
            if (SIGNED && ((wn >> (k - 1)) & 1u)) f -= d;
          }
        }
        __syncwarp();
      }
    }
    // ring slots before pos are consumed (release: their loads are done)
    if (lane == 0) st_release(cs_s, pos);
    own = __shfl_down_sync(FULL, own, adv);
    f = __shfl_down_sync(FULL, f, adv);
    wp = __shfl_down_sync(FULL, wp, adv);
    wn = __shfl_down_sync(FULL, wn, adv);
    F -= adv;
    i0 += adv;
    if (prof) {
      p_steps++;
      p_acc += adv;
    }
    if (i0 == n) {  // record_barrier (anneal.cpp:165-187)
      cutv += dcut;
      dcut = 0;
      const int Gs = UNITAB ? AG : AG / a4;
      if (lane == 0) {
        if (a.trace != nullptr) a.trace[rs * sweeps + sweep] = DevTrace{cutv, Gs, Gs};
        if (a.stamps != nullptr) a.stamps[rs * (sweeps + 1) + sweep + 1] = globaltimer_ns();
      }
      if (a.snaps != nullptr)
        for (int i = lane; i < n; i += 32) a.snaps[(rs * (sweeps + 1) + sweep + 1) * n + i] = s[i];
      sweep++;
      i0 = 0;
      F = 0;
      if (sweep < sweeps) {
        tm = a.tmask[sweep];
        en = a.thr[sweep] >= 0;
      }
    }
  }
  if (aborted) {
    if (lane == 0) {
      st_release(abort_s, 1);
      if (a.watchdog != nullptr) atomicCAS(a.watchdog, 0, 31);
    }
  }
  __syncwarp();
  if (prof && lane == 0) {
    atomicAdd(a.prof + 0, p_steps);
    atomicAdd(a.prof + 1, p_acc);
    atomicAdd(a.prof + 2, p_fill);
    atomicAdd(a.prof + 3, static_cast<unsigned long long>(clock64() - p_t0));
    atomicAdd(a.prof + 4, p_wait);
  }
  const int Gf = UNITAB ? AG : AG / a4;
  if (lane == 0) {
    a.final_out[rs] = DevTrace{cutv, Gf, Gf};
    atomicAdd(flags, 1);
  }
  for (int i = lane; i < n; i += 32) a.spins_out[rs * n + i] = s[i];
}

template <bool S, bool U>
const void* win_fn(bool gs, bool incf) {
  if (gs) return reinterpret_cast<const void*>(&k1_window<S, U, true, false>);
  return incf ? reinterpret_cast<const void*>(&k1_window<S, U, false, true>)
              : reinterpret_cast<const void*>(&k1_window<S, U, false, false>);
}

}  // namespace

int window_plan(const GraphStats& st, const PipeGraph& pg, int32_t replicas, int64_t a4, int64_t b, int32_t sweeps,
                PipePlan* plan) {
  if (!pg.ok) return -1;
  // draw positions are 32-bit: at most one visit + one tie coin per visit
  if (2.0 * static_cast<double>(sweeps) * st.n + 2 * kRing >= 2147483647.0) return -1;
  long long x = a4 < 0 ? -a4 : a4, y = b < 0 ? -b : b;
  while (y) {
    const long long t = x % y;
    x = y;
    y = t;
  }
  const long long ra = a4 / x, rb = b / x;
  const double bound = static_cast<double>(ra) * (st.n + 3) + static_cast<double>(rb) * (st.max_abs_field + 2);
  if (bound >= 2147483647.0) return -1;
  int rc = (replicas + 147) / 148;
  rc = rc < 1 ? 1 : rc > 12 ? 12 : rc;  // block <= 512 threads (__launch_bounds__) with role padding
  const int n_pad = (st.n + 1 + 15) & ~15;
  const char* force = std::getenv("GDI_FORCE_KERNEL");
  const bool gs = WinLayout::make(rc, n_pad, false, false).total > 200 * 1024 ||
                  (force && std::string(force) == "window_gmem");
  // incremental fields when they fit next to the spins (int16 bound)
  const bool incf = !gs && st.max_abs_field < 32768 && WinLayout::make(rc, n_pad, false, true).total <= 200 * 1024 &&
                    !(force && std::string(force) == "window_masks");
  const bool unitab = ra == 1 && rb == 1;
  plan->fn = st.unit ? (unitab ? win_fn<false, true>(gs, incf) : win_fn<false, false>(gs, incf))
                     : (unitab ? win_fn<true, true>(gs, incf) : win_fn<true, false>(gs, incf));
  plan->prof = false;
  plan->gw = gs;
  plan->rc = rc;
  // one producer warp: a stream costs ~36 cycles per draw on one lane (the
  // per-warp ALU issue rate, tools/xoshiro_micro.cu), which bounds a replica
  // at ~1 visit per ~40 cycles; more producer warps did not help (issue
  // contention with the consumers)
  plan->nprod = 1;
  const char* rm = std::getenv("GDI_WINDOW_ROLEMAP");  // tuning experiments
  plan->rolemap = rm ? std::atoi(rm) : 1;
  if (plan->rolemap == 1) {
    const int last = (rc - 1) + (rc - 1) / 3;  // warp of the last consumer
    plan->block = 32 * (last + 1 > 4 ? last + 1 : 4);
  } else {
    plan->block = 32 * (rc + plan->nprod);
  }
  plan->grid = (replicas + rc - 1) / rc;
  plan->smem = WinLayout::make(rc, n_pad, gs, incf).total;
  plan->n_words = n_pad;
  plan->a4 = static_cast<int32_t>(ra);
  plan->b = static_cast<int32_t>(rb);
  static const char* names[2][3][2] = {
      {{"k1_window<signed>", "k1_window<signed,ab=1>"},
       {"k1_window<signed,gmem>", "k1_window<signed,ab=1,gmem>"},
       {"k1_window<signed,incf>", "k1_window<signed,ab=1,incf>"}},
      {{"k1_window<unit>", "k1_window<unit,ab=1>"},
       {"k1_window<unit,gmem>", "k1_window<unit,ab=1,gmem>"},
       {"k1_window<unit,incf>", "k1_window<unit,ab=1,incf>"}}};
  plan->name = names[st.unit ? 1 : 0][gs ? 1 : incf ? 2 : 0][unitab ? 1 : 0];
  return 0;
}

cudaError_t window_launch(const PipePlan& plan, const PipeArgs& args, cudaStream_t stream) {
  cudaError_t err = cudaFuncSetAttribute(plan.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, plan.smem);
  if (err != cudaSuccess) return err;
  PipeArgs a = args;
  a.rc = plan.rc;
  a.a4 = plan.a4;
  a.b = plan.b;
  a.n_words = plan.n_words;
  a.nprod = plan.nprod;
  a.rolemap = plan.rolemap;
  const char* dbg = std::getenv("GDI_PIPE_DEBUG");
  a.debug = dbg ? std::atoi(dbg) : 0;
  void* params[] = {&a};
  return cudaLaunchKernel(plan.fn, dim3(plan.grid), dim3(plan.block), params, plan.smem, stream);
}

}  // namespace gdi
