// K1 v3 — bit-exact GDI sweep by speculative visit windows (sm_100a).
//
// Same contract as k1_exact.cu / k1_block.cu: bit-identical to the
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
// window masks of the k1_window layout (bit k-1 of win_pos/win_neg[v]: vertex
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
// Restricted to |w| == 1 graphs with the 32-bit decision bound
// (window_plan); spins per replica in shared memory, or in global memory (GS)
// when they do not fit (each replica's spins are private to its warp).
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>
#include <string>
#include <utility>
#include <vector>

#include "device_rng.cuh"
#include "kernels.cuh"
#include "launch.hpp"
#include "sweep_common.cuh"

namespace gdi {

namespace {

// Draw ring per replica: a power of two of draws holding more than two rounds
// of kp segments of L draws (kp lanes of the producer warp per stream; ring
// and L chosen per plan to fit shared memory)
constexpr int kRingMax = 4096;
#ifndef K1W_SPEC
#define K1W_SPEC 1  // draws read before the ring check
#endif
#ifndef K1W_PROF
#define K1W_PROF 0  // 1: step statistics (GDI_PIPE_DEBUG=4) and the no-wait timing mode (8)
#endif
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
  int ring, jump, genpos, cons, flags, spins, fields, masks, total;
  // fb: bytes per exact field (0 = no INCF fields, 1 = int8, 2 = int16)
  __host__ __device__ static WinLayout make(int rc, int n_pad, bool gs, int fb, int ring_n, int mask_words = 0,
                                            bool jt2 = false) {
    WinLayout L;
    L.ring = 0;
    L.jump = L.ring + rc * ring_n * 8;  // 256 x 32 B jump matrix, or the 128 x 4 x 32 B two-column table
    L.genpos = L.jump + (jt2 ? 128 * 4 * 32 : 256 * 32);
    L.cons = L.genpos + 4 * 32;
    L.flags = L.cons + 4 * 32;  // [0] consumers done, [1] abort
    L.spins = L.flags + 16;
    L.fields = L.spins + (gs ? 0 : rc * n_pad);
    L.masks = (L.fields + rc * n_pad * fb + 15) & ~15;
    L.total = L.masks + mask_words * n_pad * 4;
    return L;
  }
};

// INCF: every vertex's field kept exact in shared memory (int8 or int16; scattered on
// each spin change, ~2% of visits) so a window refill is two shared loads
// instead of a row gather; else rows are gathered from the natural-order
// SELL layout and pending lanes are corrected through the window masks.
template <bool SIGNED, bool UNITAB, bool GS, int INCF>  // INCF: bytes per exact field (0 = gathered rows)
__global__ void __launch_bounds__(512, 1) k1_window(const PipeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.g.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rc = a.rc;  // replica warps 0..rc-1, producer warps rc..rc+nprod-1
  const int n_pad = a.n_words;
  const int kp = a.kp, SL = a.segl, ringN = a.ring_n, rmask = ringN - 1;
  const bool jt2 = a.jump_table2 != 0;
  const WinLayout L = WinLayout::make(rc, n_pad, GS, INCF, ringN, 0, jt2);
  uint64_t* ring = reinterpret_cast<uint64_t*>(smem + L.ring);
  uint32_t* jm = reinterpret_cast<uint32_t*>(smem + L.jump);
  if (kp > 1)
    for (int i = threadIdx.x; i < (jt2 ? 2048 : 1024); i += blockDim.x)
      reinterpret_cast<uint64_t*>(jm)[i] = __ldg(a.jump + i);
  // window masks: a per-CTA shared-memory copy when it fits (plan), else global
  uint32_t* wm = reinterpret_cast<uint32_t*>(smem + L.masks);
  if (a.masks_smem)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      wm[i] = __ldg(a.win_pos + i);
      if (SIGNED) wm[n_pad + i] = __ldg(a.win_neg + i);
    }
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
    // ============================ producer ============================
    // kp lanes per replica stream (lane = l * kp + j): the stream is cut into
    // rounds of kp segments of SL draws, lane j generating segment j of every
    // round and then jumping (kp-1)*SL draws ahead to its segment of the next
    // round (Xoshiro::jump). A stream alone on one lane issues ~17 ALU
    // instructions per draw, one warp instruction every other cycle: ~36
    // cycles per draw, slower than a consumer visit; kp lanes side by side
    // cut that by ~kp (minus the jump, ~10 ALU instructions per matrix column
    // amortised over SL draws). Rounds cycle through the ring (index = draw
    // position mod the ring size) and are published whole; several rounds
    // buffered absorb the warp serving the replicas' rounds at different
    // times (a replica's round waits while others' are generated).
    const int round = kp * SL;
    const int l = lane / kp, j = lane % kp;
    const int r = blockIdx.x * rc + l;
    const bool act = l < rc && r < a.replicas;
    Xoshiro rng = Xoshiro::stream(act ? a.seeds[r] : 0ull, 1);  // anneal.cpp:191
    for (int i = 0; i < j * SL; i++) rng.step();                 // to this lane's first segment
    uint64_t* my = ring + (act ? l : 0) * ringN;
    const unsigned gp_s = saddr(genpos + (act ? l : 0)), cs_s = saddr(cons + (act ? l : 0));
    int gen = 0;  // draws published for this replica (whole rounds)
    long long idle = 0;  // consecutive polls without a round to generate (watchdog)
#pragma unroll 1
    for (;;) {
      // one consumer position per replica group (the group's lanes must agree)
      const int cpos = __shfl_sync(0xffffffffu, act ? ld_acquire(cs_s) : 0, lane - j);
      const bool can = act && gen + round <= cpos + ringN;
      if (can) {
        // 32-draw batches start at multiples of 32, so none straddles the
        // ring's end (rounds need not divide the ring)
#pragma unroll 1
        for (int b = 0; b < SL; b += 32) {
          uint64_t* dst = my + ((gen + j * SL + b) & rmask);
#pragma unroll
          for (int k = 0; k < 32; k++) dst[k] = rng.next();
        }
        if (kp > 1) {
          if (jt2)
            xoshiro_jump2(rng, jm);
          else
            rng.jump(jm);
        }
        gen += round;
        __threadfence_block();  // this lane's draws before the group's release
      }
      __syncwarp();
      if (can && j == 0) st_release(gp_s, gen);
      if (__any_sync(0xffffffffu, can)) {
        idle = 0;
      } else {
        // ring full: a short sleep keeps this warp's polling off the issue
        // slots the consumers need
        if (ld_acquire(done_s) >= rc || ld_acquire(abort_s)) break;
        __nanosleep(32);
        if (++idle > kWatchdog) {  // no consumer progress for ~2^28 polls
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
  using FT = typename std::conditional<INCF == 1, int8_t, int16_t>::type;  // exact field type
  FT* fld = reinterpret_cast<FT*>(smem + L.fields) + cw * n_pad;  // INCF only
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
      fld[v] = static_cast<FT>(acc);
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
  const uint64_t* myring = ring + cw * ringN;
  const unsigned gp_s = saddr(genpos + cw), cs_s = saddr(cons + cw);
  int gp = 0;
  int pub = 0;                    // last published consumer position (256-aligned)
  bool aborted = false;
  // loop invariants through a shuffle: kept in registers instead of being
  // re-read from the parameter bank on the step's dependency chain
  const int nn = __shfl_sync(FULL, n, 0);
  const int nsw = __shfl_sync(FULL, sweeps, 0);
  const bool msm = __shfl_sync(FULL, a.masks_smem, 0) != 0;
  // INCF deferred scatter: a spin change is scattered into the fields one step
  // later, off the step's critical path. The next step's window is the 32
  // vertices after the changed one, so its lanes add the change through the
  // changed vertex's forward masks instead (bit lane of fwd_pos/fwd_neg: the
  // vertex 1 + lane places ahead is a +1/-1 neighbour; one uniform load at the
  // event); the scatter itself is applied after that step's refill loads and
  // before the next ones. INCF requires rows of at most 128 entries (four
  // targets per lane).
  constexpr bool defer = INCF != 0;
  int sd = 0;                     // pending change (0 = none)
  int se0 = 0, se1 = 0;           // its CSR row
  uint32_t rmv = 0u, rmn = 0u;    // its forward window masks
  int sc[4] = {-1, -1, -1, -1}, sw[4] = {1, 1, 1, 1};
#if K1W_PROF
  const bool prof = (a.debug & 4) != 0 && a.prof != nullptr;  // GDI_PIPE_DEBUG=4: step statistics
  const bool nowait = (a.debug & 8) != 0;                     // timing experiment: ignore the ring
#else
  constexpr bool prof = false, nowait = false;
#endif
  unsigned long long p_steps = 0, p_acc = 0, p_fill = 0, p_wait = 0, p_t0 = prof ? clock64() : 0;

#pragma unroll 1
  while (sweep < nsw) {
    // refill the empty lanes [F, lim) of the window (vertex i0 + lane)
    const int lim = min(32, nn - i0);
    const long long p_a = prof ? clock64() : 0;
    const bool rl = lane >= F && lane < lim;
    int r_own = 0, r_f = 0;
    uint32_t r_wp = 0u, r_wn = 0u;
    if (rl) {  // loads into temporaries, then the refilled lanes take them
      const int v = i0 + lane;
      r_own = s[v];
      if (!INCF) {
        // one generic pointer for shared or global masks (measured faster than
        // selecting an explicit shared or global load per step)
        r_wp = (msm ? static_cast<const uint32_t*>(wm) : a.win_pos)[v];
        if (SIGNED) r_wn = (msm ? static_cast<const uint32_t*>(wm) + n_pad : a.win_neg)[v];
      }
      if (INCF) r_f = fld[v];
    }
    if (rl) {
      const int v = i0 + lane;
      own = r_own;
      wp = r_wp;
      wn = r_wn;
      f = 0;
      if (INCF) {
        f = r_f;
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
    }
    F = lim;
    if (defer && sd != 0) {
      // targets of the pending scatter (its row bounds were loaded at the event)
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int e = se0 + lane + 32 * q;
        sc[q] = e < se1 ? __ldg(col + e) : -1;
        if (SIGNED) sw[q] = e < se1 ? __ldg(wgt + e) : 0;
      }
      // the window misses the pending change in fld: add it through the changed
      // vertex's forward masks (loaded at the event)
      if ((rmv >> lane) & 1u) f += sd;
      if (SIGNED && ((rmn >> lane) & 1u)) f -= sd;
    }
    if (prof) p_fill += clock64() - p_a;
    // draws pos .. pos + F must be in the ring: read speculatively (they are
    // when the last acquired generator position covers them) and re-read
    // after waiting otherwise
    uint64_t d0 = 0, d1 = 0;
    if (K1W_SPEC) {
      d0 = myring[(pos + lane) & rmask];
      d1 = myring[(pos + lane + 1) & rmask];
    }
    const long long p_w = prof ? clock64() : 0;
    if (gp < pos + F + 1 && !nowait) {
      for (long long k = 0; (gp = ld_acquire(gp_s)) < pos + F + 1; k++)
        if (k > kWatchdog || ld_acquire(abort_s)) {
          aborted = true;
          break;
        }
      if (aborted) break;
      if (K1W_SPEC) {
        d0 = myring[(pos + lane) & rmask];
        d1 = myring[(pos + lane + 1) & rmask];
      }
    }
    if (!K1W_SPEC) {
      d0 = myring[(pos + lane) & rmask];
      d1 = myring[(pos + lane + 1) & rmask];
    }
    if (prof) p_wait += clock64() - p_w;
    const bool act = lane < F;
    const int diff = UNITAB ? AG - own - f : AG - a4 * own - bb * f;
    const bool tie = diff == 0;
    const int c = diff < 0 ? 1 : diff > 0 ? -1 : (static_cast<long long>(d0) < 0 ? 1 : -1);
    const uint64_t u = tie ? d1 : d0;
    const int fin = (en && u <= tm) ? -c : c;
    // the pending scatter is applied at the end of the step (its target loads,
    // issued above, come from L2)
    const int sdp = sd;
    if (defer) sd = 0;
    const unsigned m = __ballot_sync(FULL, act && (fin != own || tie));
    int adv;
    bool wrote = false;  // spin store this step (warp-uniform)
    if (m == 0u) {
      adv = F;
      pos += F;
    } else {
      const int js = __ffs(m) - 1;
      adv = js + 1;
      int fs, os, ts, fj;
      if (INCF) {  // |field| < 2^15: the event lane's values in one shuffle
        const int key = __shfl_sync(FULL, (f << 3) | (fin > 0 ? 4 : 0) | (own > 0 ? 2 : 0) | (tie ? 1 : 0), js);
        fs = (key & 4) ? 1 : -1;
        os = (key & 2) ? 1 : -1;
        ts = key & 1;
        fj = key >> 3;
      } else {
        const int key = __shfl_sync(FULL, (fin > 0 ? 4 : 0) | (own > 0 ? 2 : 0) | (tie ? 1 : 0), js);
        fs = (key & 4) ? 1 : -1;
        os = (key & 2) ? 1 : -1;
        ts = key & 1;
        fj = __shfl_sync(FULL, f, js);
      }
      pos += adv + ts;
      if (fs != os) {
        wrote = true;
        if (lane == js) s[i0 + js] = static_cast<int8_t>(fs);
        const int d = fs - os;
        AG += UNITAB ? d : a4 * d;
        dcut -= (d >> 1) * fj;
        if (defer) {
          const int v = i0 + js;  // row loads in flight until the next step
          se0 = __ldg(off + v);
          se1 = __ldg(off + v + 1);
          rmv = __ldg(a.fwd_pos + v);
          if (SIGNED) rmn = __ldg(a.fwd_neg + v);
          sd = d;
        } else {
          const int k = lane - js;  // pending lanes behind the event: field correction
          if (k >= 1) {
            if ((wp >> (k - 1)) & 1u) f += d;
            if (SIGNED && ((wn >> (k - 1)) & 1u)) f -= d;
          }
        }
      }
    }
    if (wrote) __syncwarp();  // this step's shared-memory stores before the next step's loads
    // ring slots before pos are consumed (release: their loads are done);
    // the producer works in whole rounds, so publishing every 256 draws is enough
    if ((pos & ~255) != pub) {
      if (lane == 0) st_release(cs_s, pos);
      pub = pos & ~255;
    }
    if (INCF) {  // spin and field of the pending lanes in one shuffle (decoded next step)
      const int pk = __shfl_down_sync(FULL, (f << 1) | (own > 0 ? 1 : 0), adv);
      own = (pk & 1) ? 1 : -1;
      f = pk >> 1;

    } else {
      own = __shfl_down_sync(FULL, own, adv);
      f = __shfl_down_sync(FULL, f, adv);
      wp = __shfl_down_sync(FULL, wp, adv);
      if (SIGNED) wn = __shfl_down_sync(FULL, wn, adv);
    }
    if (defer && sdp != 0) {  // the pending scatter (after this step's refill loads, before the next)
#pragma unroll
      for (int q = 0; q < 4; q++)
        if (sc[q] >= 0) fld[sc[q]] = static_cast<FT>(fld[sc[q]] + (SIGNED ? sw[q] * sdp : sdp));
      __syncwarp();
    }
    F -= adv;
    i0 += adv;
    if (prof) {
      p_steps++;
      p_acc += adv;
    }
    if (i0 == nn) {  // record_barrier (anneal.cpp:165-187)
      if (defer && sd != 0) {  // flush the pending scatter before the next sweep's refills
        for (int e = se0 + lane; e < se1; e += 32) {
          const int uu = __ldg(col + e);
          fld[uu] = static_cast<FT>(fld[uu] + (SIGNED ? __ldg(wgt + e) * sd : sd));
        }
        sd = 0;
        __syncwarp();
      }
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
      if (sweep < nsw) {
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
const void* win_fn(bool gs, int fb) {
  if (gs) return reinterpret_cast<const void*>(&k1_window<S, U, true, 0>);
  if (fb == 1) return reinterpret_cast<const void*>(&k1_window<S, U, false, 1>);
  if (fb == 2) return reinterpret_cast<const void*>(&k1_window<S, U, false, 2>);
  return reinterpret_cast<const void*>(&k1_window<S, U, false, 0>);
}

}  // namespace

int window_plan(const GraphStats& st, const PipeGraph& pg, int32_t replicas, int64_t a4, int64_t b, int32_t sweeps,
                PipePlan* plan) {
  if (!pg.ok) return -1;
  // draw positions are 32-bit: at most one visit + one tie coin per visit
  if (2.0 * static_cast<double>(sweeps) * st.n + 2 * kRingMax >= 2147483647.0) return -1;
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
  // producer lanes per replica stream: the largest power of two <= 32 / rc (<= 8)
  int kp = 1;
  while (kp < 8 && 2 * kp * rc <= 32) kp *= 2;
  if (const char* e = std::getenv("GDI_WINDOW_KP")) kp = std::atoi(e);  // tuning experiments
  const int nr = 4;  // (minimum ring for the layout checks: nr * kp * 32 draws)
  const char* ring_env = std::getenv("GDI_WINDOW_RING");  // tuning: ring size (power of two)
  const int cap = 227 * 1024, ring_min = nr * kp * 32;  // sm_100 dynamic shared memory per CTA
  const bool gs = WinLayout::make(rc, n_pad, false, false, ring_min).total > cap ||
                  (force && std::string(force) == "window_gmem");
  // incremental fields when they fit next to the spins (int16 bound)
  const bool incf = !gs && st.max_abs_field < 32768 && st.max_degree <= 128 &&
                    WinLayout::make(rc, n_pad, false, st.max_abs_field <= 127 ? 1 : 2, ring_min).total <= cap &&
                    !(force && std::string(force) == "window_masks");
  // shared-memory budget after the spins: segment length (the longest that
  // fits amortises the jump over more draws), window masks (the INCF variant
  // reads only the forward masks, once per event), the two-column jump table
  const int mw = st.unit ? 1 : 2;
  struct Fit {
    int segl;
    bool msm, jt2;
    int ring;
  };
  auto fit = [&](int fb) {
    Fit f{32, false, false, 256};
    // the largest power-of-two ring that fits; segments as long as a round of
    // kp segments stays within 3/8 of the ring (more than two rounds buffered:
    // 192 draws for kp = 4 in 2048, measured best of 128..256)
    for (int rn : {2048, 1024, 512, 256})
      if (WinLayout::make(rc, n_pad, gs, fb, rn).total <= cap) {
        f.ring = rn;
        break;
      }
    f.segl = (f.ring * 3 / 8 / kp) / 32 * 32;
    f.segl = f.segl < 32 ? 32 : f.segl > 256 ? 256 : f.segl;
    if (const char* e = std::getenv("GDI_WINDOW_SEGL")) f.segl = std::atoi(e);
    if (ring_env) f.ring = std::atoi(ring_env);
    const int rn = f.ring;
    f.msm = fb == 0 && WinLayout::make(rc, n_pad, gs, fb, rn, mw).total <= cap;
    f.jt2 = kp > 1 && WinLayout::make(rc, n_pad, gs, fb, rn, f.msm ? mw : 0, true).total <= cap;
    return f;
  };
  // exact field type: int16, or int8 (|field| <= 127) when that frees room for a
  // longer segment or the jump table (int8 fields were measured slower on their own)
  int fb = incf ? 2 : 0;
  Fit ft = fit(fb);
  if (incf && st.max_abs_field <= 127) {
    const Fit f8 = fit(1);
    if (f8.ring > ft.ring || f8.segl > ft.segl || (f8.jt2 && !ft.jt2)) {
      fb = 1;
      ft = f8;
    }
  }
  const int segl = ft.segl;
  const bool msm = ft.msm;
  bool jt2 = ft.jt2;
  if (const char* e = std::getenv("GDI_WINDOW_JT2")) jt2 = kp > 1 && std::atoi(e) != 0;
  plan->jt2 = jt2;
  plan->kp = kp;
  plan->segl = segl;
  plan->masks_smem = msm;
  plan->rounds = nr;
  plan->ring_n = ft.ring;
  const bool unitab = ra == 1 && rb == 1;
  plan->fn = st.unit ? (unitab ? win_fn<false, true>(gs, fb) : win_fn<false, false>(gs, fb))
                     : (unitab ? win_fn<true, true>(gs, fb) : win_fn<true, false>(gs, fb));
  plan->prof = false;
  plan->gw = gs;
  plan->rc = rc;
  // one producer warp, kp lanes per stream (see the kernel)
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
  plan->smem = WinLayout::make(rc, n_pad, gs, fb, plan->ring_n, msm ? mw : 0, jt2).total;
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
  cudaError_t err = allow_max_smem(plan.fn);
  if (err != cudaSuccess) return err;
  PipeArgs a = args;
  a.rc = plan.rc;
  a.a4 = plan.a4;
  a.b = plan.b;
  a.n_words = plan.n_words;
  a.nprod = plan.nprod;
  a.rolemap = plan.rolemap;
  a.kp = plan.kp;
  a.segl = plan.segl;
  a.rounds = plan.rounds;
  a.ring_n = plan.ring_n;
  a.masks_smem = plan.masks_smem ? 1 : 0;
  a.jump_table2 = plan.jt2 ? 1 : 0;
  a.jump = nullptr;
  if (plan.kp > 1) {
    // the (kp-1)*segl-draw jump matrix, built once per device and distance
    static std::mutex mu;
    static std::map<std::pair<int, int>, uint64_t*> cache;
    int dev = 0;
    if ((err = cudaGetDevice(&dev)) != cudaSuccess) return err;
    const int J = (plan.kp - 1) * plan.segl;
    std::lock_guard<std::mutex> lock(mu);
    uint64_t*& d = cache[{dev, plan.jt2 ? -J : J}];
    if (d == nullptr) {
      std::vector<uint64_t> h(256 * 4);
      xoshiro_jump_matrix(static_cast<uint64_t>(J), h.data());
      if (plan.jt2) {
        std::vector<uint64_t> t(128 * 4 * 4);
        xoshiro_jump_table2(h.data(), t.data());
        h.swap(t);
      }
      if ((err = cudaMalloc(&d, h.size() * sizeof(uint64_t))) != cudaSuccess) {
        d = nullptr;
        return err;
      }
      if ((err = cudaMemcpy(d, h.data(), h.size() * sizeof(uint64_t), cudaMemcpyHostToDevice)) != cudaSuccess)
        return err;
    }
    a.jump = d;
  }
  const char* dbg = std::getenv("GDI_PIPE_DEBUG");
  a.debug = dbg ? std::atoi(dbg) : 0;
  void* params[] = {&a};
  return cudaLaunchKernel(plan.fn, dim3(plan.grid), dim3(plan.block), params, plan.smem, stream);
}

}  // namespace gdi
