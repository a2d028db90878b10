// K1 v4 — bit-exact GDI sweep: aligned 32-vertex windows resolved to a fixed
// point, per-warp xoshiro generation (sm_100a).
//
// Contract: bit-identical to the reference's single-worker anneal
// (proj/src/anneal.cpp:132-231; visit_node :86-128; init :148-155;
// record_barrier :165-187; Rng rng.hpp:10-65), like k1_window.cu.
//
// One warp per replica. A sweep is cut into aligned windows of 32 vertices
// (lane j = vertex i0 + j). Visit j depends on the visits before it through
//   * the counter:   G_j = G + sum_{k<j} d_k              (d_k = new - old spin)
//   * its field:     f_j = f + sum_{k<j, k~j} w_kj d_k    (in-window neighbours)
//   * its draws:     position pos + j + T_j, T_j = ties among lanes k < j
// and those inputs depend only on the lanes before it, so the window is a
// triangular system: evaluate every lane from the current guess of its
// predecessors' outputs (d_k, tie_k), rebuild the inputs from the new outputs
// (ballot + popc prefixes; the field term from the in-window neighbour masks
// against the bit-reversed change ballots), repeat until no output changes.
// After t rounds lanes 0..t-1 are final, so it ends in at most 33 rounds; in
// practice (#events in the window) + 1 rounds: one round for the ~98% of
// windows late in an anneal that have no event. The fixed point is exactly
// the sequential outcome (unique solution of the triangular system), and the
// whole window is accepted: every window step advances 32 visits.
//
// State on chip per replica: spins as one bit per vertex (a window's spins
// are one 32-bit word, rewritten by one ballot), exact fields as biased
// bytes (or halves) packed in 32-bit words so that a spin change scatters
// +-2 into its neighbours' fields with shared-memory atomicAdd on the word
// (the bias keeps every lane of the word in range: no carry or borrow
// crosses into a neighbour byte because |field| <= max degree < bias).
// Per CTA (shared by its replicas): the CSR as 16-bit columns (bit 15 =
// weight -1), row offsets, in-window neighbour masks, the jump table.
//
// Draws: the warp generates its own replica's xoshiro256++ stream 1 in
// rounds of 32 segments x kL draws (lane j = segment j), then every lane
// jumps 31*kL draws ahead with a 4-bit precombined GF(2) jump table
// (xoshiro_jump4). The round sits in a per-replica ring after a 64-draw tail
// copied from the end of the previous round, so the draws still ahead of the
// consumer stay addressable at consecutive positions; segments are padded to
// kL + 1 entries so the generating lanes' stores hit distinct banks. No
// producer warp, no inter-warp synchronisation after the prologue.
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "device_rng.cuh"
#include "kernels.cuh"
#include "launch.hpp"

namespace gdi {

namespace {

constexpr int kL = 32;                               // draws per lane segment
constexpr int kRound = 32 * kL;                      // draws per generation round
constexpr int kTail = 66;                            // entries before the round (64 draws + gap)
constexpr int kRingElems = kTail + 32 * (kL + 1);    // 1122 x 8 B per replica
constexpr int kJump = 31 * kL;                       // lane jump distance per round

// ring index of draw li (relative to the round start; -64 <= li < kRound):
// segment padding for round entries, the same formula places the tail at
// kTail-66 .. kTail-2 (li >> 5 is -2 / -1 there)
__device__ __forceinline__ int ring_phys(int li) { return kTail + li + (li >> 5); }

struct BlkLayout {
  int jt, maskp, maskn, off, col, rep, rep_bytes, ring, words, fields, total;
  // rows > 0: the graph stays in global memory (row records, jump table), only
  // the replicas' state is in shared memory
  __host__ __device__ static BlkLayout make(int n, int nnz, int rc, int fb, bool sgn, int rows = 0) {
    BlkLayout L;
    L.jt = 0;                                   // 64 x 4 x 16 uint2 = 32 KB
    L.maskp = L.jt + (rows ? 0 : 64 * 4 * 16 * 8);
    L.maskn = L.maskp + (rows ? 0 : n * 4);
    L.off = L.maskn + (sgn && !rows ? n * 4 : 0);
    L.col = L.off + (rows ? 0 : (n + 1) * 4);
    L.rep = (L.col + (rows ? 0 : nnz * 2) + 15) & ~15;
    const int nw = (n + 31) / 32;
    L.ring = 0;
    L.words = kRingElems * 8;
    L.fields = L.words + nw * 4;
    const int fbytes = ((n * fb + 3) & ~3);
    L.rep_bytes = (L.fields + fbytes + 15) & ~15;
    L.total = L.rep + rc * L.rep_bytes;
    return L;
  }
};

struct BlockArgs {
  DevCsr g;
  const uint4* brow;  // ROWS: per vertex {maskp, maskn, cols 0-1, cols 2-3} (build_block_rows)
  int32_t lane_rows;  // rows short enough for a lane to walk its own (max degree <= 16)
  int32_t nnz;
  int32_t sweeps, replicas, rc;
  const uint64_t* seeds;
  const long long* thr;
  const unsigned long long* tmask;
  int32_t a4, b;
  const uint2* jump;  // xoshiro_jump4 table for kJump draws
  int8_t* spins_out;
  DevTrace* trace;
  unsigned long long* stamps;
  int8_t* snaps;
  DevTrace* final_out;
};

// xoshiro256++ jump with the matrix precombined four columns at a time:
// tab[(g * 4 + q) * 16 + v] = 64-bit word q of the XOR of the columns 4g+b
// for the bits b of v. A lane's four loads of group g hit one 128-byte row
// (16 entries x 8 B): conflict-free whatever the lanes' nibbles.
__device__ __forceinline__ void xoshiro_jump4(Xoshiro& r, const uint2* tab) {
  uint32_t o0 = 0, o1 = 0, o2 = 0, o3 = 0, o4 = 0, o5 = 0, o6 = 0, o7 = 0;
  const uint32_t w[8] = {static_cast<uint32_t>(r.s0), static_cast<uint32_t>(r.s0 >> 32),
                         static_cast<uint32_t>(r.s1), static_cast<uint32_t>(r.s1 >> 32),
                         static_cast<uint32_t>(r.s2), static_cast<uint32_t>(r.s2 >> 32),
                         static_cast<uint32_t>(r.s3), static_cast<uint32_t>(r.s3 >> 32)};
#pragma unroll
  for (int h = 0; h < 8; h++) {
    uint32_t x = w[h];
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const uint2* e = tab + (h * 8 + i) * 64 + (x & 15u);
      x >>= 4;
      const uint2 p0 = e[0], p1 = e[16], p2 = e[32], p3 = e[48];
      o0 ^= p0.x;
      o1 ^= p0.y;
      o2 ^= p1.x;
      o3 ^= p1.y;
      o4 ^= p2.x;
      o5 ^= p2.y;
      o6 ^= p3.x;
      o7 ^= p3.y;
    }
  }
  r.s0 = o0 | (static_cast<uint64_t>(o1) << 32);
  r.s1 = o2 | (static_cast<uint64_t>(o3) << 32);
  r.s2 = o4 | (static_cast<uint64_t>(o5) << 32);
  r.s3 = o6 | (static_cast<uint64_t>(o7) << 32);
}

template <int FB>
__device__ __forceinline__ int field_at(const unsigned char* fld, int v) {
  if (FB == 1) return static_cast<int>(fld[v]) - 128;
  return static_cast<int>(reinterpret_cast<const uint16_t*>(fld)[v]) - 32768;
}

// add dv to the biased field of vertex t (word-wide atomic, see the header)
template <int FB>
__device__ __forceinline__ void field_add(unsigned char* fld, int t, int dv) {
  unsigned* w = reinterpret_cast<unsigned*>(fld);
  if (FB == 1)
    atomicAdd(w + (t >> 2), static_cast<unsigned>(dv) << ((t & 3) * 8));
  else
    atomicAdd(w + (t >> 1), static_cast<unsigned>(dv) << ((t & 1) * 16));
}

// ROWS (= 4): graphs whose CSR and window masks do not fit shared memory
// next to the replicas (G81+-1: 20000 vertices), with max degree <= 4: each
// vertex's window masks and its (<= 4) 16-bit columns form one 16-byte row
// record in global memory, loaded two windows ahead into registers; every
// changed lane scatters its own record's columns (all changes of a window at
// once); the jump table is read through L1.
template <bool SIGNED, bool UNITAB, int FB, int ROWS>
__global__ void __launch_bounds__(512, 1) k1_block(const BlockArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.g.n, nnz = a.nnz;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const BlkLayout L = BlkLayout::make(n, nnz, a.rc, FB, SIGNED, ROWS);
  uint2* jt = ROWS ? const_cast<uint2*>(a.jump) : reinterpret_cast<uint2*>(smem + L.jt);
  uint32_t* maskp = reinterpret_cast<uint32_t*>(smem + L.maskp);
  uint32_t* maskn = reinterpret_cast<uint32_t*>(smem + L.maskn);
  int32_t* offs = reinterpret_cast<int32_t*>(smem + L.off);
  uint16_t* cols = reinterpret_cast<uint16_t*>(smem + L.col);
  const unsigned FULL = 0xffffffffu;

  // ---- prologue (whole CTA): jump table, CSR, in-window masks ----
  if (!ROWS) {
  for (int i = threadIdx.x; i < 64 * 4 * 16; i += blockDim.x) jt[i] = __ldg(a.jump + i);
  for (int i = threadIdx.x; i <= n; i += blockDim.x) offs[i] = __ldg(a.g.off + i);
  for (int e = threadIdx.x; e < nnz; e += blockDim.x) {
    const int c = __ldg(a.g.col + e);
    cols[e] = static_cast<uint16_t>(SIGNED && __ldg(a.g.w + e) < 0 ? (c | 0x8000) : c);
  }
  // bit k-1 of maskp[v] (maskn[v]): vertex v-k is a +1 (-1) neighbour in v's
  // own window (k <= v mod 32)
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    uint32_t mp = 0u, mn = 0u;
    const int lo = v & ~31, e1 = __ldg(a.g.off + v + 1);
    for (int e = __ldg(a.g.off + v); e < e1; e++) {
      const int u = __ldg(a.g.col + e);
      if (u < v && u >= lo) {
        if (SIGNED && __ldg(a.g.w + e) < 0)
          mn |= 1u << (v - u - 1);
        else
          mp |= 1u << (v - u - 1);
      }
    }
    maskp[v] = mp;
    if (SIGNED) maskn[v] = mn;
  }
  }
  __syncthreads();

  const int r = blockIdx.x * a.rc + warp;
  if (warp >= a.rc || r >= a.replicas) return;  // no block-wide sync below
  const size_t rs = static_cast<size_t>(r);
  unsigned char* rep = smem + L.rep + warp * L.rep_bytes;
  uint64_t* ring = reinterpret_cast<uint64_t*>(rep + L.ring);
  uint32_t* words = reinterpret_cast<uint32_t*>(rep + L.words);
  unsigned char* fld = rep + L.fields;
  const int nw = (n + 31) / 32;
  const int sweeps = a.sweeps;
  const uint64_t seed = a.seeds[r];

  // ---- init (anneal.cpp:148-155): the serial stream-0 coins, one bit per vertex
  int G = 0;
  {
    Xoshiro r0 = Xoshiro::stream(seed, 0);
    for (int w = 0; w < nw; w++) {
      bool mine = false;
      const int lim = min(32, n - w * 32);
#pragma unroll 4
      for (int l = 0; l < lim; l++) {
        const bool up = (r0.next() >> 63) != 0;
        G += up ? 1 : -1;
        mine = l == lane ? up : mine;
      }
      const unsigned word = __ballot_sync(FULL, mine);
      if (lane == 0) words[w] = word;
    }
  }
  __syncwarp();
  auto spin = [&](int v) { return ((words[v >> 5] >> (v & 31)) & 1u) ? 1 : -1; };
  // exact initial cut (evaluate.cpp:10-18) and fields
  long long cut = 0;
  for (int u = lane; u < n; u += 32) {
    const int su = spin(u);
    int acc = 0;
    auto entry = [&](int c) {
      const int v = SIGNED ? (c & 0x7fff) : c;
      const int wt = SIGNED && (c & 0x8000) ? -1 : 1;
      const int sv = spin(v);
      acc += wt * sv;
      if (v > u && sv != su) cut += wt;
    };
    if (ROWS) {
      const uint4 rr = __ldg(a.brow + u);
      const unsigned cw[2] = {rr.z, rr.w};
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const unsigned c = (cw[k >> 1] >> (16 * (k & 1))) & 0xffffu;
        if (c != 0xffffu) entry(static_cast<int>(c));
      }
    } else {
      for (int e = offs[u]; e < offs[u + 1]; e++) entry(cols[e]);
    }
    if (FB == 1)
      fld[u] = static_cast<unsigned char>(acc + 128);
    else
      reinterpret_cast<uint16_t*>(fld)[u] = static_cast<uint16_t>(acc + 32768);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cut += __shfl_xor_sync(FULL, cut, o);
  __syncwarp();
  if (a.snaps != nullptr)
    for (int i = lane; i < n; i += 32) a.snaps[rs * (sweeps + 1) * n + i] = static_cast<int8_t>(spin(i));
  if (lane == 0 && a.stamps != nullptr) a.stamps[rs * (sweeps + 1)] = globaltimer_ns();

  // ---- draws: stream 1 (anneal.cpp:191), lane j = segment j of each round
  Xoshiro rng = Xoshiro::stream(seed, 1);
  for (int i = 0; i < lane * kL; i++) rng.step();
  int pos = 0, rbase = -kRound, gend = 0;  // absolute draw positions

  const int a4 = a.a4, bb = a.b;
  int AG = UNITAB ? G : a4 * G;
  long long cutv = cut;
  int dcut = 0;  // this lane's share of the sweep's cut change
  const unsigned lt = (1u << lane) - 1u;
  const int nn = __shfl_sync(FULL, n, 0);
  const int nsw = __shfl_sync(FULL, sweeps, 0);
  // ROWS: row records of the current window and the next (loaded two
  // windows ahead; the windows repeat sweep after sweep)
  const int nwin32 = ((nn + 31) >> 5) << 5;
  auto ldrow = [&](int w0) -> uint4 {
    const int vv = w0 + lane;
    return vv < nn ? __ldg(a.brow + vv) : make_uint4(0u, 0u, 0xffffffffu, 0xffffffffu);
  };
#ifndef K1_ROWS_AHEAD
#define K1_ROWS_AHEAD 2
#endif
  uint4 rw0 = make_uint4(0u, 0u, 0u, 0u), rw1 = rw0, rw2 = rw0;
  if (ROWS) {
    rw0 = ldrow(0);
    rw1 = ldrow(32 % nwin32);
    if (K1_ROWS_AHEAD > 2) rw2 = ldrow(64 % nwin32);
  }

#pragma unroll 1
  for (int sweep = 0; sweep < nsw; sweep++) {
    const unsigned long long tm = a.tmask[sweep];
    const bool en = a.thr[sweep] >= 0;
#pragma unroll 1
    for (int i0 = 0; i0 < nn; i0 += 32) {
      if (gend - pos < 64) {
        // next round: keep the last 64 draws (all still ahead of pos) in the
        // tail, then every lane writes its segment and jumps
        const uint64_t t0 = ring[ring_phys(kRound - 64 + lane)], t1 = ring[ring_phys(kRound - 32 + lane)];
        __syncwarp();
        ring[ring_phys(lane - 64)] = t0;
        ring[ring_phys(lane - 32)] = t1;
        uint64_t* seg = ring + kTail + lane * (kL + 1);
#pragma unroll 8
        for (int k = 0; k < kL; k++) seg[k] = rng.next();
        xoshiro_jump4(rng, jt);
        rbase += kRound;
        gend += kRound;
        __syncwarp();
      }
      const int v = i0 + lane;
      const bool act = v < nn;
      const unsigned word = words[i0 >> 5];
      const int own = ((word >> lane) & 1u) ? 1 : -1;
      int f0 = 0;
      uint32_t wp = 0u, wn = 0u;
      uint4 rcur = rw0;
      if (ROWS) {
        rw0 = rw1;
        int wa = i0 + 32 * K1_ROWS_AHEAD;  // (the window K1_ROWS_AHEAD ahead, cyclically; no division)
        if (wa >= nwin32) wa -= nwin32;
        if (wa >= nwin32) wa -= nwin32;
        if (K1_ROWS_AHEAD > 2) {
          rw1 = rw2;
          rw2 = ldrow(wa);
        } else {
          rw1 = ldrow(wa);
        }
        wp = rcur.x;
        if (SIGNED) wn = rcur.y;
        if (act) f0 = field_at<FB>(fld, v);
      } else if (act) {
        f0 = field_at<FB>(fld, v);
        wp = maskp[v];
        if (SIGNED) wn = maskn[v];
      }
      const int lb = pos - rbase + lane;
      uint64_t d0 = ring[ring_phys(lb)], d1 = ring[ring_phys(lb + 1)];
      unsigned U = 0u, D = 0u, Tm = 0u;
      int T = 0, fin = own, f = f0;
#pragma unroll 1
      for (int it = 0; it < 40; it++) {
        int ag = AG, ff = f0;
        if (it > 0) {
          const int dg = __popc(U & lt) - __popc(D & lt);
          ag += UNITAB ? 2 * dg : 2 * a4 * dg;
          const unsigned sh = 32u - lane;
          const unsigned xu = __funnelshift_rc(__brev(U), 0u, sh), xd = __funnelshift_rc(__brev(D), 0u, sh);
          int df = __popc(wp & xu) - __popc(wp & xd);
          if (SIGNED) df -= __popc(wn & xu) - __popc(wn & xd);
          ff += 2 * df;
          const int Tn = __popc(Tm & lt);
          if (Tn != T) {
            T = Tn;
            d0 = ring[ring_phys(lb + T)];
            d1 = ring[ring_phys(lb + T + 1)];
          }
        }
        const int diff = UNITAB ? ag - own - ff : ag - a4 * own - bb * ff;
        const bool tie = diff == 0;
        const int c = diff < 0 ? 1 : diff > 0 ? -1 : (static_cast<long long>(d0) < 0 ? 1 : -1);
        const uint64_t u = tie ? d1 : d0;
        fin = (en && u <= tm) ? -c : c;
        f = ff;
        const unsigned nU = __ballot_sync(FULL, act && fin > own);
        const unsigned nD = __ballot_sync(FULL, act && fin < own);
        const unsigned nT = __ballot_sync(FULL, act && tie);
        const bool same = nU == U && nD == D && nT == Tm;
        U = nU;
        D = nD;
        Tm = nT;
        if (same) break;
      }
      pos += min(32, nn - i0) + __popc(Tm);
      if (U | D) {
        // commit: the window's spin word, the counter, the exact cut change
        // -(d/2) * field, and the scatter of every change into its
        // neighbours' fields (before the next window loads them)
        const unsigned nwd = __ballot_sync(FULL, act && fin > 0);
        if (lane == 0) words[i0 >> 5] = nwd;
        AG += (UNITAB ? 2 : 2 * a4) * (__popc(U) - __popc(D));
        if (act && fin != own) dcut += fin > own ? -f : f;
        if (ROWS) {
          // every changed lane scatters its own record's (<= 4) columns,
          // all changed lanes at once (shared-memory atomics on the packed
          // fields; no shuffles)
          if (act && fin != own) {
            const int dv = fin > own ? 2 : -2;
#pragma unroll
            for (int k = 0; k < 4; k++) {
              const unsigned c = ((k < 2 ? rcur.z : rcur.w) >> (16 * (k & 1))) & 0xffffu;
              if (c != 0xffffu) {
                if (SIGNED)
                  field_add<FB>(fld, static_cast<int>(c & 0x7fffu), (c & 0x8000u) ? -dv : dv);
                else
                  field_add<FB>(fld, static_cast<int>(c), dv);
              }
            }
          }
          __syncwarp();
          continue;
        }
        // row bounds of every changed lane in one round trip, then one pass
        // per change with the lanes over its row (rows of <= 64 entries in
        // two predicated steps)
        int r0 = 0, r1 = 0;
        if (act && fin != own) {
          r0 = offs[v];
          r1 = offs[v + 1];
        }
        auto scat = [&](int e, int dv) {
          const int cc = cols[e];
          if (SIGNED)
            field_add<FB>(fld, cc & 0x7fff, (cc & 0x8000) ? -dv : dv);
          else
            field_add<FB>(fld, cc, dv);
        };
        unsigned C = U | D;
        // two or more changes and short rows (max degree <= 16): every changed
        // lane walks its own row, all at once (G55: 70.6 -> 66.7 ms; with the
        // long rows of G22 / G1 (max degree ~35 / ~70) the lane walks were
        // slower than the row-parallel passes below)
        if (a.lane_rows && __popc(C) >= 2) {
          if (act && fin != own) {
            const int dv = fin > own ? 2 : -2;
#pragma unroll 1
            for (int e = r0; e < r1; e++) scat(e, dv);
          }
          C = 0u;
        }
        if (C)
#pragma unroll 1
        do {
          const int cl = __ffs(C) - 1;
          C &= C - 1u;
          const int b0 = __shfl_sync(FULL, r0, cl) + lane, b1 = __shfl_sync(FULL, r1, cl);
          const int dv = ((U >> cl) & 1u) ? 2 : -2;
          if (b0 < b1) scat(b0, dv);
          if (b0 + 32 < b1) scat(b0 + 32, dv);
#pragma unroll 1
          for (int e = b0 + 64; e < b1; e += 32) scat(e, dv);
        } while (C);
        __syncwarp();
      }
    }
    // record_barrier (anneal.cpp:165-187)
    int dsum = dcut;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(FULL, dsum, o);
    cutv += dsum;
    dcut = 0;
    const int Gs = UNITAB ? AG : AG / a4;
    if (lane == 0) {
      if (a.trace != nullptr) a.trace[rs * sweeps + sweep] = DevTrace{cutv, Gs, Gs};
      if (a.stamps != nullptr) a.stamps[rs * (sweeps + 1) + sweep + 1] = globaltimer_ns();
    }
    if (a.snaps != nullptr)
      for (int i = lane; i < n; i += 32)
        a.snaps[(rs * (sweeps + 1) + sweep + 1) * n + i] = static_cast<int8_t>(spin(i));
  }
  const int Gf = UNITAB ? AG : AG / a4;
  if (lane == 0) a.final_out[rs] = DevTrace{cutv, Gf, Gf};
  for (int i = lane; i < n; i += 32) a.spins_out[rs * n + i] = static_cast<int8_t>(spin(i));
}

template <bool S, bool U>
const void* blk_fn(int fb, int rows) {
  if (rows)
    return fb == 1 ? reinterpret_cast<const void*>(&k1_block<S, U, 1, 4>)
                   : reinterpret_cast<const void*>(&k1_block<S, U, 2, 4>);
  return fb == 1 ? reinterpret_cast<const void*>(&k1_block<S, U, 1, 0>)
                 : reinterpret_cast<const void*>(&k1_block<S, U, 2, 0>);
}

}  // namespace

// Host: the 4-bit table for xoshiro_jump4 from a jump matrix (256 x 4 uint64
// columns) -> 64 groups x 4 words x 16 values of uint64.
void xoshiro_jump_table4(const uint64_t* mat, uint64_t* tab) {
  for (int g = 0; g < 64; g++)
    for (int v = 0; v < 16; v++)
      for (int q = 0; q < 4; q++) {
        uint64_t x = 0;
        for (int b = 0; b < 4; b++)
          if (v & (1 << b)) x ^= mat[(4 * g + b) * 4 + q];
        tab[(g * 4 + q) * 16 + v] = x;
      }
}

int block_plan(const GraphStats& st, int32_t replicas, int64_t a4, int64_t b, int32_t sweeps, BlockPlan* plan) {
  // |w| == 1 only (in-window masks and the sign bit of the 16-bit columns)
  if (!st.unit && !st.pm1) return -1;
  const bool sgn = !st.unit;
  if (st.n < 1 || st.n > (sgn ? 32767 : 65535)) return -1;
  if (2.0 * static_cast<double>(sweeps) * st.n + 4.0 * kRound >= 2147483647.0) return -1;  // 32-bit positions
  long long x = a4 < 0 ? -a4 : a4, y = b < 0 ? -b : b;
  while (y) {
    const long long t = x % y;
    x = y;
    y = t;
  }
  const long long ra = a4 / x, rb = b / x;
  const double bound = static_cast<double>(ra) * (2.0 * st.n + 3) + static_cast<double>(rb) * (st.max_abs_field + 66);
  if (bound >= 2147483647.0) return -1;
  int fb = st.max_abs_field <= 127 ? 1 : st.max_abs_field <= 32767 ? 2 : 0;
  if (fb == 0) return -1;
  const int nnz = static_cast<int>(2 * st.m);
  int rc = (replicas + 147) / 148;
  rc = rc < 1 ? 1 : rc > 16 ? 16 : rc;
  const int cap = 227 * 1024;
  // the CSR and window masks in shared memory next to the replicas, else
  // (degree <= 4) row records in global memory (ROWS). With more replicas
  // than fit one wave (R > 148 x the replicas a CTA holds), fewer replicas
  // per CTA and several waves rather than the global-memory kernels (4096
  // replicas x 1000 sweeps: G55 412 -> 265 ms, G81+-1 3033 -> 1099 ms, G1 58
  // -> 34 ms)
  int rows = 0;
  while (rc > 1 && BlkLayout::make(st.n, nnz, rc, fb, sgn).total > cap &&
         !(st.max_degree <= 4 && BlkLayout::make(st.n, nnz, rc, fb, sgn, 4).total <= cap))
    rc--;
  if (BlkLayout::make(st.n, nnz, rc, fb, sgn).total > cap) {
    if (st.max_degree > 4 || BlkLayout::make(st.n, nnz, rc, fb, sgn, 4).total > cap) return -1;
    rows = 4;
  }
  if (const char* e = std::getenv("GDI_BLOCK_ROWS"))  // tests: force the row-record variant
    if (std::atoi(e) != 0 && st.max_degree <= 4 && BlkLayout::make(st.n, nnz, rc, fb, sgn, 4).total <= cap) rows = 4;
  const bool unitab = ra == 1 && rb == 1;
  plan->fn = sgn ? (unitab ? blk_fn<true, true>(fb, rows) : blk_fn<true, false>(fb, rows))
                 : (unitab ? blk_fn<false, true>(fb, rows) : blk_fn<false, false>(fb, rows));
  plan->rows = rows;
  int lane_maxdeg = 16;
  if (const char* e = std::getenv("GDI_K1_LANE_MAXDEG")) lane_maxdeg = std::atoi(e);  // A/B
  plan->lane_rows = st.max_degree <= lane_maxdeg;
  plan->rc = rc;
  plan->block = 32 * rc;
  plan->grid = (replicas + rc - 1) / rc;
  plan->smem = BlkLayout::make(st.n, nnz, rc, fb, sgn, rows).total;
  plan->a4 = static_cast<int32_t>(ra);
  plan->b = static_cast<int32_t>(rb);
  plan->nnz = nnz;
  static const char* names[2][2][2] = {{{"k1_block<signed>", "k1_block<signed,ab=1>"},
                                        {"k1_block<unit>", "k1_block<unit,ab=1>"}},
                                       {{"k1_block<signed,rows>", "k1_block<signed,ab=1,rows>"},
                                        {"k1_block<unit,rows>", "k1_block<unit,ab=1,rows>"}}};
  plan->name = names[rows ? 1 : 0][sgn ? 0 : 1][unitab ? 1 : 0];
  return 0;
}

cudaError_t block_launch(const BlockPlan& plan, const ExactArgs& ex, cudaStream_t stream) {
  cudaError_t err = allow_max_smem(plan.fn);
  if (err != cudaSuccess) return err;
  BlockArgs a{};
  a.g = ex.g;
  a.brow = ex.brow;
  a.lane_rows = plan.lane_rows;
  if (plan.rows && a.brow == nullptr) return cudaErrorInvalidValue;  // (ensure_brow first)
  a.nnz = plan.nnz;
  a.sweeps = ex.sweeps;
  a.replicas = ex.replicas;
  a.rc = plan.rc;
  a.seeds = ex.seeds;
  a.thr = ex.thr;
  a.tmask = ex.tmask;
  a.a4 = plan.a4;
  a.b = plan.b;
  a.spins_out = ex.spins_out;
  a.trace = ex.trace;
  a.stamps = ex.stamps;
  a.snaps = ex.snaps;
  a.final_out = ex.final_out;
  {
    // the kJump-draw 4-bit jump table, built once per device
    static std::mutex mu;
    static std::map<int, uint2*> cache;
    int dev = 0;
    if ((err = cudaGetDevice(&dev)) != cudaSuccess) return err;
    std::lock_guard<std::mutex> lock(mu);
    uint2*& d = cache[dev];
    if (d == nullptr) {
      std::vector<uint64_t> m(256 * 4), t(64 * 4 * 16);
      xoshiro_jump_matrix(static_cast<uint64_t>(kJump), m.data());
      xoshiro_jump_table4(m.data(), t.data());
      if ((err = cudaMalloc(&d, t.size() * sizeof(uint64_t))) != cudaSuccess) {
        d = nullptr;
        return err;
      }
      if ((err = cudaMemcpy(d, t.data(), t.size() * sizeof(uint64_t), cudaMemcpyHostToDevice)) != cudaSuccess)
        return err;
    }
    a.jump = d;
  }
  void* params[] = {&a};
  return cudaLaunchKernel(plan.fn, dim3(plan.grid), dim3(plan.block), params, plan.smem, stream);
}

}  // namespace gdi
