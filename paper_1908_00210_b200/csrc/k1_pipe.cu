// K1 v2 — bit-exact GDI sweep, warp-specialised pipeline (sm_100a).
//
// Same contract as k1_exact.cu (bit-identical to the reference's
// single-worker anneal, reference proj/src/anneal.cpp:132-231), restructured
// so the serial per-replica chain carries only ALU work:
//
//  * lane = replica. A CTA owns RC <= 32 replicas; their spins of vertex v
//    are one 32-bit word words[v] (bit l = replica l is +1) in shared memory,
//    written by the decider with one __ballot_sync per visit.
//  * gatherer warps (1..NG) run ahead of the decider. For global visit
//    U = sweep*n + i they compute, for all lanes at once, the neighbour field
//    of vertex i EXCLUDING the L=32 vertices visited immediately before U
//    ((i-1)..(i-L) mod n). Every other neighbour's latest visit is <= U-L-1,
//    so its word is final once the decider has published progress P >= U-L,
//    and no later write can happen before U. The spin-independent split of
//    each adjacency row into "far" entries and a 32-bit "window" mask is
//    precomputed once per graph on the host (gdi_graph_create).
//  * the decider warp (0) adds the window part exactly from a 32-bit history
//    of its own last 32 decisions: field = f_far + 2*popc(hist & mask+) -
//    2*popc(hist & mask-) (constants folded into f_far), then runs the
//    reference decision (anneal.cpp:94-127) in 32-bit arithmetic (selected
//    only when |4A|(n+1) + |B| max_i sum_j |w_ij| < 2^31, so it equals the
//    int64 reference), the xoshiro256++ stream-1 draws (coin only on exact
//    ties) and the flip test x <= floor(pf*2^53)*2^11 + 2047.
//  * gatherer -> decider: queue of QB batches x B visits of {f_far, own} per
//    lane + the window masks; release/acquire on per-batch sequence numbers.
//    decider -> gatherers: progress counter P (release per batch).
//
// Restricted to |w| == 1 graphs (unit or +-1), n >= 2L, sweeps*n < 2^31;
// everything else runs k1_exact.cu. Incremental exact cut for the trace as
// in k1_exact.cu.
#include <cuda/atomic>
#include <cuda_runtime.h>

#include "device_rng.cuh"
#include "kernels.cuh"
#include "launch.hpp"

namespace gdi {

namespace {

constexpr int kWin = 32;   // window L (history bits)
constexpr int kBatch = 4;  // visits per queue batch (B)
constexpr int kQB = 16;    // queue depth in batches (QB*B > L + 1)

__device__ __forceinline__ int ld_acquire(const int* p) {
  cuda::atomic_ref<const int, cuda::thread_scope_block> r(*p);
  return r.load(cuda::memory_order_acquire);
}
__device__ __forceinline__ void st_release(int* p, int v) {
  cuda::atomic_ref<int, cuda::thread_scope_block> r(*p);
  r.store(v, cuda::memory_order_release);
}

struct PipeSmem {
  uint32_t* words;  // [n_pad] (+1 zero word at index n for padding entries)
  int2* q;          // [QB][B][32] {f_far, own}
  uint2* qm;        // [QB][B] {mask+, mask-}
  int* ready;       // [QB]
  int* progress;    // [1]
  long long* part;  // [NW][32] initial-cut partials
};

__device__ __forceinline__ PipeSmem carve(unsigned char* base, int n_words, int nwarps) {
  PipeSmem s;
  s.words = reinterpret_cast<uint32_t*>(base);
  unsigned char* p = base + static_cast<size_t>(n_words) * 4;
  s.q = reinterpret_cast<int2*>(p);
  p += sizeof(int2) * kQB * kBatch * 32;
  s.qm = reinterpret_cast<uint2*>(p);
  p += sizeof(uint2) * kQB * kBatch;
  s.part = reinterpret_cast<long long*>(p);
  p += sizeof(long long) * nwarps * 32;
  s.ready = reinterpret_cast<int*>(p);
  p += sizeof(int) * kQB;
  s.progress = reinterpret_cast<int*>(p);
  return s;
}

template <bool SIGNED, int NG>
__global__ void __launch_bounds__(32 * (NG + 1), 1) k1_pipe(const PipeArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int NW = NG + 1;
  const int n = a.g.n;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int replica = blockIdx.x * a.rc + lane;
  const bool active = lane < a.rc && replica < a.replicas;
  PipeSmem sm = carve(smem_raw, a.n_words, NW);
  const long long total = static_cast<long long>(a.sweeps) * n;
  const int nbatches = static_cast<int>((total + kBatch - 1) / kBatch);

  // ---------------- init (anneal.cpp:148-155): lane = replica, stream 0
  int G = 0;  // meaningful in warp 0 (the decider) only
  if (warp == 0) {
    const uint64_t seed = active ? a.seeds[replica] : 0ull;
    Xoshiro r0 = Xoshiro::stream(seed, 0);
    for (int i = 0; i < n; i++) {
      const bool up = (r0.next() >> 63) != 0;
      G += up ? 1 : -1;
      const unsigned w = __ballot_sync(0xffffffffu, up);
      if (lane == 0) sm.words[i] = w;
    }
    if (lane == 0) {
      for (int i = n; i < a.n_words; i++) sm.words[i] = 0u;  // padding entries read 0
      *sm.progress = 0;
    }
    if (lane < kQB) sm.ready[lane] = -1;
  }
  __syncthreads();

  // exact initial cut, all warps (evaluate.cpp:10-18), per lane = replica
  long long cut = 0;
  for (int u = warp; u < n; u += NW) {
    const unsigned su = (sm.words[u] >> lane) & 1u;
    const int e1 = __ldg(a.g.off + u + 1);
    for (int e = __ldg(a.g.off + u); e < e1; e++) {
      const int v = __ldg(a.g.col + e);
      if (v > u && ((sm.words[v] >> lane) & 1u) != su) cut += SIGNED ? __ldg(a.g.w + e) : 1;
    }
  }
  sm.part[warp * 32 + lane] = cut;
  __syncthreads();

  if (warp == 0) {
    // ============================ decider ============================
    for (int w = 1; w < NW; w++) cut += sm.part[w * 32 + lane];
    const size_t rs = static_cast<size_t>(replica);
    const int sweeps = a.sweeps;
    if (active && a.stamps != nullptr) a.stamps[rs * (sweeps + 1)] = globaltimer_ns();
    if (active && a.snaps != nullptr)
      for (int i = 0; i < n; i++) a.snaps[rs * (sweeps + 1) * n + i] = ((sm.words[i] >> lane) & 1u) ? 1 : -1;
    // history: bit k-1 = spin of vertex (0 - k) mod n, k = 1..L
    uint32_t hist = 0;
    for (int k = kWin; k >= 1; k--) hist = (hist << 1) | ((sm.words[n - k] >> lane) & 1u);

    const uint64_t seed = active ? a.seeds[replica] : 0ull;
    Xoshiro rng = Xoshiro::stream(seed, 1);
    const int a4 = a.a4, bb = a.b;
    int AG = a4 * G;
    int sweep = 0, i = 0;
    unsigned long long tm = a.tmask[0];
    bool en = a.thr[0] >= 0;

    for (int b = 0; b < nbatches; b++) {
      const int slot = b % kQB;
      while (ld_acquire(sm.ready + slot) != b) {
      }
      const int2* qs = sm.q + slot * kBatch * 32;
      const uint2* ms = sm.qm + slot * kBatch;
      const int nv = static_cast<int>(min(static_cast<long long>(kBatch), total - static_cast<long long>(b) * kBatch));
#pragma unroll
      for (int t = 0; t < kBatch; t++) {
        if (t < nv) {
          const int2 fo = qs[t * 32 + lane];
          const uint2 mw = ms[t];
          int f = fo.x + 2 * __popc(hist & mw.x);
          if (SIGNED) f -= 2 * __popc(hist & mw.y);
          const int own = fo.y;
          const int diff = AG - a4 * own - bb * f;
          uint64_t x = rng.next();
          int c;
          if (diff == 0) {  // exact tie: coin, then the unit draw (anneal.cpp:106-121)
            c = (static_cast<long long>(x) < 0) ? 1 : -1;
            x = rng.next();
          } else {
            c = diff < 0 ? 1 : -1;
          }
          const int fin = (en && x <= tm) ? -c : c;
          const int d = fin - own;
          AG += a4 * d;
          G += d;
          cut -= static_cast<long long>(d >> 1) * f;
          hist = (hist << 1) | static_cast<uint32_t>(fin > 0);
          const unsigned w = __ballot_sync(0xffffffffu, fin > 0);
          if (lane == 0) sm.words[i] = w;
          if (++i == n) {  // record_barrier (anneal.cpp:165-187)
            if (active) {
              if (a.trace != nullptr) a.trace[rs * sweeps + sweep] = DevTrace{cut, G, G};
              if (a.stamps != nullptr) a.stamps[rs * (sweeps + 1) + sweep + 1] = globaltimer_ns();
            }
            if (a.snaps != nullptr) {
              __syncwarp();
              if (active) {
                int8_t* dst = a.snaps + (rs * (sweeps + 1) + sweep + 1) * n;
                for (int v = 0; v < n; v++) dst[v] = ((sm.words[v] >> lane) & 1u) ? 1 : -1;
              }
            }
            i = 0;
            if (++sweep < sweeps) {
              tm = a.tmask[sweep];
              en = a.thr[sweep] >= 0;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) st_release(sm.progress, (b + 1) * kBatch);
    }
    if (active) a.final_out[rs] = DevTrace{cut, G, G};
  } else {
    // ============================ gatherers ============================
    const int g = warp - 1;
    const int4* __restrict__ fcol = a.far_col;
    const int4* __restrict__ meta = a.far_meta;
    for (int b = g; b < nbatches; b += NG) {
      const long long U0 = static_cast<long long>(b) * kBatch;
      const int need = static_cast<int>(U0) + kBatch - 1 - kWin;
      if (need > 0)
        while (ld_acquire(sm.progress) < need) __nanosleep(32);
      const int slot = b % kQB;
      int i = static_cast<int>(U0 % n);
      const int nv = static_cast<int>(min(static_cast<long long>(kBatch), total - U0));
      for (int t = 0; t < nv; t++) {
        const int4 md = __ldg(meta + i);  // {off4, pos4, neg4, fconst}
        int cp = 0, cn = 0;
        const int e_pos = md.x + md.y;
        for (int e = md.x; e < e_pos; e++) {
          const int4 c = __ldg(fcol + e);
          cp += ((sm.words[c.x] >> lane) & 1u) + ((sm.words[c.y] >> lane) & 1u) +
                ((sm.words[c.z] >> lane) & 1u) + ((sm.words[c.w] >> lane) & 1u);
        }
        if (SIGNED) {
          const int e_neg = e_pos + md.z;
          for (int e = e_pos; e < e_neg; e++) {
            const int4 c = __ldg(fcol + e);
            cn += ((sm.words[c.x] >> lane) & 1u) + ((sm.words[c.y] >> lane) & 1u) +
                  ((sm.words[c.z] >> lane) & 1u) + ((sm.words[c.w] >> lane) & 1u);
          }
        }
        const int own = ((sm.words[i] >> lane) & 1u) ? 1 : -1;
        sm.q[(slot * kBatch + t) * 32 + lane] = make_int2(2 * (cp - cn) - md.w, own);
        if (lane == 0) sm.qm[slot * kBatch + t] = make_uint2(__ldg(a.win_pos + i), SIGNED ? __ldg(a.win_neg + i) : 0u);
        if (++i == n) i = 0;
      }
      __syncwarp();
      if (lane == 0) st_release(sm.ready + slot, b);
    }
  }

  __syncthreads();
  // final spins, all warps: spins_out[r][v] (lane = replica)
  if (active)
    for (int v = warp; v < n; v += NW)
      a.spins_out[static_cast<size_t>(replica) * n + v] = ((sm.words[v] >> lane) & 1u) ? 1 : -1;
}

template <bool S, int NG>
const void* pipe_fn() {
  return reinterpret_cast<const void*>(&k1_pipe<S, NG>);
}

}  // namespace

size_t pipe_smem_bytes(int n_words, int nwarps) {
  return static_cast<size_t>(n_words) * 4 + sizeof(int2) * kQB * kBatch * 32 + sizeof(uint2) * kQB * kBatch +
         sizeof(long long) * nwarps * 32 + sizeof(int) * (kQB + 1);
}

int pipe_window() { return kWin; }

int pipe_plan(const GraphStats& st, const PipeGraph& pg, int32_t replicas, int64_t a4, int64_t b,
              int32_t sweeps, PipePlan* plan) {
  if (!pg.ok) return -1;
  if (static_cast<long long>(sweeps) * st.n >= (1LL << 31) - 64) return -1;
  const long long absa4 = a4 < 0 ? -a4 : a4, absb = b < 0 ? -b : b;
  // narrow arithmetic must be exact: |AG - a4*own - b*f| < 2^31 always
  const double bound = static_cast<double>(absa4) * (st.n + 1) + static_cast<double>(absb) * st.max_abs_field;
  if (bound >= 2147483647.0) return -1;
  constexpr int NG = 7;
  const int nw = NG + 1;
  const int n_words = pg.n_words;
  const size_t smem = pipe_smem_bytes(n_words, nw);
  if (smem > 200 * 1024) return -1;
  // replicas per CTA: spread R over the SMs (the per-replica chain is the
  // bound, so fewer lanes per CTA only adds parallel CTAs)
  int rc = (replicas + 147) / 148;
  rc = rc < 1 ? 1 : rc > 32 ? 32 : rc;
  plan->fn = st.unit ? pipe_fn<false, NG>() : pipe_fn<true, NG>();
  plan->rc = rc;
  plan->block = 32 * nw;
  plan->grid = (replicas + rc - 1) / rc;
  plan->smem = static_cast<int>(smem);
  plan->name = st.unit ? "k1_pipe<unit>" : "k1_pipe<signed>";
  return 0;
}

cudaError_t pipe_launch(const PipePlan& plan, const PipeArgs& args, cudaStream_t stream) {
  cudaError_t err = cudaFuncSetAttribute(plan.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, plan.smem);
  if (err != cudaSuccess) return err;
  PipeArgs a = args;
  a.rc = plan.rc;
  void* params[] = {&a};
  return cudaLaunchKernel(plan.fn, dim3(plan.grid), dim3(plan.block), params, plan.smem, stream);
}

}  // namespace gdi
