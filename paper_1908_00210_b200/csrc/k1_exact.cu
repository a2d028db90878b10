// K1 — bit-exact replica-batched GDI sweep kernel (sm_100a).
//
// Restates, per replica, the reference's deterministic single-worker anneal
// (reference proj/src/anneal.cpp:132-231 with workers == 1; visit_node at
// :86-128; record_barrier at :165-187), so that final spins, every trace
// record and the final score are bit-identical to the CPU reference.
//
// Why this shape. Within one replica the visit sequence is inherently
// serial: visit i reads the live counter G (changed by visit i-1), the
// neighbour spins (possibly changed earlier in the sweep) and the xoshiro
// stream position (advanced by one draw per visit plus one per exact tie).
// Parallelism therefore comes from (a) independent replicas and (b) the
// neighbour gather of a single visit. A group of GS lanes owns one replica:
// lanes split the adjacency row (lane k takes entries k, k+GS, ...), reduce
// the partial fields with xor-shuffles, then every lane of the group
// evaluates the identical decision on identical register state (G, cut,
// xoshiro), so no broadcast is needed. Spins live in shared memory as int8,
// one n-byte row per replica. Every lane of the group writes a changed spin,
// so each lane later reads its own store in program order: no __syncwarp is
// needed between visits. All replicas of a warp visit the same vertex at the
// same time, so the CSR row loads are warp-wide broadcasts through L1.
//
// The per-sweep trace is incremental and exact: flipping sigma_i from s to
// -s changes the cut by exactly s * field_i (= -(fin - own) * field / 2),
// and the field is already reduced in registers; the initial cut is computed
// once in-kernel. This replaces the reference's full CSR pass per sweep
// (anneal.cpp:64-70, 174) at zero cost.
//
// The flip test `next_unit() <= pf` (anneal.cpp:120-123) is evaluated as the
// exactly equivalent integer test (x >> 11) <= floor(pf * 2^53), thresholds
// precomputed on the host from the iterated product pf *= decay (:183).
#include <cuda_runtime.h>

#include "device_rng.cuh"
#include "kernels.cuh"
#include "launch.hpp"

namespace gdi {

namespace {

template <int GS, typename T>
__device__ __forceinline__ T group_sum(T v) {
#pragma unroll
  for (int off = GS / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

template <int GS, bool WEIGHTED, bool FIELD64>
__global__ void __launch_bounds__(256) k1_exact(const ExactArgs a) {
  using Field = typename std::conditional<FIELD64, long long, int>::type;
  extern __shared__ __align__(16) int8_t smem_spins[];

  const int n = a.g.n;
  const int lane = threadIdx.x % GS;
  const int group = threadIdx.x / GS;
  const int replica = blockIdx.x * (blockDim.x / GS) + group;
  const bool active = replica < a.replicas;
  int8_t* s = smem_spins + static_cast<size_t>(group) * a.n_pad;
  const int32_t* __restrict__ off = a.g.off;
  const int32_t* __restrict__ col = a.g.col;
  const int32_t* __restrict__ wt = a.g.w;

  const uint64_t seed = active ? a.seeds[replica] : 0ull;

  // anneal.cpp:148-155 — stream 0 coins, G = sum. Every lane walks the
  // stream (it is serial); lane k stores indices i = k mod GS.
  long long G = 0;
  {
    Xoshiro r0 = Xoshiro::stream(seed, 0);
    for (int i = 0; i < n; i++) {
      const int v = (r0.next() >> 63) ? 1 : -1;
      G += v;
      if ((i % GS) == lane) s[i] = static_cast<int8_t>(v);
    }
  }
  __syncthreads();

  // Exact initial cut, each edge once (evaluate.cpp:10-18).
  long long cut = 0;
  for (int u = lane; u < n; u += GS) {
    const int su = s[u];
    const int e1 = __ldg(off + u + 1);
    for (int e = __ldg(off + u); e < e1; e++) {
      const int v = __ldg(col + e);
      if (u < v && su != s[v]) cut += WEIGHTED ? __ldg(wt + e) : 1;
    }
  }
  cut = group_sum<GS>(cut);

  const int sweeps = a.sweeps;
  const size_t rs = static_cast<size_t>(replica);
  if (active && a.snaps != nullptr)
    for (int i = lane; i < n; i += GS) a.snaps[rs * (sweeps + 1) * n + i] = s[i];
  if (active && lane == 0 && a.stamps != nullptr) a.stamps[rs * (sweeps + 1)] = globaltimer_ns();

  Xoshiro rng = Xoshiro::stream(seed, 1);  // anneal.cpp:191
  const unsigned long long a4 = static_cast<unsigned long long>(a.a4);
  const unsigned long long bb = static_cast<unsigned long long>(a.b);

  for (int sweep = 0; sweep < sweeps; sweep++) {
    const long long thr = __ldg(a.thr + sweep);
    int beg = __ldg(off);
    for (int i = 0; i < n; i++) {
      const int end = __ldg(off + i + 1);
      const int own = s[i];
      Field f = 0;
      for (int e = beg + lane; e < end; e += GS) {
        const int j = __ldg(col + e);
        if (WEIGHTED)
          f += static_cast<Field>(__ldg(wt + e)) * s[j];
        else
          f += s[j];
      }
      beg = end;
      f = group_sum<GS>(f);

      // diff = 4A * (G - own) - B * field, int64 with two's-complement wrap
      // (anneal.cpp:104-105).
      const long long diff = static_cast<long long>(
          a4 * static_cast<unsigned long long>(G - own) - bb * static_cast<unsigned long long>(
                                                               static_cast<long long>(f)));
      uint64_t x = rng.next();
      int c;
      if (diff == 0) {  // exact tie: coin first, then the unit draw (:106-112, :120)
        c = (x >> 63) ? 1 : -1;
        x = rng.next();
      } else {
        c = diff < 0 ? 1 : -1;
      }
      const int fin = (static_cast<long long>(x >> 11) <= thr) ? -c : c;
      if (fin != own) {
        s[i] = static_cast<int8_t>(fin);
        G += fin - own;
        cut -= static_cast<long long>(fin) * static_cast<long long>(f);
      }
    }
    // record_barrier (anneal.cpp:165-187): exact cut, spin sum, counter.
    if (active) {
      if (lane == 0 && a.trace != nullptr) a.trace[rs * sweeps + sweep] = DevTrace{cut, G, G};
      if (lane == 0 && a.stamps != nullptr)
        a.stamps[rs * (sweeps + 1) + sweep + 1] = globaltimer_ns();
      if (a.snaps != nullptr) {
        int8_t* dst = a.snaps + (rs * (sweeps + 1) + sweep + 1) * n;
        for (int i = lane; i < n; i += GS) dst[i] = s[i];
      }
    }
  }

  if (active) {
    for (int i = lane; i < n; i += GS) a.spins_out[rs * n + i] = s[i];
    if (lane == 0) a.final_out[rs] = DevTrace{cut, G, G};
  }
}

template <int GS, bool W, bool F64>
const void* pick3() {
  return reinterpret_cast<const void*>(&k1_exact<GS, W, F64>);
}

template <int GS>
const void* pick2(bool weighted, bool field64) {
  if (weighted) return field64 ? pick3<GS, true, true>() : pick3<GS, true, false>();
  return field64 ? pick3<GS, false, true>() : pick3<GS, false, false>();
}

}  // namespace

int exact_plan(const GraphStats& st, int32_t replicas, ExactPlan* plan) {
  // Lanes per replica from the mean degree: enough lanes that a typical row
  // is one or two strided passes, few enough that warps hold several
  // replicas (tuned on B200).
  const double mean_deg = st.n > 0 ? 2.0 * static_cast<double>(st.m) / st.n : 0.0;
  int gs = mean_deg <= 6 ? 4 : mean_deg <= 12 ? 8 : mean_deg <= 24 ? 16 : 32;
  const int n_pad = (st.n + 15) & ~15;
  const int smem_cap = 200 * 1024;
  int block = 128;
  // Shrink the block, then widen the group, until one block's spins fit.
  while (block > 32 && static_cast<long long>(block / gs) * n_pad > smem_cap) block /= 2;
  while (gs < 32 && static_cast<long long>(block / gs) * n_pad > smem_cap) gs *= 2;
  if (static_cast<long long>(block / gs) * n_pad > smem_cap) return -1;  // capacity
  const bool weighted = !st.unit;
  const bool field64 = st.max_abs_field > 0x7fffffffLL;
  const void* fn = nullptr;
  switch (gs) {
    case 4: fn = pick2<4>(weighted, field64); break;
    case 8: fn = pick2<8>(weighted, field64); break;
    case 16: fn = pick2<16>(weighted, field64); break;
    default: fn = pick2<32>(weighted, field64); break;
  }
  plan->fn = fn;
  plan->group = gs;
  plan->block = block;
  plan->n_pad = n_pad;
  plan->smem = (block / gs) * n_pad;
  plan->grid = (replicas + block / gs - 1) / (block / gs);
  plan->name = "k1_exact";
  return 0;
}

cudaError_t exact_launch(const ExactPlan& plan, const ExactArgs& args, cudaStream_t stream) {
  cudaError_t err = allow_max_smem(plan.fn);
  if (err != cudaSuccess) return err;
  ExactArgs a = args;
  void* params[] = {&a};
  return cudaLaunchKernel(plan.fn, dim3(plan.grid), dim3(plan.block), params, plan.smem, stream);
}

}  // namespace gdi
