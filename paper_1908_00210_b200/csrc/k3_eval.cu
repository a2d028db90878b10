// K3 — fused exact partition evaluation (sm_100a): cut and spin sum of R spin
// vectors, the reference's cut_value / imbalance / score (proj/src/evaluate.cpp:
// 10-32; the same cut as record_barrier's cut_of, anneal.cpp:64-70).
// H_scaled = a * sum^2 + b * cut is formed on the host from the two integers.
//
// Input: int8 spins [R][n] in HBM (+1 / -1; any other byte sets the `bad`
// flag, the reference's "spin must be -1 or +1" domain error). The graph is
// the canonical edge list (u < v, build_eval_layout): one word u | v << 16
// per edge when n <= 65536, else int2; +1 edges first for +-1 weights.
//
// Two kernels, by shape:
//
// k3_sliced (many replicas, |w| == 1, n small enough for 4n bytes of shared
// memory): bit-sliced over 32 replicas. A CTA takes a group of 32 replicas
// and a slice of the edges. It first transposes the group's spins into
// shared memory, one 32-bit word per vertex (bit r = replica 32g + r is +1):
// lane r reads 32 consecutive spin bytes of its replica, 32 ballots turn
// them into the 32 vertex words. Then every edge costs one coalesced load
// and two shared-memory loads for all 32 replicas: x = T[u] ^ T[v] is the
// mask of replicas that cut the edge, summed per bit position by a
// carry-save (Harley-Seal) adder tree into bit-sliced counters. At the end
// a 32 x 32 bit transpose per counter level (warp shuffles) and a popcount
// give each lane its replica's count. ~14 instructions per edge for 32
// replicas instead of ~6 per edge per replica.
//
// k3_pack + k3_bits (one or few replicas, large graphs such as the
// 1M-vertex config, or general weights): k3_pack packs each replica's spins
// into bit words (+ spin sum); k3_bits copies one replica's words into
// shared memory (125 KB for 1M vertices) and streams the edges: one
// coalesced 8-byte load and two shared-memory bit lookups per edge, so the
// kernel is bound by the edge stream (8 B per edge from HBM / L2).
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"
#include "launch.hpp"

namespace gdi {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kSliceBlock = 256;
constexpr int kBitsBlock = 1024;
constexpr int kLevels = 20;  // bit-sliced counter levels above the Harley-Seal eights: < 8 * 2^20 edges per thread

__device__ __forceinline__ void csa(unsigned& h, unsigned& l, unsigned a, unsigned b, unsigned c) {
  const unsigned u = a ^ b;
  h = (a & b) | (u & c);
  l = u ^ c;
}

// 32 x 32 bit transpose across the warp: lane t holds row t (bit c = column
// c) on entry, column t on exit (bit r = row r's bit t).
__device__ __forceinline__ unsigned transpose32(unsigned x, int lane) {
  const unsigned masks[5] = {0x0000ffffu, 0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int s = 0; s < 5; s++) {
    const int j = 16 >> s;
    const unsigned m = masks[s];
    const unsigned y = __shfl_xor_sync(FULL, x, j);
    x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
  }
  return x;
}

// +1 mask of the four spin bytes of x (bit 7 of each byte), and whether every
// byte is +1 (0x01) or -1 (0xff)
__device__ __forceinline__ unsigned pos_bits(unsigned x) { return ~x & 0x80808080u; }
__device__ __forceinline__ bool valid4(unsigned x) {
  const unsigned s = (x >> 7) & 0x01010101u;
  return x == ((s * 0xffu) | (s ^ 0x01010101u));
}

// Bit-sliced per-replica counter: ones/twos/fours + levels of eights.
struct Sliced {
  unsigned ones = 0, twos = 0, fours = 0, lv[kLevels];
  __device__ Sliced() {
#pragma unroll
    for (int i = 0; i < kLevels; i++) lv[i] = 0;
  }
  __device__ __forceinline__ void add8(const unsigned (&x)[8]) {
    unsigned ta, tb, fa, fb, e;
    csa(ta, ones, ones, x[0], x[1]);
    csa(tb, ones, ones, x[2], x[3]);
    csa(fa, twos, twos, ta, tb);
    csa(ta, ones, ones, x[4], x[5]);
    csa(tb, ones, ones, x[6], x[7]);
    csa(fb, twos, twos, ta, tb);
    csa(e, fours, fours, fa, fb);
#pragma unroll
    for (int i = 0; i < kLevels; i++) {
      const unsigned t = lv[i] & e;
      lv[i] ^= e;
      e = t;
    }
  }
  // this warp's count for replica `lane` (levels that are zero in every lane
  // are skipped)
  __device__ __forceinline__ long long count(int lane) const {
    long long c = 0;
    if (__any_sync(FULL, ones)) c += __popc(transpose32(ones, lane));
    if (__any_sync(FULL, twos)) c += 2ll * __popc(transpose32(twos, lane));
    if (__any_sync(FULL, fours)) c += 4ll * __popc(transpose32(fours, lane));
#pragma unroll
    for (int i = 0; i < kLevels; i++)
      if (__any_sync(FULL, lv[i])) c += (8ll << i) * __popc(transpose32(lv[i], lane));
    return c;
  }
};

template <bool NARROW>
__device__ __forceinline__ void edge_at(const EvalArgs& a, long long e, int& u, int& v) {
  if (NARROW) {
    const unsigned x = __ldg(static_cast<const unsigned*>(a.edges) + e);
    u = static_cast<int>(x & 0xffffu);
    v = static_cast<int>(x >> 16);
  } else {
    const int2 x = __ldg(static_cast<const int2*>(a.edges) + e);
    u = x.x;
    v = x.y;
  }
}

// This thread's cut count over edges [lo, hi) for the 32 replicas of T.
template <bool NARROW>
__device__ __forceinline__ long long sliced_range(const EvalArgs& a, const unsigned* T, long long lo, long long hi,
                                                  int lane) {
  Sliced acc;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  long long e = lo + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  while (__any_sync(FULL, e < hi)) {
    unsigned x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      x[k] = 0u;
      const long long ek = e + k * stride;
      if (ek < hi) {
        int u, v;
        edge_at<NARROW>(a, ek, u, v);
        x[k] = T[u] ^ T[v];
      }
    }
    acc.add8(x);
    e += 8 * stride;
  }
  return acc.count(lane);
}

// 32 spin bytes (8 words) -> 32 bits, bit j = byte j is +1
__device__ __forceinline__ unsigned pack32(const unsigned (&w)[8]) {
  unsigned bits = 0u;
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const unsigned t = (~w[k] >> 7) & 0x01010101u;   // byte b -> bit 8b
    bits |= ((t * 0x01020408u) >> 24 & 0xfu) << (4 * k);  // bits 24..27 = bytes 0..3
  }
  return bits;
}

// 32 spin bytes of one replica row from v0 on (lim valid bytes; +1 padding)
__device__ __forceinline__ void load32(const int8_t* row, int v0, int lim, bool aligned4, unsigned (&w)[8]) {
  if (aligned4 && lim >= 32) {
    const uint4* q = reinterpret_cast<const uint4*>(row + v0);
    if ((reinterpret_cast<uintptr_t>(q) & 15) == 0) {
      const uint4 x = __ldg(q), y = __ldg(q + 1);
      w[0] = x.x, w[1] = x.y, w[2] = x.z, w[3] = x.w, w[4] = y.x, w[5] = y.y, w[6] = y.z, w[7] = y.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; k++) w[k] = __ldg(reinterpret_cast<const unsigned*>(row + v0) + k);
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < 8; k++) {
    unsigned x = 0x01010101u;
    for (int b = 0; b < 4; b++)
      if (4 * k + b < lim)
        x = (x & ~(0xffu << (8 * b))) | (static_cast<unsigned>(static_cast<uint8_t>(row[v0 + 4 * k + b])) << (8 * b));
    w[k] = x;
  }
}

// Transpose of a replica group's spins into vertex words T[g][v] (bit r =
// replica 32g + r is +1), with the spin sums and the byte check. Warp = one
// 32-vertex block of one group: lane r packs its replica's 32 bytes into one
// word, a 32 x 32 bit transpose hands lane j the word of vertex v0 + j.
__global__ void __launch_bounds__(256) k3_slice(const EvalArgs a) {
  const int n = a.n, lane = threadIdx.x & 31, g = blockIdx.y, r = 32 * g + lane;
  const bool live = r < a.R;
  const int8_t* row = a.spins + static_cast<size_t>(live ? r : 0) * n;
  const int nb = (n + 31) >> 5, gw = gridDim.x * (blockDim.x >> 5);
  long long pop = 0;
  bool ok = true;
  for (int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += gw) {
    const int v0 = 32 * b, lim = n - v0;
    unsigned w[8];
    load32(row, v0, lim, a.aligned4, w);
#pragma unroll
    for (int k = 0; k < 8; k++) ok &= valid4(w[k]);
    unsigned bits = live ? pack32(w) : 0u;
    if (lim < 32) bits &= (1u << lim) - 1u;
    pop += __popc(bits);
    const unsigned col = transpose32(bits, lane);
    if (lane < lim) a.work[static_cast<size_t>(g) * n + v0 + lane] = col;
  }
  ok = __all_sync(FULL, ok || !live);
  const long long add = 2 * pop - (blockIdx.x == 0 && threadIdx.x < 32 ? n : 0);  // spin sum; one warp adds -n
  if (live && add != 0) atomicAdd(a.out + 2 * r + 1, static_cast<unsigned long long>(add));
  if (!ok && lane == 0) atomicOr(a.bad, 1u);
}

// The cut of a replica group over one slice of the edges, T[g] staged in
// shared memory.
template <bool NARROW, bool SIGNED>
__global__ void __launch_bounds__(kSliceBlock) k3_sliced(const EvalArgs a) {
  extern __shared__ __align__(16) unsigned T[];
  __shared__ long long cnt[32];
  const int n = a.n, lane = threadIdx.x & 31, g = blockIdx.y;
  const unsigned* src = a.work + static_cast<size_t>(g) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) T[i] = __ldg(src + i);
  if (threadIdx.x < 32) cnt[threadIdx.x] = 0;
  __syncthreads();
  long long c = sliced_range<NARROW>(a, T, 0, a.mpos, lane);
  if (SIGNED) c -= sliced_range<NARROW>(a, T, a.mpos, a.m, lane);
  if (c != 0) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[lane]), static_cast<unsigned long long>(c));
  __syncthreads();
  if (threadIdx.x < 32 && 32 * g + threadIdx.x < a.R && cnt[threadIdx.x] != 0)
    atomicAdd(a.out + 2 * (32 * g + threadIdx.x), static_cast<unsigned long long>(cnt[threadIdx.x]));
}

// int8 spins -> bit words [R][nwp] + the spin sum. Thread = one word of one
// replica (32 bytes: two 16-byte loads when the rows are aligned).
__global__ void __launch_bounds__(256) k3_pack(const EvalArgs a) {
  const int n = a.n, nw = (n + 31) >> 5, r = blockIdx.y;
  const int8_t* row = a.spins + static_cast<size_t>(r) * n;
  unsigned pop = 0;
  bool ok = true;
  for (int wi = blockIdx.x * blockDim.x + threadIdx.x; wi < nw; wi += gridDim.x * blockDim.x) {
    const int v0 = 32 * wi, lim = n - v0;
    unsigned w[8];
    load32(row, v0, lim, a.aligned4, w);
#pragma unroll
    for (int k = 0; k < 8; k++) ok &= valid4(w[k]);
    unsigned bits = pack32(w);
    if (lim < 32) bits &= (1u << lim) - 1u;
    pop += __popc(bits);
    a.work[static_cast<size_t>(r) * a.nwp + wi] = bits;
  }
  pop = __reduce_add_sync(FULL, pop);
  ok = __all_sync(FULL, ok);
  if ((threadIdx.x & 31) == 0) {
    // the spin sum 2 * pop - n: every warp adds 2 * its pop, the first warp also -n
    const long long add = 2ll * pop - (blockIdx.x == 0 && threadIdx.x == 0 ? n : 0);
    if (add != 0) atomicAdd(a.out + 2 * r + 1, static_cast<unsigned long long>(add));
    if (!ok) atomicOr(a.bad, 1u);
  }
}

// One replica's cut over a slice of the edges, bit words in shared memory
// (SM) or, for graphs whose words do not fit it, read through L1 (__ldg).
template <bool NARROW, int WK, bool SM>
__global__ void __launch_bounds__(kBitsBlock) k3_bits(const EvalArgs a) {
  extern __shared__ __align__(16) unsigned S[];
  __shared__ long long red[kBitsBlock / 32];
  const int r = blockIdx.y, nw4 = a.nwp >> 2;
  const unsigned* words = a.work + static_cast<size_t>(r) * a.nwp;
  if (SM) {
    const uint4* src = reinterpret_cast<const uint4*>(words);
#pragma unroll 8
    for (int i = threadIdx.x; i < nw4; i += blockDim.x) reinterpret_cast<uint4*>(S)[i] = __ldcg(src + i);
    __syncthreads();
  }
  auto bit = [&](int v) { return ((SM ? S[v >> 5] : __ldg(words + (v >> 5))) >> (v & 31)) & 1u; };
  long long cut = 0;
  auto one = [&](int u, int v, long long e) {
    const bool c = bit(u) != bit(v);
    if (WK == 0) cut += c;
    if (WK == 1) cut += c ? (e < a.mpos ? 1 : -1) : 0;
    if (WK == 2) cut += c ? __ldg(a.w + e) : 0;
  };
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long m = a.m;
  // 16-byte edge loads (4 narrow / 2 wide edges), 4 issued before any is
  // used (out-of-range slots are the edge (0, 0): never cut)
  constexpr int PER = NARROW ? 4 : 2;
  const long long mq = m / PER;
  const uint4* E = static_cast<const uint4*>(a.edges);
  for (long long q0 = tid; q0 < mq; q0 += 4 * stride) {
    uint4 x[4];
#pragma unroll
    for (int k = 0; k < 4; k++) x[k] = q0 + k * stride < mq ? __ldg(E + q0 + k * stride) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const long long e = (q0 + k * stride) * PER;
      if (NARROW) {
        one(x[k].x & 0xffffu, x[k].x >> 16, e);
        one(x[k].y & 0xffffu, x[k].y >> 16, e + 1);
        one(x[k].z & 0xffffu, x[k].z >> 16, e + 2);
        one(x[k].w & 0xffffu, x[k].w >> 16, e + 3);
      } else {
        one(static_cast<int>(x[k].x), static_cast<int>(x[k].y), e);
        one(static_cast<int>(x[k].z), static_cast<int>(x[k].w), e + 1);
      }
    }
  }
  for (long long e = mq * PER + tid; e < m; e += stride) {
    int u, v;
    edge_at<NARROW>(a, e, u, v);
    one(u, v, e);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cut += __shfl_xor_sync(FULL, cut, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cut;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < kBitsBlock / 32; w++) t += red[w];
    if (t != 0) atomicAdd(a.out + 2 * r, static_cast<unsigned long long>(t));
  }
}

template <bool NARROW, bool SM>
const void* bits_fn(int wkind) {
  return wkind == 0   ? reinterpret_cast<const void*>(&k3_bits<NARROW, 0, SM>)
         : wkind == 1 ? reinterpret_cast<const void*>(&k3_bits<NARROW, 1, SM>)
                      : reinterpret_cast<const void*>(&k3_bits<NARROW, 2, SM>);
}

int sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

}  // namespace

bool eval_sliced(int n, int replicas, int wkind) {
  return wkind != 2 && replicas >= 16 && static_cast<long long>(n) * 4 <= 200 * 1024;
}

long long eval_work_words(int n, int replicas, int wkind) {
  if (eval_sliced(n, replicas, wkind)) return static_cast<long long>((replicas + 31) / 32) * n;
  return static_cast<long long>(replicas) * (((n + 31) / 32 + 3) & ~3);
}

cudaError_t eval_launch(EvalArgs a, int wkind, cudaStream_t stream, int* launches) {
  const int sms = sm_count();
  const int n = a.n;
  a.aligned4 = n % 4 == 0 && (reinterpret_cast<uintptr_t>(a.spins) & 3) == 0;
  const bool narrow = a.narrow;
  if (wkind == 0) a.mpos = a.m;
  cudaError_t e;
  if (eval_sliced(n, a.R, wkind)) {
    const int groups = (a.R + 31) / 32;
    // transpose: 8 vertex blocks per CTA, ~4 CTAs per SM in all
    {
      const long long nb = (n + 31) / 32;
      long long gx = (nb + 7) / 8;
      const long long cap = (4LL * sms + groups - 1) / groups;
      if (gx > cap) gx = cap;
      if (gx < 1) gx = 1;
      k3_slice<<<dim3(static_cast<unsigned>(gx), groups), 256, 0, stream>>>(a);
      if ((e = cudaGetLastError())) return e;
    }
    // cut: slices per group for ~2 CTAs per SM in all, >= 16 edges per thread
    const size_t smem = static_cast<size_t>(n) * 4;
    long long S = (2LL * sms + groups - 1) / groups;
    const long long maxs = a.m / (16LL * kSliceBlock);
    if (S > maxs) S = maxs;
    if (S < 1) S = 1;
    const void* fn = narrow ? (wkind == 1 ? reinterpret_cast<const void*>(&k3_sliced<true, true>)
                                          : reinterpret_cast<const void*>(&k3_sliced<true, false>))
                            : (wkind == 1 ? reinterpret_cast<const void*>(&k3_sliced<false, true>)
                                          : reinterpret_cast<const void*>(&k3_sliced<false, false>));
    if (smem > 48 * 1024 && (e = allow_max_smem(fn))) return e;
    void* params[] = {&a};
    if (launches) *launches = 2;
    return cudaLaunchKernel(fn, dim3(static_cast<unsigned>(S), groups), dim3(kSliceBlock), params, smem, stream);
  }
  a.nwp = ((n + 31) / 32 + 3) & ~3;
  {
    const int nw = (n + 31) / 32;
    const int gx = (nw + 255) / 256 < 4 * sms ? (nw + 255) / 256 : 4 * sms;
    k3_pack<<<dim3(gx < 1 ? 1 : gx, a.R), 256, 0, stream>>>(a);
  }
  if ((e = cudaGetLastError())) return e;
  bool sm = static_cast<long long>(a.nwp) * 4 <= 227 * 1024;
  if (const char* x = std::getenv("GDI_K3_SMEM")) sm = sm && std::atoi(x) != 0;  // A/B: L1-cached lookups
  const size_t smem = sm ? static_cast<size_t>(a.nwp) * 4 : 0;
  long long per = (static_cast<long long>(sms) + a.R - 1) / a.R;  // ~1 CTA per SM in all
  const long long maxs = (a.m + 4LL * kBitsBlock - 1) / (4LL * kBitsBlock);
  if (per > maxs) per = maxs;
  if (per < 1) per = 1;
  const void* fn = narrow ? (sm ? bits_fn<true, true>(wkind) : bits_fn<true, false>(wkind))
                          : (sm ? bits_fn<false, true>(wkind) : bits_fn<false, false>(wkind));
  if (smem > 48 * 1024 && (e = allow_max_smem(fn))) return e;
  void* params[] = {&a};
  if (launches) *launches = 2;
  return cudaLaunchKernel(fn, dim3(static_cast<unsigned>(per), a.R), dim3(kBitsBlock), params, smem, stream);
}

}  // namespace gdi
