// K3 — fused exact partition evaluation (sm_100a).
//
// One pass over the CSR per replica computes the exact cut (each edge once,
// u < v, reference proj/src/evaluate.cpp:10-18 and anneal.cpp:64-70) and the
// spin sum (evaluate.cpp:20-23) together; H_scaled = a*sum^2 + b*cut is
// formed on the host from the two integers (evaluate.cpp:25-32).
//
// Layout: grid.y = replica, grid.x = vertex chunks of that replica. A thread
// owns one vertex: it reads its own spin once, walks its adjacency row and
// compares against the neighbour spins (L1/L2 resident for every config in
// BASELINE.json). Partial sums are reduced warp -> block with shuffles and
// shared memory, then one 64-bit atomic per block and quantity.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "launch.hpp"

namespace gdi {

namespace {

constexpr int kEvalBlock = 256;
constexpr int kEvalVertsPerThread = 4;

template <bool WEIGHTED>
__global__ void __launch_bounds__(kEvalBlock) k3_eval(const EvalArgs a) {
  const int n = a.g.n;
  const int r = blockIdx.y;
  const int8_t* __restrict__ s = a.spins + static_cast<size_t>(r) * n;
  long long cut = 0, sum = 0;
  const int stride = gridDim.x * blockDim.x;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride) {
    const int su = s[u];
    sum += su;
    const int e1 = __ldg(a.g.off + u + 1);
    for (int e = __ldg(a.g.off + u); e < e1; e++) {
      const int v = __ldg(a.g.col + e);
      if (u < v && su != s[v]) cut += WEIGHTED ? __ldg(a.g.w + e) : 1;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cut += __shfl_xor_sync(0xffffffffu, cut, o);
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
  __shared__ long long red[2][kEvalBlock / 32];
  const int warp = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0) {
    red[0][warp] = cut;
    red[1][warp] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long c = 0, t = 0;
    for (int w = 0; w < kEvalBlock / 32; w++) {
      c += red[0][w];
      t += red[1][w];
    }
    atomicAdd(a.out + 2 * r, static_cast<unsigned long long>(c));
    atomicAdd(a.out + 2 * r + 1, static_cast<unsigned long long>(t));
  }
}

}  // namespace

cudaError_t eval_launch(const EvalArgs& args, bool weighted, cudaStream_t stream) {
  const int per_block = kEvalBlock * kEvalVertsPerThread;
  int chunks = (args.g.n + per_block - 1) / per_block;
  if (chunks < 1) chunks = 1;
  if (chunks > 4096) chunks = 4096;
  dim3 grid(chunks, args.replicas);
  if (weighted)
    k3_eval<true><<<grid, kEvalBlock, 0, stream>>>(args);
  else
    k3_eval<false><<<grid, kEvalBlock, 0, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace gdi
