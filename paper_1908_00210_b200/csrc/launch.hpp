// Host-side kernel selection and launch helpers (internal to libgdi).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace gdi {

// Dynamic shared memory above 48 KB needs a per-function opt-in. Sessions on
// different host threads launch the same kernels with different sizes, so the
// opt-in is always the device maximum (one value from every thread: setting
// each launch's own size raced with another thread's launch of the same
// function, "invalid argument"). The launch's own size is what it uses.
inline cudaError_t allow_max_smem(const void* fn) {
  int dev = 0, mx = 0;
  cudaFuncAttributes fa{};
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, fn);  // (the opt-in covers static + dynamic)
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             mx - static_cast<int>(fa.sharedSizeBytes));
  return e;
}


struct GraphStats {
  int32_t n = 0;
  int64_t m = 0;
  int32_t max_degree = 0;
  bool unit = true;
  bool pm1 = false;             // every |w| == 1 (unit or +-1)
  long long max_abs_field = 0;  // max_i sum_j |w_ij|
};

struct ExactPlan {
  const void* fn = nullptr;
  int group = 32;  // lanes per replica
  int block = 128;
  int grid = 1;
  int n_pad = 0;
  int smem = 0;
  const char* name = "";
};

// Returns 0, or -1 when no K1 variant fits (capacity).
int exact_plan(const GraphStats& st, int32_t replicas, ExactPlan* plan);
cudaError_t exact_launch(const ExactPlan& plan, const ExactArgs& args, cudaStream_t stream);

// Spin-independent preprocessing of a graph for k1_window (built once in
// gdi_graph_create when every |w| == 1 and n >= 64).
struct PipeGraph {
  bool ok = false;
  int32_t n_words = 0;
  uint32_t* win_pos = nullptr;
  uint32_t* win_neg = nullptr;
  uint32_t* fwd_pos = nullptr;  // forward window masks (layout.cu k_fwd_masks)
  uint32_t* fwd_neg = nullptr;
  int32_t* wsell = nullptr;  // k1_window rows
  int32_t* wsell_off = nullptr;
};

struct PipePlan {
  const void* fn = nullptr;
  int32_t a4 = 4, b = 4;  // coefficients reduced by gcd(4A, B)
  int rc = 8;
  int block = 256;
  int grid = 1;
  int smem = 0;
  bool prof = false;
  bool gw = false;  // spin words in global memory (graph too large for shared memory)
  int n_words = 0;  // k1_window: per-replica spin stride
  int nprod = 1;    // k1_window: RNG producer warps
  int rolemap = 1;  // k1_window: warp role layout
  int kp = 1;       // k1_window: producer lanes per replica stream
  int segl = 64;    // k1_window: draws per producer segment
  int rounds = 4;   // k1_window: producer rounds buffered per replica
  int ring_n = 2048;  // k1_window: draws per replica ring
  bool masks_smem = false;  // k1_window: window masks in shared memory
  bool jt2 = false;         // k1_window: two-column jump table
  const char* name = "";
};

constexpr int pipe_window() { return 32; }  // k1_window masks: 32 visits back / ahead
// k1_window (speculative visit windows)
int window_plan(const GraphStats& st, const PipeGraph& pg, int32_t replicas, int64_t a4, int64_t b,
                int32_t sweeps, PipePlan* plan);
cudaError_t window_launch(const PipePlan& plan, const PipeArgs& args, cudaStream_t stream);

// k1_block (aligned windows resolved to a fixed point, per-warp draws)
struct BlockPlan {
  const void* fn = nullptr;
  int32_t a4 = 4, b = 4;  // coefficients reduced by gcd(4A, B)
  int rc = 1;             // replica warps per CTA
  int rows = 0;           // > 0: row records in global memory (ExactArgs::brow, build_block_rows)
  int lane_rows = 0;      // max degree <= 16
  int block = 32, grid = 1, smem = 0, nnz = 0;
  const char* name = "";
};
int block_plan(const GraphStats& st, int32_t replicas, int64_t a4, int64_t b, int32_t sweeps, BlockPlan* plan);
cudaError_t block_launch(const BlockPlan& plan, const ExactArgs& args, cudaStream_t stream);

struct ThruPlan {
  const void* fn = nullptr;
  int32_t a4 = 4, b = 4;
  int block = 128, grid = 1, smem = 0, n_pad = 0;
  bool chains = false;  // k2_chains (cfg) rather than k2_sweep / k2_incf
  ChainCfg cfg{};
  const char* name = "";
};
// standard: the literal O(n)-per-visit `standard` strategy (anneal.cpp:97-101)
int thru_plan(const GraphStats& st, int wkind, int32_t replicas, int64_t a4, int64_t b, bool standard,
              ThruPlan* plan);
cudaError_t thru_launch(const ThruPlan& plan, const ThruArgs& args, cudaStream_t stream);

struct PartPlan {
  const void* sweep_fn = nullptr;
  const void* finish_fn = nullptr;
  int32_t a4 = 4, b = 4;
  int ctas = 1;        // sweep CTAs per replica (32 chains each)
  int chains = 32;     // per replica on this device (one per warp)
  int tail = 0;        // global tail chunks (exact counter) per sweep, one device
  int tail_multi = 0;  // the same when the graph is partitioned over ranks
  int cta_tail = 4;    // chains per CTA deferring their last chunk to the CTA tail
  int block = 1024;    // sweep CTA: 32 x warps threads
  int warps = 32;      // sweep CTA warps: chains + the refresher
  int fin_block = 1024;
  int fin_grid = 1;    // finishing CTAs per replica
  int nwp = 0;         // spin words per replica (part_words)
  int smem = 0;        // dynamic shared memory of the sweep kernel (the spin copy)
  int fin_smem = 0;    // dynamic shared memory of the finishing kernel (0: lookups through L1)
  long long m_main = 0, m_main_multi = 0;  // position-space edges between main vertices (tail / tail_multi)
  int mcast = 1;       // sweep CTAs per cluster sharing the initial copy (part_plan_mcast)
  bool smem_copy = false;
  int refresh = 1;     // 1: a refresher warp keeps re-copying the shared spin copy (0: never)
  int fresh = 0;       // 1: the last two bands of chunks read from the global words (k4_sweep SMODE 2)
  const char* name = "";
};
int part_plan(const GraphStats& st, int wkind, int32_t replicas, int64_t a4, int64_t b, PartPlan* plan);
// plan->mcast for the plan's sweep grid (after any change of ctas / block)
void part_plan_mcast(PartPlan* plan, int replicas);
// Enqueues init + sweeps x (sweep, finish) kernels: 1 + 2 * sweeps launches.
// spins_out [R][n] receives the final spins in vertex order.
cudaError_t part_launch(const PartPlan& plan, const PartArgs& args, int8_t* spins_out, cudaStream_t stream);
// The same sequence in pieces, for the vertex-partitioned multi-rank driver:
// init; per sweep: sweep (args.send = this sweep's send buffer), [caller
// all-gathers the send buffers], finish (recv = the gathered buffers).
cudaError_t part_init_launch(const PartPlan& plan, const PartArgs& args, cudaStream_t stream);
cudaError_t part_sweep_launch(const PartPlan& plan, const PartArgs& args, int sweep, cudaStream_t stream);
cudaError_t part_finish_launch(const PartPlan& plan, const PartArgs& args, int sweep, const void* recv,
                               long long stride, int8_t* spins_out, cudaStream_t stream);
long long part_exchange_bytes(int n, int world, bool peer);  // per-rank send buffer bytes (16-aligned)
int part_launch_count(const PartPlan& plan, int32_t sweeps);
int part_words(int n);  // spin words per replica: ceil(n/32) + 1 zero word, padded to 4

// L2-resident read bandwidth (GB/s) for roofline denominators.
cudaError_t probe_l2_read(size_t bytes, int iters, double* gbs);

// K3 fused exact evaluation (k3_eval.cu): {cut, spin sum} per replica
// into a zeroed buffer. wkind: 0 unit, 1 +-1, 2 general weights. The
// bit-packed path needs eval_work_words(...) words of scratch in args.work.
bool eval_sliced(int n, int replicas, int wkind);
long long eval_work_words(int n, int replicas, int wkind);
cudaError_t eval_launch(EvalArgs args, int wkind, cudaStream_t stream, int* launches);

}  // namespace gdi
