// C ABI of libgdi (include/gdi.h): graph upload, sessions, batch anneal and
// fused evaluation. Everything here is host code around the sm_100a kernels
// in k1_exact.cu / k2_throughput.cu / k3_eval.cu.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "devbuf.hpp"
#include "host/parallel.hpp"
#include "gdi.h"
#include "kernels.cuh"
#include "launch.hpp"
#include "layout.hpp"

namespace {
// NVTX range over a host-side phase (upload, launch, fetch show
// up by name in nsys / ncu --nvtx timelines); header-only NVTX 3, no library.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

using namespace gdi;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(GDI_ERR_RUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
}

#define GDI_CUDA(call)                                 \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

// Selects the device and checks it is a Blackwell (sm_100) part: the
// kernels are compiled for sm_100a only and there is no fallback.
int use_device(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(GDI_ERR_RUNTIME, "no CUDA device available (gdi-b200 has no CPU fallback)");
  if (device < 0 || device >= count)
    return fail(GDI_ERR_CONFIG, "device index " + std::to_string(device) + " out of range");
  GDI_CUDA(cudaSetDevice(device));
  int major = 0;
  GDI_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major != 10) return fail(GDI_ERR_RUNTIME, "gdi-b200 kernels require an sm_100 (B200) device");
  // keep freed pool memory cached across sessions (see devbuf.hpp)
  static std::once_flag pool_once[64];
  if (device < 64)
    std::call_once(pool_once[device], [device]() {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        unsigned long long keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
    });
  return GDI_OK;
}

}  // namespace

struct gdi_graph {
  int device = 0;
  GraphStats st;
  DevBuf off, col, w;
  int wkind = 0;  // 0 unit, 1 +-1 (sign bit), 2 general
  // kernel layouts, built on the device the first time a session needs one
  std::mutex mu;
  bool thru_built = false, pipe_built = false, part_built = false, eval_built = false, brow_built = false;
  ThruLayout thru;   // K2/K4: degree-binned order, SELL-32 rows, edge list
  DevBuf psell, pdeg, pedges, pedge_w;  // K4: SELL rows over visit-order positions, degree by position, edges by position
  PipeLayout pipel;  // k1_window: window masks, forward masks, SELL rows
  PipeGraph pipe;    // k1_window view (ok = eligible; pointers once built)
  EvalLayout evl;    // K3: canonical edge list
  DevBuf brow;       // k1_block row records (rows variant)
  DevCsr csr() const { return DevCsr{off.as<int32_t>(), col.as<int32_t>(), st.unit ? nullptr : w.as<int32_t>(), st.n}; }
  int64_t bytes() const {
    return static_cast<int64_t>(off.bytes + col.bytes + w.bytes + thru.order.bytes + thru.sell.bytes +
                                thru.sell_off.bytes + thru.sell_w.bytes + thru.edges.bytes + thru.edge_w.bytes + thru.poff.bytes + thru.pcol.bytes + thru.ppos.bytes + psell.bytes + pdeg.bytes + pedges.bytes + pedge_w.bytes +
                                pipel.win_pos.bytes +
                                pipel.win_neg.bytes + pipel.fwd_pos.bytes + pipel.fwd_neg.bytes + pipel.wsell.bytes +
                                pipel.wsell_off.bytes + evl.edges.bytes + evl.w.bytes + brow.bytes);
  }
};

struct gdi_session {
  const gdi_graph* g = nullptr;
  gdi_params p{};
  int32_t replicas = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ExactPlan plan;
  BlockPlan bplan;
  PipePlan pplan;
  ThruPlan tplan;
  PartPlan kplan;
  bool use_block = false;  // k1_block (exact mode default)
  bool use_win = false;  // k1_window (pplan)
  bool use_thru = false;
  bool use_part = false;
  cudaGraphExec_t part_exec = nullptr;  // k4: 1 + 2M launches replayed as one graph
  std::vector<double> pf;        // flip probability per sweep (iterated product)
  std::vector<long long> thr;    // integer flip threshold per sweep
  std::vector<unsigned long long> tmask;  // thr * 2^11 + 2047, saturated
  DevBuf seeds, thr_d, tmask_d, spins, trace, stamps, snaps, final_out, watchdog, prof, gspins;
  DevBuf live, gsum, gdelta, acc, done, finished;  // k4 state (live: position-space spin words)
  DevTrace* tr = nullptr;              // trace records: s->trace, or pinned host memory
  unsigned long long* st = nullptr;    // sweep timestamps: s->stamps, or pinned host memory
  bool host_trace = false;             // one-shot batch: kernels write the trace straight to the host
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool launched = false;
  ~gdi_session() {
    if (part_exec) cudaGraphExecDestroy(part_exec);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
};

namespace {

// AnnealParams::validated() (reference anneal.cpp:24-37) plus the coefficient
// sanity of MinCutProblem::make_unchecked (model.cpp:76-82).
int check_params(const gdi_params* p) {
  if (!p) return fail(GDI_ERR_CONFIG, "params is NULL");
  if (p->sweeps < 1) return fail(GDI_ERR_CONFIG, "sweeps must be >= 1");
  if (!(p->flip_fraction0 >= 0.0 && p->flip_fraction0 <= 1.0))
    return fail(GDI_ERR_CONFIG, "flip_fraction0 must be in [0, 1]");
  if (!(p->decay_rate > 0.0 && p->decay_rate < 1.0))
    return fail(GDI_ERR_CONFIG, "decay_rate must be in (0, 1)");
  if (p->strategy != GDI_STRATEGY_GDI && p->strategy != GDI_STRATEGY_STANDARD)
    return fail(GDI_ERR_CONFIG, "unknown strategy");
  if (p->mode != GDI_MODE_EXACT && p->mode != GDI_MODE_THROUGHPUT)
    return fail(GDI_ERR_CONFIG, "unknown mode");
  if (p->a_num <= 0 || p->b_num <= 0 || p->denom <= 0)
    return fail(GDI_ERR_CONFIG, "coefficients must be positive");
  return GDI_OK;
}

// pf_k by the reference's iterated product (anneal.cpp:183, :39-45) and the
// exactly equivalent integer threshold on the 53-bit draw:
//   (x>>11) * 2^-53 <= pf  <=>  (x>>11) <= floor(pf * 2^53)   (pf > 0)
// The pipe kernel tests the raw draw directly: (x >> 11) <= T  <=>
// x <= T*2^11 + 2047, with T clamped to 2^53 - 1 (x >> 11 never exceeds it).
void schedule(const gdi_params& p, std::vector<double>& pf, std::vector<long long>& thr,
              std::vector<unsigned long long>& tmask) {
  pf.resize(p.sweeps);
  thr.resize(p.sweeps);
  tmask.resize(p.sweeps);
  double v = p.flip_fraction0;
  for (int k = 0; k < p.sweeps; k++) {
    pf[k] = v;
    thr[k] = v > 0.0 ? static_cast<long long>(std::floor(std::ldexp(v, 53))) : -1LL;
    const unsigned long long t = thr[k] < 0 ? 0ull : std::min<unsigned long long>(thr[k], (1ull << 53) - 1);
    tmask[k] = (t << 11) | 2047ull;
    v *= p.decay_rate;
  }
}

// Lazy layout builders (layout.cu), serialised per graph.
int ensure_thru(gdi_graph* g) {
  std::lock_guard<std::mutex> lock(g->mu);
  if (g->thru_built) return GDI_OK;
  cudaStream_t st = nullptr;
  GDI_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const cudaError_t e = build_thru_layout(g->csr(), g->st.m, g->wkind, &g->thru, st);
  cudaStreamDestroy(st);
  if (e == cudaErrorInvalidValue) return fail(GDI_ERR_CAPACITY, "SELL layout exceeds 2^31 entries");
  GDI_CUDA(e);
  g->thru_built = true;
  return GDI_OK;
}

// K4 rows over positions (after ensure_thru)
int ensure_part(gdi_graph* g) {
  int rc = ensure_thru(g);
  if (rc) return rc;
  std::lock_guard<std::mutex> lock(g->mu);
  if (g->part_built) return GDI_OK;
  cudaStream_t st = nullptr;
  GDI_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const cudaError_t e = build_part_layout(g->csr(), g->thru, g->st.m, g->wkind, g->psell, g->pdeg, g->pedges, g->pedge_w, st);
  cudaStreamDestroy(st);
  GDI_CUDA(e);
  g->part_built = true;
  return GDI_OK;
}

// K4 plan: the edges between main vertices for both tail lengths
int part_splits(const gdi_graph* g, PartPlan* plan) {
  const int nck = (g->st.n + 31) / 32;
  GDI_CUDA(part_edges_below(g->pedges, g->st.m, 32 * (nck - plan->tail), &plan->m_main));
  GDI_CUDA(part_edges_below(g->pedges, g->st.m, 32 * (nck - plan->tail_multi), &plan->m_main_multi));
  return GDI_OK;
}

// k1_block row records
int ensure_brow(gdi_graph* g) {
  std::lock_guard<std::mutex> lock(g->mu);
  if (g->brow_built) return GDI_OK;
  cudaStream_t st = nullptr;
  GDI_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const cudaError_t e = build_block_rows(g->csr(), g->brow, st);
  cudaStreamDestroy(st);
  GDI_CUDA(e);
  g->brow_built = true;
  return GDI_OK;
}

// K3 edge list
int ensure_eval(gdi_graph* g) {
  std::lock_guard<std::mutex> lock(g->mu);
  if (g->eval_built) return GDI_OK;
  cudaStream_t st = nullptr;
  GDI_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const cudaError_t e = build_eval_layout(g->csr(), g->st.m, g->wkind, &g->evl, st);
  cudaStreamDestroy(st);
  GDI_CUDA(e);
  g->eval_built = true;
  return GDI_OK;
}

int ensure_pipe(gdi_graph* g) {
  std::lock_guard<std::mutex> lock(g->mu);
  if (g->pipe_built) return GDI_OK;
  cudaStream_t st = nullptr;
  GDI_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const cudaError_t e = build_pipe_layout(g->csr(), pipe_window(), &g->pipel, st);
  cudaStreamDestroy(st);
  GDI_CUDA(e);
  g->pipe.win_pos = g->pipel.win_pos.as<uint32_t>();
  g->pipe.win_neg = g->pipel.win_neg.as<uint32_t>();
  g->pipe.fwd_pos = g->pipel.fwd_pos.as<uint32_t>();
  g->pipe.fwd_neg = g->pipel.fwd_neg.as<uint32_t>();
  g->pipe.wsell = g->pipel.wsell.as<int32_t>();
  g->pipe.wsell_off = g->pipel.wsell_off.as<int32_t>();
  g->pipe_built = true;
  return GDI_OK;
}

const char* forced_kernel() {
  const char* e = std::getenv("GDI_FORCE_KERNEL");
  return e ? e : "";
}

}  // namespace

extern "C" {

int gdi_abi_version(void) { return GDI_ABI_VERSION; }

const char* gdi_last_error(void) { return g_last_error.c_str(); }

int gdi_device_count(int* count) {
  if (!count) return fail(GDI_ERR_CONFIG, "count is NULL");
  *count = 0;
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  return GDI_OK;
}

}  // extern "C"

namespace {

// graph.cpp:47-61 invariants on the host, before any device work, so that a
// bad CSR is a domain error on every machine (the statistics come from the
// device pass). Rows are split over host threads for large graphs.
// Host validation of the caller's CSR (domain errors come before any device
// work). With stage != nullptr the same row-parallel pass copies offsets,
// adjacency (stride 1 or 2 int32 per entry) and weights into the pinned
// staging buffer (layout: offsets | adjacency | weights), so the upload runs
// at link speed instead of the driver's pageable staging.
int validate_host(int32_t n, const int64_t* offsets, const int32_t* nbr, int stride, const int32_t* weights = nullptr,
                  char* stage = nullptr) {
  const int64_t nnz = offsets[n];
  int64_t* st_off = reinterpret_cast<int64_t*>(stage);
  int32_t* st_adj = stage ? reinterpret_cast<int32_t*>(stage + (static_cast<size_t>(n) + 1) * 8) : nullptr;
  int32_t* st_w = stage ? st_adj + static_cast<size_t>(nnz) * stride : nullptr;
  auto rows = [&](int32_t lo, int32_t hi) -> int {
    for (int32_t i = lo; i < hi; i++) {
      const int64_t o0 = offsets[i], o1 = offsets[i + 1];
      // bounds before any adjacency read or staging copy: a monotone prefix
      // that overshoots nnz must not read past the caller's arrays
      if (o1 < o0 || o0 < 0 || o1 > nnz) return 1;
      for (int64_t e = o0; e < o1; e++) {
        const int32_t v = nbr[e * stride];
        if (v < 0 || v >= n) return 2;
        if (v == i) return 3;
      }
    }
    if (stage) {  // rows valid, so offsets[lo] <= offsets[hi] <= nnz
      const int64_t e0 = offsets[lo], e1 = offsets[hi];
      std::memcpy(st_off + lo, offsets + lo, static_cast<size_t>(hi - lo + (hi == n ? 1 : 0)) * 8);
      std::memcpy(st_adj + e0 * stride, nbr + e0 * stride, static_cast<size_t>(e1 - e0) * stride * 4);
      if (weights) std::memcpy(st_w + e0, weights + e0, static_cast<size_t>(e1 - e0) * 4);
    }
    return 0;
  };
  // rows are split evenly; below ~1M adjacency entries one thread does it all
  const size_t min_rows = nnz < (1 << 20) ? static_cast<size_t>(n) + 1 : 0;
  std::vector<int> codes(16, 0);
  std::atomic<unsigned> slot{0};
  parallel_rows(static_cast<size_t>(n), min_rows, [&](size_t lo, size_t hi) {
    codes[slot.fetch_add(1)] = rows(static_cast<int32_t>(lo), static_cast<int32_t>(hi));
  });
  for (int c : codes) {
    if (c == 1) return fail(GDI_ERR_DOMAIN, "offsets not monotone");
    if (c == 2) return fail(GDI_ERR_DOMAIN, "edge endpoint out of range");
    if (c == 3) return fail(GDI_ERR_DOMAIN, "self-loop");
  }
  return GDI_OK;
}

// nbr/weights (separate arrays) or pairs (interleaved {node, weight}).
int create_graph(int device, int32_t n, const int64_t* offsets, const int32_t* nbr, const int32_t* weights,
                 const int32_t* pairs, gdi_graph** out) {
  NvtxRange nvtx_range("gdi_graph_create");
  if (!out) return fail(GDI_ERR_CONFIG, "out is NULL");
  *out = nullptr;
  if (n <= 0) return fail(GDI_ERR_DOMAIN, "graph needs a positive node count");
  if (!offsets) return fail(GDI_ERR_DOMAIN, "offsets is NULL");
  const int64_t nnz = offsets[n];
  if (offsets[0] != 0 || nnz < 0 || (nnz % 2) != 0)
    return fail(GDI_ERR_DOMAIN, "offsets must start at 0 and hold an even entry count");
  if (nnz > 0x7fffffffLL) return fail(GDI_ERR_CAPACITY, "more than 2^31-1 adjacency entries");
  if (nnz > 0 && !(pairs ? pairs : nbr)) return fail(GDI_ERR_DOMAIN, "adjacency is NULL");
  const bool timing = std::getenv("GDI_TIMING") != nullptr;  // phase times on stderr (tuning)
  const auto t0 = std::chrono::steady_clock::now();
  auto ms = [&]() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
  // large graphs: validated and staged into pinned memory in one pass
  // (pinned allocation is host-only; the device is touched after validation)
  const int stride = pairs ? 2 : 1;
  const size_t stage_bytes = (static_cast<size_t>(n) + 1) * 8 + static_cast<size_t>(nnz) * stride * 4 +
                             (weights && !pairs ? static_cast<size_t>(nnz) * 4 : 0);
  thread_local PinnedBuf upload_stage;
  char* stage = nullptr;
  if (nnz >= (1 << 20) && upload_stage.ensure(stage_bytes) == cudaSuccess) stage = upload_stage.as<char>();
  int rc = validate_host(n, offsets, pairs ? pairs : nbr, stride, pairs ? nullptr : weights, stage);
  if (rc) return rc;
  if (stage) {  // upload from the staged copy
    const int64_t* so = reinterpret_cast<const int64_t*>(stage);
    const int32_t* sa = reinterpret_cast<const int32_t*>(stage + (static_cast<size_t>(n) + 1) * 8);
    offsets = so;
    if (pairs)
      pairs = sa;
    else
      nbr = sa;
    if (weights && !pairs) weights = sa + static_cast<size_t>(nnz);
  }
  const double t_val = ms();

  auto g = std::make_unique<gdi_graph>();
  g->device = device;
  g->st.n = n;
  g->st.m = nnz / 2;
  if ((rc = use_device(device))) return rc;
  // upload + validation + statistics on the device (layout.cu)
  GraphScan scan{};
  cudaStream_t st = nullptr;
  GDI_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const double t_dev = ms();
  const cudaError_t ue = upload_and_scan(offsets, nbr, weights, pairs, n, nnz, g->off, g->col, g->w, &scan, st);
  cudaStreamDestroy(st);
  GDI_CUDA(ue);
  if (timing)
    std::fprintf(stderr, "[gdi_graph_create] validate %.2f ms, device setup %.2f ms, upload+scan %.2f ms\n", t_val,
                 t_dev - t_val, ms() - t_dev);
  if (scan.bad & 1u) return fail(GDI_ERR_DOMAIN, "offsets not monotone");
  if (scan.bad & 2u) return fail(GDI_ERR_DOMAIN, "edge endpoint out of range");
  if (scan.bad & 4u) return fail(GDI_ERR_DOMAIN, "self-loop");
  g->st.unit = !(weights || pairs) || !scan.non_unit;
  g->st.max_abs_field = static_cast<long long>(scan.max_abs_field);
  g->st.max_degree = scan.max_degree;
  g->wkind = g->st.unit ? 0 : (!scan.non_pm1 ? 1 : 2);
  g->st.pm1 = g->wkind <= 1;
  // k1_window eligibility (every |w| == 1, n >= 2L); its layout is built lazily
  g->pipe.ok = n >= 2 * pipe_window() && (g->st.unit || !scan.non_pm1);
  g->pipe.n_words = (n + 1 + 3) & ~3;
  *out = g.release();
  return GDI_OK;
}

}  // namespace

extern "C" {

int gdi_graph_create(int device, int32_t n, const int64_t* offsets, const int32_t* nbr, const int32_t* weights,
                     gdi_graph** out) {
  return create_graph(device, n, offsets, nbr, weights, nullptr, out);
}

int gdi_graph_create_pairs(int device, int32_t n, const int64_t* offsets, const int32_t* pairs, gdi_graph** out) {
  return create_graph(device, n, offsets, nullptr, nullptr, pairs, out);
}

int gdi_graph_destroy(gdi_graph* g) {
  if (g) {
    cudaSetDevice(g->device);
    delete g;
  }
  return GDI_OK;
}

int gdi_graph_query(const gdi_graph* g, gdi_graph_info* info) {
  if (!g || !info) return fail(GDI_ERR_CONFIG, "NULL argument");
  info->n = g->st.n;
  info->m = g->st.m;
  info->max_degree = g->st.max_degree;
  info->device = g->device;
  info->all_unit_weights = g->st.unit ? 1 : 0;
  info->device_bytes = g->bytes();
  return GDI_OK;
}

}  // extern "C"

namespace {

// Pinned, device-mapped trace staging, one per host thread, reused across
// calls (one-shot batches create a session per call). Sessions that
// gdi_anneal_batch creates write their trace records straight into it over
// PCIe while the kernel runs (~32 B per replica-sweep, far below link rate),
// so no trace copy is left for after the kernel.
PinnedBuf& trace_stage() {
  thread_local PinnedBuf stage;
  return stage;
}

int session_create(const gdi_graph* g, const gdi_params* p, int32_t replicas, void* stream, gdi_session** out,
                   bool host_trace);

}  // namespace

extern "C" {

int gdi_session_create(const gdi_graph* g, const gdi_params* p, int32_t replicas, void* stream,
                       gdi_session** out) {
  return session_create(g, p, replicas, stream, out, false);
}

}  // extern "C"

namespace {

int session_create(const gdi_graph* g, const gdi_params* p, int32_t replicas, void* stream, gdi_session** out,
                   bool host_trace) {
  NvtxRange nvtx_range("gdi_session_create");
  if (!out) return fail(GDI_ERR_CONFIG, "out is NULL");
  *out = nullptr;
  if (!g) return fail(GDI_ERR_CONFIG, "graph is NULL");
  int rc = check_params(p);
  if (rc) return rc;
  if (replicas < 1) return fail(GDI_ERR_CONFIG, "replicas must be >= 1");
  if ((rc = use_device(g->device))) return rc;

  auto s = std::make_unique<gdi_session>();
  s->g = g;
  s->p = *p;
  s->replicas = replicas;
  schedule(s->p, s->pf, s->thr, s->tmask);
  // Both strategies coincide in the exact mode (reference acceptance.cpp
  // criterion 8).
  const std::string force = forced_kernel();
  // THROUGHPUT: the racy pooled-mode kernel. Any exact-mode result is also a
  // legal outcome of the racy contract (one worker claiming every chunk), so
  // the exact kernels serve as its fallback when k2 does not apply.
  // K2 (one warp per replica, spins in shared memory) when it fits and either
  // the replicas fill the GPU or the graph is small; else K4 (vertex-
  // partitioned chains, spins in L2/HBM). K4 keeps ~P*32 vertices in flight
  // at once: harmless on large graphs (1M: cut within 0.3% of the sequential
  // run) but a large fraction of a small one, where lattices (torus) then
  // degrade as under Jacobi updates.
  const bool thru_ok = p->mode == GDI_MODE_THROUGHPUT && force != "exact" && force.rfind("window", 0) != 0 &&
                       force != "block";
  // (the literal `standard` strategy only exists in K2: its O(n) traversal per
  // visit needs the replica's spins on chip)
  if (thru_ok && force != "part" &&
      (replicas >= 148 || g->st.n <= 32768 || p->strategy == GDI_STRATEGY_STANDARD) &&
      thru_plan(g->st, g->wkind, replicas, 4 * p->a_num, p->b_num, p->strategy == GDI_STRATEGY_STANDARD, &s->tplan) == 0)
    s->use_thru = true;
  else if (thru_ok && part_plan(g->st, g->wkind, replicas, 4 * p->a_num, p->b_num, &s->kplan) == 0)
    s->use_part = s->use_thru = true;
  else if (thru_ok && force != "part" &&
           thru_plan(g->st, g->wkind, replicas, 4 * p->a_num, p->b_num, p->strategy == GDI_STRATEGY_STANDARD, &s->tplan) == 0)
    s->use_thru = true;
  // K2 without concurrent chains (one chain per replica on small graphs such
  // as G1, or the one-warp-per-replica k2_sweep where k2_chains does not fit,
  // e.g. G81) is one serial decision chain per replica, like the exact mode,
  // and slower than the exact kernels' windows (G1: 14.9 vs 9.9 ms, G81+-1:
  // 599 vs 485 ms for 1024 replicas x 1000 sweeps): use the exact kernel,
  // whose sequential result is a legal outcome of the racy contract
  if (s->use_thru && !s->use_part && (force.empty() || force == "auto") && p->strategy != GDI_STRATEGY_STANDARD &&
      !(s->tplan.chains && s->tplan.cfg.chains >= 2)) {
    if (block_plan(g->st, replicas, 4 * p->a_num, p->b_num, p->sweeps, &s->bplan) == 0)
      s->use_block = true;
    else if (window_plan(g->st, g->pipe, replicas, 4 * p->a_num, p->b_num, p->sweeps, &s->pplan) == 0)
      s->use_win = true;
    if (s->use_block || s->use_win) s->use_thru = false;
  }
  // exact mode: k1_block (fixed-point windows) by default; k1_window
  // (speculative windows) where k1_block does not fit (graphs whose CSR does
  // not fit shared memory, e.g. G81); k1_exact for everything else
  // (GDI_FORCE_KERNEL=block|window|exact picks one for tests)
  if (!s->use_thru && (force.empty() || force == "auto" || force == "block") &&
      block_plan(g->st, replicas, 4 * p->a_num, p->b_num, p->sweeps, &s->bplan) == 0)
    s->use_block = true;
  if (force == "block" && !s->use_block)
    return fail(GDI_ERR_CAPACITY, "GDI_FORCE_KERNEL=block but k1_block does not apply");
  if (!s->use_block && !s->use_thru && force != "exact" &&
      window_plan(g->st, g->pipe, replicas, 4 * p->a_num, p->b_num, p->sweeps, &s->pplan) == 0)
    s->use_win = true;
  if (force.rfind("window", 0) == 0 && !s->use_win)
    return fail(GDI_ERR_CAPACITY, "GDI_FORCE_KERNEL=window but k1_window does not apply");
  if (!s->use_thru && !s->use_block && !s->use_win && exact_plan(g->st, replicas, &s->plan))
    return fail(GDI_ERR_CAPACITY, "graph too large for the exact kernel's shared-memory spins");
  gdi_graph* gm = const_cast<gdi_graph*>(g);  // layouts are a lazily built cache
  if (s->use_thru && (rc = ensure_thru(gm))) return rc;
  if (s->use_part && ((rc = ensure_part(gm)) || (rc = part_splits(gm, &s->kplan)))) return rc;
  if (s->use_win && (rc = ensure_pipe(gm))) return rc;
  if (s->use_block && s->bplan.rows && (rc = ensure_brow(gm))) return rc;

  if (stream) {
    s->stream = static_cast<cudaStream_t>(stream);
  } else {
    GDI_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    s->own_stream = true;
  }
  GDI_CUDA(cudaEventCreate(&s->ev0));
  GDI_CUDA(cudaEventCreate(&s->ev1));
  const size_t R = replicas, n = g->st.n, S = p->sweeps;
  GDI_CUDA(s->seeds.alloc(R * sizeof(uint64_t)));
  GDI_CUDA(s->thr_d.alloc(S * sizeof(long long)));
  GDI_CUDA(s->tmask_d.alloc(S * sizeof(unsigned long long)));
  GDI_CUDA(s->spins.alloc(R * n));
  GDI_CUDA(s->final_out.alloc(R * sizeof(DevTrace)));
  GDI_CUDA(s->watchdog.alloc(8 * sizeof(int)));
  GDI_CUDA(s->prof.alloc(16 * sizeof(unsigned long long)));
  if (s->use_win && s->pplan.gw)
    GDI_CUDA(s->gspins.alloc(static_cast<size_t>(replicas) * s->pplan.n_words));
  if (p->flags & GDI_FLAG_TRACE) {
    const size_t tb = R * S * sizeof(DevTrace), sb = R * (S + 1) * sizeof(unsigned long long);
    if (host_trace) {
      PinnedBuf& stage = trace_stage();
      GDI_CUDA(stage.ensure(tb + sb));
      void* d = nullptr;
      GDI_CUDA(cudaHostGetDevicePointer(&d, stage.p, 0));
      s->tr = static_cast<DevTrace*>(d);
      s->st = reinterpret_cast<unsigned long long*>(static_cast<char*>(d) + tb);
      s->host_trace = true;
    } else {
      GDI_CUDA(s->trace.alloc(tb));
      GDI_CUDA(s->stamps.alloc(sb));
      s->tr = s->trace.as<DevTrace>();
      s->st = s->stamps.as<unsigned long long>();
    }
  }
  if (p->flags & GDI_FLAG_SNAPSHOTS) GDI_CUDA(s->snaps.alloc(R * (S + 1) * n));
  if (s->use_part) {
    GDI_CUDA(s->live.alloc(R * part_words(g->st.n) * sizeof(uint32_t)));
    GDI_CUDA(s->gsum.alloc(R * sizeof(long long)));
    GDI_CUDA(s->gdelta.alloc(R * sizeof(long long)));
    GDI_CUDA(s->acc.alloc(2 * R * sizeof(unsigned long long)));
    GDI_CUDA(s->done.alloc(R * sizeof(unsigned int)));
    GDI_CUDA(s->finished.alloc(R * sizeof(unsigned int)));
  }
  GDI_CUDA(cudaMemcpyAsync(s->thr_d.p, s->thr.data(), S * sizeof(long long),
                           cudaMemcpyHostToDevice, s->stream));
  GDI_CUDA(cudaMemcpyAsync(s->tmask_d.p, s->tmask.data(), S * sizeof(unsigned long long),
                           cudaMemcpyHostToDevice, s->stream));
  GDI_CUDA(cudaStreamSynchronize(s->stream));
  *out = s.release();
  return GDI_OK;
}

}  // namespace

extern "C" {
static int check_watchdog(gdi_session* s);  // defined with the session entry points below
}

namespace {

// gdi_session_fetch, with the trace optionally in column form (cols)
int fetch_impl(gdi_session* s, gdi_outputs* out, const gdi_trace_columns* cols) {
  NvtxRange nvtx_range("gdi_session_fetch");
  if (!s || !out) return fail(GDI_ERR_CONFIG, "NULL argument");
  if (!s->launched) return fail(GDI_ERR_CONFIG, "session has not been launched");
  GDI_CUDA(cudaSetDevice(s->g->device));
  GDI_CUDA(cudaStreamSynchronize(s->stream));
  if (int rc = check_watchdog(s)) return rc;
  const size_t R = s->replicas, n = s->g->st.n, S = s->p.sweeps;
  const long long A = s->p.a_num, B = s->p.b_num;
  const double denom = static_cast<double>(s->p.denom);
  float ms = 0.f;
  GDI_CUDA(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
  out->seconds = ms * 1e-3;
  if (out->spins)
    GDI_CUDA(cudaMemcpy(out->spins, s->spins.p, R * n, cudaMemcpyDeviceToHost));
  if (out->scores) {
    std::vector<DevTrace> fin(R);
    GDI_CUDA(cudaMemcpy(fin.data(), s->final_out.p, R * sizeof(DevTrace), cudaMemcpyDeviceToHost));
    for (size_t r = 0; r < R; r++) {
      const long long sum = fin[r].sum, cut = fin[r].cut;
      gdi_score& sc = out->scores[r];
      sc.cut = cut;
      sc.imbalance = sum < 0 ? -sum : sum;
      sc.hamiltonian_scaled = A * sum * sum + B * cut;
      sc.hamiltonian = static_cast<double>(sc.hamiltonian_scaled) / denom;
      sc.balance_counter = fin[r].counter;
    }
  }
  const bool want_cols = cols != nullptr && (cols->hcut_imb || cols->seconds || cols->flip_probability);
  if (want_cols && cols->flip_probability)
    for (size_t k = 0; k < S; k++) cols->flip_probability[k] = s->pf[k];
  if (out->trace || out->counters || (want_cols && (cols->hcut_imb || cols->seconds))) {
    if (!(s->p.flags & GDI_FLAG_TRACE))
      return fail(GDI_ERR_CONFIG, "trace requested but the session was created without GDI_FLAG_TRACE");
    // pinned staging: the trace is the bulk of a batch's
    // result (24 B per sweep per replica + a timestamp), pageable copies of it
    // cost more than the conversion
    const size_t tb = R * S * sizeof(DevTrace), sb = R * (S + 1) * sizeof(unsigned long long);
    // (one buffer per host thread, reused across sessions: one-shot batches
    // create a session per call)
    PinnedBuf& stage = trace_stage();
    if (!s->host_trace) {  // else the kernels wrote the records there already
      GDI_CUDA(stage.ensure(tb + sb));
      GDI_CUDA(cudaMemcpyAsync(stage.p, s->trace.p, tb, cudaMemcpyDeviceToHost, s->stream));
      GDI_CUDA(cudaMemcpyAsync(stage.as<char>() + tb, s->stamps.p, sb, cudaMemcpyDeviceToHost, s->stream));
      GDI_CUDA(cudaStreamSynchronize(s->stream));
    }
    const DevTrace* tr = stage.as<DevTrace>();
    const unsigned long long* st = reinterpret_cast<const unsigned long long*>(stage.as<char>() + tb);
    parallel_rows(R, 64 * 1024 / (S + 1) + 1, [&](size_t r0, size_t r1) {
    for (size_t r = r0; r < r1; r++)
      for (size_t k = 0; k < S; k++) {
        const DevTrace& d = tr[r * S + k];
        if (out->counters) out->counters[r * S + k] = d.counter;
        if (want_cols) {
          const long long hs = A * d.sum * d.sum + B * d.cut;
          if (cols->hcut_imb) {
            int64_t* c3 = cols->hcut_imb + 3 * (r * S + k);
            c3[0] = hs;
            c3[1] = d.cut;
            c3[2] = d.sum < 0 ? -d.sum : d.sum;
          }
          if (cols->seconds)
            cols->seconds[r * S + k] = static_cast<double>(st[r * (S + 1) + k + 1] - st[r * (S + 1) + k]) * 1e-9;
        }
        if (out->trace) {
          gdi_trace_rec& t = out->trace[r * S + k];
          t.cut = d.cut;
          t.imbalance = d.sum < 0 ? -d.sum : d.sum;
          t.hamiltonian_scaled = A * d.sum * d.sum + B * d.cut;
          t.hamiltonian = static_cast<double>(t.hamiltonian_scaled) / denom;
          t.flip_probability = s->pf[k];
          t.seconds = static_cast<double>(st[r * (S + 1) + k + 1] - st[r * (S + 1) + k]) * 1e-9;
        }
      }
    });
  }
  if (out->snapshots) {
    if (!(s->p.flags & GDI_FLAG_SNAPSHOTS))
      return fail(GDI_ERR_CONFIG, "snapshots requested but the session was created without GDI_FLAG_SNAPSHOTS");
    GDI_CUDA(cudaMemcpy(out->snapshots, s->snaps.p, R * (S + 1) * n, cudaMemcpyDeviceToHost));
  }
  return GDI_OK;
}

}  // namespace

extern "C" {

int gdi_session_set_seeds(gdi_session* s, const uint64_t* seeds) {
  if (!s || !seeds) return fail(GDI_ERR_CONFIG, "NULL argument");
  GDI_CUDA(cudaSetDevice(s->g->device));
  GDI_CUDA(cudaMemcpyAsync(s->seeds.p, seeds, s->replicas * sizeof(uint64_t),
                           cudaMemcpyHostToDevice, s->stream));
  return GDI_OK;
}

int gdi_session_launch(gdi_session* s) {
  NvtxRange nvtx_range("gdi_session_launch");
  if (!s) return fail(GDI_ERR_CONFIG, "session is NULL");
  GDI_CUDA(cudaSetDevice(s->g->device));
  if (s->use_part) {
    if (!s->part_exec) {
      PartArgs a{};
      a.g = s->g->csr();
      a.order = s->g->thru.order.as<int32_t>();
      a.psell = s->g->psell.as<int4>();
      a.pdeg = s->g->pdeg.as<int32_t>();
      a.pedges = s->g->pedges.as<int2>();
      a.pedge_w = s->g->pedge_w.as<int32_t>();
      a.m_edges = s->g->st.m;
      a.sell_off = s->g->thru.sell_off.as<int32_t>();
      a.sell_w = s->g->thru.sell_w.as<int4>();
      a.chains = s->kplan.chains;
      a.world_chains = s->kplan.chains;
      a.chain0 = 0;
      a.chain_stride = 1;
      a.rank = 0;
      a.world = 1;
      a.sweeps = s->p.sweeps;
      a.replicas = s->replicas;
      a.seeds = s->seeds.as<uint64_t>();
      a.thr = s->thr_d.as<long long>();
      a.tmask = s->tmask_d.as<unsigned long long>();
      a.bits = s->live.as<uint32_t>();
      a.gsum = s->gsum.as<long long>();
      a.gdelta = s->gdelta.as<long long>();
      a.acc = s->acc.as<unsigned long long>();
      a.done = s->done.as<unsigned int>();
      a.finished = s->finished.as<unsigned int>();
      a.trace = s->tr;
      a.stamps = s->st;
      a.snaps = s->snaps.as<int8_t>();
      a.final_out = s->final_out.as<DevTrace>();
      a.watchdog = s->watchdog.as<int>();
      cudaGraph_t graph = nullptr;
      GDI_CUDA(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
      const cudaError_t le = part_launch(s->kplan, a, s->spins.as<int8_t>(), s->stream);
      const cudaError_t ce = cudaStreamEndCapture(s->stream, &graph);
      if (le != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        return cuda_fail(le, "part_launch (capture)");
      }
      GDI_CUDA(ce);
      const cudaError_t ie = cudaGraphInstantiate(&s->part_exec, graph, 0);
      cudaGraphDestroy(graph);
      GDI_CUDA(ie);
    }
    GDI_CUDA(cudaMemsetAsync(s->watchdog.p, 0, s->watchdog.bytes, s->stream));
    GDI_CUDA(cudaEventRecord(s->ev0, s->stream));
    GDI_CUDA(cudaGraphLaunch(s->part_exec, s->stream));
    GDI_CUDA(cudaEventRecord(s->ev1, s->stream));
    s->launched = true;
    return GDI_OK;
  }
  if (s->use_thru) {
    ThruArgs a{};
    a.g = s->g->csr();
    a.order = s->g->thru.order.as<int32_t>();
    a.sell = s->g->thru.sell.as<int4>();
    a.sell_off = s->g->thru.sell_off.as<int32_t>();
    a.sell_w = s->g->thru.sell_w.as<int4>();
    a.edges = s->g->thru.edges.as<int2>();
    a.poff = s->g->thru.poff.as<int32_t>();
    a.pcol = s->g->thru.pcol.as<int32_t>();
    a.ppos = s->g->thru.ppos.as<int32_t>();
    a.edge_w = s->g->thru.edge_w.as<int32_t>();
    a.m = s->g->st.m;
    a.sweeps = s->p.sweeps;
    a.replicas = s->replicas;
    a.seeds = s->seeds.as<uint64_t>();
    a.thr = s->thr_d.as<long long>();
    a.tmask = s->tmask_d.as<unsigned long long>();
    a.spins_out = s->spins.as<int8_t>();
    a.trace = s->tr;
    a.stamps = s->st;
    a.snaps = s->snaps.as<int8_t>();
    a.final_out = s->final_out.as<DevTrace>();
    GDI_CUDA(cudaEventRecord(s->ev0, s->stream));
    GDI_CUDA(thru_launch(s->tplan, a, s->stream));
    GDI_CUDA(cudaEventRecord(s->ev1, s->stream));
    s->launched = true;
    return GDI_OK;
  }
  if (s->use_win) {
    PipeArgs a{};
    a.g = s->g->csr();
    a.win_pos = s->g->pipe.win_pos;
    a.win_neg = s->g->pipe.win_neg;
    a.fwd_pos = s->g->pipe.fwd_pos;
    a.fwd_neg = s->g->pipe.fwd_neg;
    a.wsell = s->g->pipe.wsell;
    a.wsell_off = s->g->pipe.wsell_off;
    a.n_words = s->g->pipe.n_words;
    a.gspins = s->pplan.gw ? s->gspins.as<int8_t>() : nullptr;
    a.sweeps = s->p.sweeps;
    a.replicas = s->replicas;
    a.seeds = s->seeds.as<uint64_t>();
    a.thr = s->thr_d.as<long long>();
    a.tmask = s->tmask_d.as<unsigned long long>();
    a.a4 = static_cast<int32_t>(4 * s->p.a_num);
    a.b = static_cast<int32_t>(s->p.b_num);
    a.spins_out = s->spins.as<int8_t>();
    a.trace = s->tr;
    a.stamps = s->st;
    a.snaps = s->snaps.as<int8_t>();
    a.final_out = s->final_out.as<DevTrace>();
    a.watchdog = s->watchdog.as<int>();
    a.prof = s->prof.as<unsigned long long>();
    GDI_CUDA(cudaMemsetAsync(s->watchdog.p, 0, s->watchdog.bytes, s->stream));
    GDI_CUDA(cudaMemsetAsync(s->prof.p, 0, s->prof.bytes, s->stream));
    GDI_CUDA(cudaEventRecord(s->ev0, s->stream));
    GDI_CUDA(window_launch(s->pplan, a, s->stream));
    GDI_CUDA(cudaEventRecord(s->ev1, s->stream));
    s->launched = true;
    return GDI_OK;
  }
  ExactArgs a{};
  a.g = s->g->csr();
  a.brow = s->g->brow.as<uint4>();
  a.n_pad = s->plan.n_pad;
  a.sweeps = s->p.sweeps;
  a.replicas = s->replicas;
  a.seeds = s->seeds.as<uint64_t>();
  a.thr = s->thr_d.as<long long>();
  a.tmask = s->tmask_d.as<unsigned long long>();
  a.a4 = 4 * s->p.a_num;
  a.b = s->p.b_num;
  a.spins_out = s->spins.as<int8_t>();
  a.trace = s->tr;
  a.stamps = s->st;
  a.snaps = s->snaps.as<int8_t>();
  a.final_out = s->final_out.as<DevTrace>();
  GDI_CUDA(cudaEventRecord(s->ev0, s->stream));
  GDI_CUDA(s->use_block ? block_launch(s->bplan, a, s->stream) : exact_launch(s->plan, a, s->stream));
  GDI_CUDA(cudaEventRecord(s->ev1, s->stream));
  s->launched = true;
  return GDI_OK;
}

// A stalled k1_window producer/consumer pipeline aborts itself (watchdog)
// instead of hanging; surface that as a runtime error rather than returning
// wrong results.
static int check_watchdog(gdi_session* s) {
  if (s->use_part) {  // k4 has no inter-warp waits; debug counters only
    if (std::getenv("GDI_K4_DEBUG")) {
      int d[8] = {0};
      GDI_CUDA(cudaMemcpy(d, s->watchdog.p, sizeof d, cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "[k4 debug] %d %d %d %d %d %d %d %d\n", d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7]);
    }
    return GDI_OK;
  }
  if (!s->use_win) return GDI_OK;
  if (std::getenv("GDI_PIPE_DEBUG") && (std::atoi(std::getenv("GDI_PIPE_DEBUG")) & 4)) {
    unsigned long long c[16] = {0};
    GDI_CUDA(cudaMemcpy(c, s->prof.p, sizeof c, cudaMemcpyDeviceToHost));
    const double st = c[0] ? static_cast<double>(c[0]) : 1.0;
    std::fprintf(stderr, "[k1_window prof] steps %llu, visits/step %.2f, cycles/step %.0f (refill %.0f, draw wait %.0f)\n",
                 c[0], c[1] / st, c[3] / st, c[2] / st, c[4] / st);
  }
  int w[8] = {0};
  GDI_CUDA(cudaMemcpy(w, s->watchdog.p, sizeof w, cudaMemcpyDeviceToHost));
  if (w[0] != 0)
    return fail(GDI_ERR_RUNTIME, "k1_window watchdog fired: stage " + std::to_string(w[0]) + " block " +
                                     std::to_string(w[1]) + " thread " + std::to_string(w[2]) + " (" +
                                     std::to_string(w[3]) + ", " + std::to_string(w[4]) + ")");
  return GDI_OK;
}

int gdi_session_sync(gdi_session* s) {
  if (!s) return fail(GDI_ERR_CONFIG, "session is NULL");
  GDI_CUDA(cudaSetDevice(s->g->device));
  GDI_CUDA(cudaStreamSynchronize(s->stream));
  return check_watchdog(s);
}

int gdi_session_fetch(gdi_session* s, gdi_outputs* out) { return fetch_impl(s, out, nullptr); }

int gdi_session_launch_count(const gdi_session* s, int32_t* count) {
  if (!s || !count) return fail(GDI_ERR_CONFIG, "NULL argument");
  *count = s->use_part ? part_launch_count(s->kplan, s->p.sweeps) : 1;
  return GDI_OK;
}

const char* gdi_session_kernel(const gdi_session* s) {
  if (!s) return "";
  if (s->use_part) return s->kplan.name;
  if (s->use_thru) return s->tplan.name;
  if (s->use_block) return s->bplan.name;
  return s->use_win ? s->pplan.name : s->plan.name;
}

int gdi_session_destroy(gdi_session* s) {
  if (s) {
    cudaSetDevice(s->g->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    delete s;
  }
  return GDI_OK;
}

int gdi_anneal_batch(const gdi_graph* g, const gdi_params* p, const uint64_t* seeds,
                     int32_t replicas, gdi_outputs* out) {
  return gdi_anneal_batch_columns(g, p, seeds, replicas, out, nullptr);
}

int gdi_anneal_batch_columns(const gdi_graph* g, const gdi_params* p, const uint64_t* seeds, int32_t replicas,
                             gdi_outputs* out, const gdi_trace_columns* cols) {
  if (!seeds || !out || !p) return fail(GDI_ERR_CONFIG, "NULL argument");
  gdi_params q = *p;
  gdi_outputs o = *out;
  if (cols) o.trace = nullptr, o.counters = nullptr;  // the columns replace the records
  if (o.trace || o.counters || (cols && (cols->hcut_imb || cols->seconds))) q.flags |= GDI_FLAG_TRACE;
  if (out->snapshots) q.flags |= GDI_FLAG_SNAPSHOTS;
  gdi_session* s = nullptr;
  // trace written by the kernels straight into pinned host memory (fetched from there below)
  int rc = session_create(g, &q, replicas, nullptr, &s, (q.flags & GDI_FLAG_TRACE) != 0);
  if (rc) return rc;
  std::unique_ptr<gdi_session, int (*)(gdi_session*)> guard(s, gdi_session_destroy);
  if ((rc = gdi_session_set_seeds(s, seeds))) return rc;
  if ((rc = gdi_session_launch(s))) return rc;
  if ((rc = gdi_session_sync(s))) return rc;
  rc = fetch_impl(s, &o, cols);
  out->seconds = o.seconds;
  return rc;
}

// K3 on device-resident spins: scratch + {cut, spin sum} + bad flag in one
// pool allocation, results into d_out (cut, sum) per replica. Asynchronous on
// `st` when the graph's edge list is already built.
namespace {
struct EvalScratch {
  DevBuf buf;
  size_t out_off = 0, bad_off = 0, work_off = 0;
};
int eval_enqueue(gdi_graph* g, const int8_t* d_spins, int32_t R, EvalScratch& sc, cudaStream_t st, int* launches) {
  int rc = ensure_eval(g);
  if (rc) return rc;
  const long long ww = eval_work_words(g->st.n, R, g->wkind);
  sc.out_off = 0;
  sc.bad_off = static_cast<size_t>(R) * 16;
  sc.work_off = (sc.bad_off + 4 + 15) & ~static_cast<size_t>(15);
  const size_t bytes = sc.work_off + static_cast<size_t>(ww) * 4;
  if (sc.buf.bytes < bytes) GDI_CUDA(sc.buf.alloc(bytes));
  char* base = sc.buf.as<char>();
  GDI_CUDA(cudaMemsetAsync(base, 0, sc.work_off, st));
  EvalArgs a{};
  a.n = g->st.n;
  a.m = g->evl.m;
  a.mpos = g->evl.mpos;
  a.narrow = g->evl.narrow;
  a.edges = g->evl.edges.p;
  a.w = g->evl.w.as<int32_t>();
  a.spins = d_spins;
  a.R = R;
  a.work = reinterpret_cast<uint32_t*>(base + sc.work_off);
  a.out = reinterpret_cast<unsigned long long*>(base + sc.out_off);
  a.bad = reinterpret_cast<unsigned*>(base + sc.bad_off);
  GDI_CUDA(eval_launch(a, g->wkind, st, launches));
  return GDI_OK;
}
void eval_scores(const long long* res, int32_t R, int64_t a_num, int64_t b_num, int64_t denom,
                 gdi_score* scores) {
  for (int32_t r = 0; r < R; r++) {
    const long long cut = res[2 * r], sum = res[2 * r + 1];
    scores[r].cut = cut;
    scores[r].imbalance = sum < 0 ? -sum : sum;
    scores[r].hamiltonian_scaled = a_num * sum * sum + b_num * cut;
    scores[r].hamiltonian = static_cast<double>(scores[r].hamiltonian_scaled) / static_cast<double>(denom);
    scores[r].balance_counter = sum;
  }
}
}  // namespace

int gdi_evaluate_batch(const gdi_graph* g, const int8_t* spins, int32_t replicas, int64_t a_num,
                       int64_t b_num, int64_t denom, gdi_score* scores) {
  NvtxRange nvtx_range("gdi_evaluate_batch");
  if (!g || !spins || !scores) return fail(GDI_ERR_CONFIG, "NULL argument");
  if (replicas < 1) return fail(GDI_ERR_CONFIG, "replicas must be >= 1");
  if (denom <= 0) return fail(GDI_ERR_CONFIG, "denom must be positive");
  int rc = use_device(g->device);
  if (rc) return rc;
  const size_t R = replicas, n = g->st.n;
  DevBuf d_s;
  EvalScratch sc;
  GDI_CUDA(d_s.alloc(R * n));
  GDI_CUDA(cudaMemcpy(d_s.p, spins, R * n, cudaMemcpyHostToDevice));
  if ((rc = eval_enqueue(const_cast<gdi_graph*>(g), d_s.as<int8_t>(), replicas, sc, nullptr, nullptr))) return rc;
  std::vector<long long> res(R * 2 + 2);
  GDI_CUDA(cudaMemcpy(res.data(), sc.buf.p, sc.bad_off + 4, cudaMemcpyDeviceToHost));
  unsigned bad = 0;
  std::memcpy(&bad, reinterpret_cast<const char*>(res.data()) + sc.bad_off, 4);
  if (bad) return fail(GDI_ERR_DOMAIN, "spin must be -1 or +1");
  eval_scores(res.data(), replicas, a_num, b_num, denom, scores);
  return GDI_OK;
}

int gdi_evaluate_device(const gdi_graph* g, const int8_t* d_spins, int32_t replicas, int64_t* d_cut_sum,
                        uint32_t* d_bad, void* stream) {
  if (!g || !d_spins || !d_cut_sum) return fail(GDI_ERR_CONFIG, "NULL argument");
  if (replicas < 1) return fail(GDI_ERR_CONFIG, "replicas must be >= 1");
  int rc = use_device(g->device);
  if (rc) return rc;
  gdi_graph* gm = const_cast<gdi_graph*>(g);
  if ((rc = ensure_eval(gm))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // per-thread scratch kept between calls (the bench times back-to-back
  // calls); a call on another stream first waits for the previous call's
  // kernels (the scratch is reused)
  struct Scratch {
    DevBuf work;
    int dev = -1;
    cudaEvent_t done = nullptr;
    ~Scratch() {
      if (done) cudaEventDestroy(done);
    }
  };
  thread_local Scratch sc;
  DevBuf& work = sc.work;
  if (sc.dev != g->device) {
    if (sc.done) cudaEventDestroy(sc.done);
    sc.done = nullptr;
    work.reset();
    sc.dev = g->device;
  }
  if (!sc.done) GDI_CUDA(cudaEventCreateWithFlags(&sc.done, cudaEventDisableTiming));
  cudaEvent_t done = sc.done;
  GDI_CUDA(cudaStreamWaitEvent(st, done, 0));
  const size_t ww = static_cast<size_t>(eval_work_words(g->st.n, replicas, g->wkind)) * 4 + 16;
  if (work.bytes < ww) {
    GDI_CUDA(cudaEventSynchronize(done));  // (the old buffer may still be in use)
    GDI_CUDA(work.alloc(ww));
  }
  // results straight into the caller's buffer (zeroed here), the bad flag
  // into the caller's word or the scratch's last 4 bytes
  uint32_t* bad = d_bad ? d_bad : reinterpret_cast<uint32_t*>(work.as<char>() + ww - 4);
  GDI_CUDA(cudaMemsetAsync(d_cut_sum, 0, static_cast<size_t>(replicas) * 16, st));
  GDI_CUDA(cudaMemsetAsync(bad, 0, 4, st));
  EvalArgs a{};
  a.n = g->st.n;
  a.m = g->evl.m;
  a.mpos = g->evl.mpos;
  a.narrow = g->evl.narrow;
  a.edges = g->evl.edges.p;
  a.w = g->evl.w.as<int32_t>();
  a.spins = d_spins;
  a.R = replicas;
  a.work = work.as<uint32_t>();
  a.out = reinterpret_cast<unsigned long long*>(d_cut_sum);
  a.bad = bad;
  GDI_CUDA(eval_launch(a, g->wkind, st, nullptr));
  GDI_CUDA(cudaEventRecord(done, st));
  return GDI_OK;
}

// ---- vertex-partitioned sessions (gdi.h) ------------------------------------

}  // extern "C"

struct gdi_part {
  gdi_graph* g = nullptr;
  gdi_params p{};
  int world = 1, rank = 0;
  PartPlan plan;
  PartArgs args{};
  cudaStream_t stream = nullptr;
  std::vector<double> pf;
  std::vector<long long> thr;
  std::vector<unsigned long long> tmask;
  DevBuf seeds, thr_d, tmask_d, live, spins, gsum, gdelta, acc, done, finished, trace, stamps, final_out, watchdog;
  bool inited = false;
  bool peer = false;                 // fused exchange attached (gdi_part_attach_*)
  std::vector<void*> ipc_opened;     // peer spin copies opened through CUDA IPC
  ~gdi_part() {
    for (void* q : ipc_opened) cudaIpcCloseMemHandle(q);
  }
};

extern "C" {

int gdi_part_create(const gdi_graph* g, const gdi_params* p, int32_t world, int32_t rank, uint64_t seed,
                    void* stream, gdi_part** out) {
  if (!out) return fail(GDI_ERR_CONFIG, "out is NULL");
  *out = nullptr;
  if (!g) return fail(GDI_ERR_CONFIG, "graph is NULL");
  int rc = check_params(p);
  if (rc) return rc;
  if (p->mode != GDI_MODE_THROUGHPUT) return fail(GDI_ERR_CONFIG, "vertex partitioning is a throughput-mode path");
  if (world < 1 || rank < 0 || rank >= world) return fail(GDI_ERR_CONFIG, "bad world / rank");
  if ((rc = use_device(g->device))) return rc;
  auto s = std::make_unique<gdi_part>();
  s->g = const_cast<gdi_graph*>(g);
  s->p = *p;
  s->world = world;
  s->rank = rank;
  s->stream = static_cast<cudaStream_t>(stream);
  // chains per rank as for one replica on one device; chunks per rank shrink by W
  if (part_plan(g->st, g->wkind, 1, 4 * p->a_num, p->b_num, &s->plan))
    return fail(GDI_ERR_CAPACITY, "decision arithmetic exceeds the 32-bit kernel bound");
  // the in-flight bound is global: W ranks share the one device's chain count
  {
    const int refresher = s->plan.refresh != 0 ? 1 : 0, cmax = 32 - refresher;
    const int want = std::max(1, s->plan.chains / world);
    const int ctas = std::max(1, std::min(148, want));
    const int cw = std::max(1, std::min(cmax, (want + ctas - 1) / ctas));
    s->plan.ctas = ctas;
    s->plan.chains = ctas * cw;
    s->plan.warps = cw + refresher;
    s->plan.block = 32 * s->plan.warps;
    part_plan_mcast(&s->plan, 1);
  }
  if ((rc = ensure_part(s->g)) || (rc = part_splits(s->g, &s->plan))) return rc;
  schedule(s->p, s->pf, s->thr, s->tmask);
  const size_t n = g->st.n, S = p->sweeps;
  GDI_CUDA(s->seeds.alloc(sizeof(uint64_t)));
  GDI_CUDA(s->thr_d.alloc(S * sizeof(long long)));
  GDI_CUDA(s->tmask_d.alloc(S * sizeof(unsigned long long)));
  GDI_CUDA(s->live.alloc_plain(part_words(g->st.n) * sizeof(uint32_t)));  // exportable to the other ranks (CUDA IPC)
  GDI_CUDA(s->spins.alloc(n));
  GDI_CUDA(s->gsum.alloc(sizeof(long long)));
  GDI_CUDA(s->gdelta.alloc(sizeof(long long)));
  GDI_CUDA(s->acc.alloc(2 * sizeof(unsigned long long)));
  GDI_CUDA(s->done.alloc(sizeof(unsigned int)));
  GDI_CUDA(s->finished.alloc(sizeof(unsigned int)));
  GDI_CUDA(s->trace.alloc(S * sizeof(DevTrace)));
  GDI_CUDA(s->stamps.alloc((S + 1) * sizeof(unsigned long long)));
  GDI_CUDA(s->final_out.alloc(sizeof(DevTrace)));
  GDI_CUDA(s->watchdog.alloc(8 * sizeof(int)));
  GDI_CUDA(cudaMemcpy(s->seeds.p, &seed, sizeof seed, cudaMemcpyHostToDevice));
  GDI_CUDA(cudaMemcpy(s->thr_d.p, s->thr.data(), S * sizeof(long long), cudaMemcpyHostToDevice));
  GDI_CUDA(cudaMemcpy(s->tmask_d.p, s->tmask.data(), S * sizeof(unsigned long long), cudaMemcpyHostToDevice));
  GDI_CUDA(cudaMemset(s->watchdog.p, 0, s->watchdog.bytes));
  PartArgs& a = s->args;
  a.g = g->csr();
  a.order = g->thru.order.as<int32_t>();
  a.psell = g->psell.as<int4>();
  a.pdeg = g->pdeg.as<int32_t>();
  a.pedges = g->pedges.as<int2>();
  a.pedge_w = g->pedge_w.as<int32_t>();
  a.m_edges = g->st.m;
  a.sell_off = g->thru.sell_off.as<int32_t>();
  a.sell_w = g->thru.sell_w.as<int4>();
  a.chains = s->plan.chains;
  a.world_chains = s->plan.chains * world;
  a.chain0 = rank;
  a.chain_stride = world;
  a.rank = rank;
  a.world = world;
  a.sweeps = p->sweeps;
  a.replicas = 1;
  a.seeds = s->seeds.as<uint64_t>();
  a.thr = s->thr_d.as<long long>();
  a.tmask = s->tmask_d.as<unsigned long long>();
  a.bits = s->live.as<uint32_t>();
  a.gsum = s->gsum.as<long long>();
  a.gdelta = s->gdelta.as<long long>();
  a.acc = s->acc.as<unsigned long long>();
  a.done = s->done.as<unsigned int>();
  a.finished = s->finished.as<unsigned int>();
  a.trace = s->trace.as<DevTrace>();
  a.stamps = s->stamps.as<unsigned long long>();
  a.final_out = s->final_out.as<DevTrace>();
  a.watchdog = s->watchdog.as<int>();
  *out = s.release();
  return GDI_OK;
}

int gdi_part_exchange_bytes(const gdi_part* s, int64_t* bytes) {
  if (!s || !bytes) return fail(GDI_ERR_CONFIG, "NULL argument");
  *bytes = part_exchange_bytes(s->g->st.n, s->world, s->peer);
  return GDI_OK;
}

int gdi_part_ipc_handle(const gdi_part* s, void* handle) {
  if (!s || !handle) return fail(GDI_ERR_CONFIG, "NULL argument");
  GDI_CUDA(cudaSetDevice(s->g->device));
  cudaIpcMemHandle_t h;
  GDI_CUDA(cudaIpcGetMemHandle(&h, s->live.p));
  std::memcpy(handle, &h, sizeof h);
  return GDI_OK;
}

namespace {
int attach(gdi_part* s, const std::vector<uint32_t*>& ptrs) {
  if (s->inited) return fail(GDI_ERR_CONFIG, "attach peers before gdi_part_init");
  if (static_cast<int>(ptrs.size()) != s->world - 1 || s->world - 1 > 7)
    return fail(GDI_ERR_CONFIG, "fused exchange needs world - 1 <= 7 peers");
  for (int q = 0; q < s->world - 1; q++) s->args.peer[q] = ptrs[q];
  s->args.npeer = s->world - 1;
  s->peer = s->world > 1;
  return GDI_OK;
}
}  // namespace

int gdi_part_attach_peers(gdi_part* s, const void* handles) {
  if (!s || !handles) return fail(GDI_ERR_CONFIG, "NULL argument");
  GDI_CUDA(cudaSetDevice(s->g->device));
  std::vector<uint32_t*> ptrs;
  for (int q = 0; q < s->world; q++) {
    if (q == s->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + q * GDI_IPC_HANDLE_BYTES, sizeof h);
    void* p = nullptr;
    GDI_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    s->ipc_opened.push_back(p);
    ptrs.push_back(static_cast<uint32_t*>(p));
  }
  return attach(s, ptrs);
}

int gdi_part_attach_local(gdi_part* s, gdi_part* const* parts) {
  if (!s || !parts) return fail(GDI_ERR_CONFIG, "NULL argument");
  std::vector<uint32_t*> ptrs;
  for (int q = 0; q < s->world; q++) {
    if (q == s->rank) continue;
    if (!parts[q] || parts[q]->g->device != s->g->device)
      return fail(GDI_ERR_CONFIG, "local peers must be partitions on the same device");
    ptrs.push_back(parts[q]->live.as<uint32_t>());
  }
  return attach(s, ptrs);
}

int gdi_part_init(gdi_part* s) {
  NvtxRange nvtx_range("gdi_part_init");
  if (!s) return fail(GDI_ERR_CONFIG, "NULL argument");
  GDI_CUDA(cudaSetDevice(s->g->device));
  GDI_CUDA(part_init_launch(s->plan, s->args, s->stream));
  s->inited = true;
  return GDI_OK;
}

int gdi_part_sweep(gdi_part* s, int32_t sweep, void* send) {
  NvtxRange nvtx_range("gdi_part_sweep");
  if (!s || !send) return fail(GDI_ERR_CONFIG, "NULL argument");
  if (!s->inited) return fail(GDI_ERR_CONFIG, "gdi_part_init not called");
  if (sweep < 0 || sweep >= s->p.sweeps) return fail(GDI_ERR_CONFIG, "sweep out of range");
  GDI_CUDA(cudaSetDevice(s->g->device));
  PartArgs a = s->args;
  a.send = static_cast<unsigned char*>(send);
  GDI_CUDA(part_sweep_launch(s->plan, a, sweep, s->stream));
  return GDI_OK;
}

int gdi_part_finish(gdi_part* s, int32_t sweep, const void* recv) {
  NvtxRange nvtx_range("gdi_part_finish");
  if (!s || !recv) return fail(GDI_ERR_CONFIG, "NULL argument");
  if (sweep < 0 || sweep >= s->p.sweeps) return fail(GDI_ERR_CONFIG, "sweep out of range");
  GDI_CUDA(cudaSetDevice(s->g->device));
  GDI_CUDA(part_finish_launch(s->plan, s->args, sweep, recv, part_exchange_bytes(s->g->st.n, s->world, s->peer),
                              s->spins.as<int8_t>(), s->stream));
  return GDI_OK;
}

int gdi_part_fetch(gdi_part* s, gdi_outputs* out) {
  NvtxRange nvtx_range("gdi_part_fetch");
  if (!s || !out) return fail(GDI_ERR_CONFIG, "NULL argument");
  GDI_CUDA(cudaSetDevice(s->g->device));
  GDI_CUDA(cudaStreamSynchronize(s->stream));
  int w = 0;
  GDI_CUDA(cudaMemcpy(&w, s->watchdog.p, sizeof w, cudaMemcpyDeviceToHost));
  if (w != 0) return fail(GDI_ERR_RUNTIME, "k4 watchdog fired");
  const size_t n = s->g->st.n, S = s->p.sweeps;
  const long long A = s->p.a_num, B = s->p.b_num;
  const double denom = static_cast<double>(s->p.denom);
  if (out->spins) GDI_CUDA(cudaMemcpy(out->spins, s->spins.p, n, cudaMemcpyDeviceToHost));
  std::vector<DevTrace> tr(S);
  std::vector<unsigned long long> st(S + 1);
  GDI_CUDA(cudaMemcpy(tr.data(), s->trace.p, S * sizeof(DevTrace), cudaMemcpyDeviceToHost));
  GDI_CUDA(cudaMemcpy(st.data(), s->stamps.p, (S + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  out->seconds = static_cast<double>(st[S] - st[0]) * 1e-9;
  if (out->scores) {
    const DevTrace& f = tr[S - 1];
    gdi_score& sc = out->scores[0];
    sc.cut = f.cut;  // this rank's share
    sc.imbalance = f.sum < 0 ? -f.sum : f.sum;
    sc.hamiltonian_scaled = A * f.sum * f.sum + B * f.cut;
    sc.hamiltonian = static_cast<double>(sc.hamiltonian_scaled) / denom;
    sc.balance_counter = f.counter;
  }
  for (size_t k = 0; k < S; k++) {
    if (out->counters) out->counters[k] = tr[k].counter;
    if (out->trace) {
      gdi_trace_rec& t = out->trace[k];
      t.cut = tr[k].cut;
      t.imbalance = tr[k].sum < 0 ? -tr[k].sum : tr[k].sum;
      t.hamiltonian_scaled = A * tr[k].sum * tr[k].sum + B * tr[k].cut;
      t.hamiltonian = static_cast<double>(t.hamiltonian_scaled) / denom;
      t.flip_probability = s->pf[k];
      t.seconds = static_cast<double>(st[k + 1] - st[k]) * 1e-9;
    }
  }
  return GDI_OK;
}

int gdi_part_detach(gdi_part* s) {
  if (!s) return fail(GDI_ERR_CONFIG, "NULL argument");
  GDI_CUDA(cudaSetDevice(s->g->device));
  if (s->stream) GDI_CUDA(cudaStreamSynchronize(s->stream));
  for (void* q : s->ipc_opened) GDI_CUDA(cudaIpcCloseMemHandle(q));
  s->ipc_opened.clear();
  for (int q = 0; q < 7; q++) s->args.peer[q] = nullptr;
  s->args.npeer = 0;
  s->peer = false;
  return GDI_OK;
}

int gdi_part_destroy(gdi_part* s) {
  if (s) {
    cudaSetDevice(s->g->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    delete s;
  }
  return GDI_OK;
}

int gdi_probe_l2_bandwidth(int device, int64_t bytes, int32_t iters, double* gbs) {
  if (!gbs || bytes < (1 << 20) || iters < 1) return fail(GDI_ERR_CONFIG, "bad probe arguments");
  int rc = use_device(device);
  if (rc) return rc;
  GDI_CUDA(probe_l2_read(static_cast<size_t>(bytes), iters, gbs));
  return GDI_OK;
}

}  // extern "C"
