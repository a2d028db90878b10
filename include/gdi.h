/* gdi-b200 C ABI — the drop-in boundary of the GDI annealing hot path.
 *
 * Replaces, for host callers, the reference's in-process CPU annealer
 * (reference proj/include/ising/anneal.hpp:74-75 `ising::anneal`, implemented
 * at proj/src/anneal.cpp:132-231) and its exact per-sweep scoring
 * (proj/src/anneal.cpp:64-70 `cut_of`, proj/src/evaluate.cpp:10-32
 * `cut_value`/`imbalance`/`score`). Plain C types only: pointers, sizes,
 * POD structs. No C++ exceptions and no torch types cross this boundary.
 *
 * Status codes map 1:1 onto the reference exception taxonomy
 * (proj/include/ising/errors.hpp:8-38):
 *   GDI_ERR_CONFIG   -> config_error   (anneal.cpp:24-37 validated())
 *   GDI_ERR_DOMAIN   -> domain_error   (graph.cpp:47-61 invalid CSR)
 *   GDI_ERR_CAPACITY -> capacity_error (graph too large for a kernel variant)
 *   GDI_ERR_RUNTIME  -> std::runtime_error (CUDA failure, no device)
 * gdi_last_error() returns the thread-local message of the last failure.
 *
 * Ownership: host buffers are caller-owned; the library owns device memory.
 * Threading: every entry point is reentrant; distinct host threads may run
 * concurrently on distinct graphs/sessions (one CUDA stream per session).
 * There is no CPU fallback: without a usable sm_100 device calls fail with
 * GDI_ERR_RUNTIME.
 */
#ifndef GDI_H
#define GDI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GDI_ABI_VERSION 1

enum {
  GDI_OK = 0,
  GDI_ERR_CONFIG = -1,
  GDI_ERR_DOMAIN = -2,
  GDI_ERR_CAPACITY = -3,
  GDI_ERR_RUNTIME = -4
};

/* anneal.hpp:13 Strategy */
enum { GDI_STRATEGY_STANDARD = 0, GDI_STRATEGY_GDI = 1 };

/* Kernel family. EXACT reproduces the reference's deterministic / single
 * worker mode bit for bit (xoshiro256++ stream 1, visit order 0..n-1;
 * anneal.cpp:189-202). THROUGHPUT is the reference's pooled racy mode
 * (anneal.cpp:203-225): vertex-parallel sweeps, Philox counter RNG keyed by
 * (seed, sweep, vertex), statistically equivalent, not bit-exact. */
enum { GDI_MODE_EXACT = 0, GDI_MODE_THROUGHPUT = 1 };

/* gdi_params.flags */
#define GDI_FLAG_TRACE 0x1u     /* record per-sweep cut / balance / timestamp */
#define GDI_FLAG_SNAPSHOTS 0x2u /* record spins after init and every sweep (hooks) */

typedef struct gdi_graph gdi_graph;     /* device-resident CSR, one device */
typedef struct gdi_session gdi_session; /* device buffers for R replicas  */

/* anneal.hpp:18-30 AnnealParams (validated) + model.hpp:27-34 Coefficients */
typedef struct {
  int32_t sweeps;
  int32_t strategy; /* GDI_STRATEGY_* */
  int32_t mode;     /* GDI_MODE_* */
  uint32_t flags;   /* GDI_FLAG_* */
  double flip_fraction0;
  double decay_rate;
  int64_t a_num;
  int64_t b_num;
  int64_t denom;
} gdi_params;

/* anneal.hpp:39-46 TraceRecord, field for field */
typedef struct {
  int64_t hamiltonian_scaled;
  double hamiltonian;
  int64_t cut;
  int64_t imbalance;
  double flip_probability;
  double seconds;
} gdi_trace_rec;

/* evaluate.hpp:9-14 PartitionScore + the balance counter G at the end */
typedef struct {
  int64_t cut;
  int64_t imbalance;
  int64_t hamiltonian_scaled;
  double hamiltonian;
  int64_t balance_counter;
} gdi_score;

/* Output buffers of one batch; every pointer may be NULL (not wanted).
 * Row-major over replicas: spins[r*n + i], trace[r*sweeps + k],
 * snapshots[(r*(sweeps+1) + k)*n + i] (k=0 is the initial state),
 * counters[r*sweeps + k] = balance counter at barrier k. */
typedef struct {
  int8_t* spins;
  gdi_trace_rec* trace;
  gdi_score* scores;
  int8_t* snapshots;
  int64_t* counters;
  double seconds; /* out: device time of the sweep kernel(s) */
} gdi_outputs;

typedef struct {
  int32_t n;
  int64_t m;
  int32_t max_degree;
  int32_t device;
  int32_t all_unit_weights;
  int64_t device_bytes;
} gdi_graph_info;

int gdi_abi_version(void);
const char* gdi_last_error(void);
int gdi_device_count(int* count);

/* Upload a CSR graph (reference layout graph.hpp:66-67, split into arrays):
 * offsets[n+1] (int64), nbr[offsets[n]] (int32), weights[offsets[n]] or NULL
 * for all-unit weights. Validates symmetry-free invariants cheaply (ranges,
 * self loops); the caller's Graph already enforces the rest. */
int gdi_graph_create(int device, int32_t n, const int64_t* offsets, const int32_t* nbr,
                     const int32_t* weights, gdi_graph** out);
/* The same from the reference's own adjacency array (graph.hpp:67:
 * Neighbor{int32 node, int32 weight}, interleaved): pairs[2e] = neighbour,
 * pairs[2e+1] = weight, split on the device (one upload, no host copy). */
int gdi_graph_create_pairs(int device, int32_t n, const int64_t* offsets, const int32_t* pairs, gdi_graph** out);
int gdi_graph_destroy(gdi_graph* g);
int gdi_graph_query(const gdi_graph* g, gdi_graph_info* info);

/* One-shot batch: R independent anneals (seeds[r]) of the same problem,
 * host in / host out. Equivalent to R calls of the reference anneal() with
 * params.seed = seeds[r]. */
int gdi_anneal_batch(const gdi_graph* g, const gdi_params* p, const uint64_t* seeds,
                     int32_t replicas, gdi_outputs* out);

/* The trace in column form (what array-oriented bindings such as pyising
 * return): hcut_imb[(r*sweeps + k)*3 + {0,1,2}] = {hamiltonian_scaled, cut,
 * imbalance}, seconds[r*sweeps + k], flip_probability[k]. Any pointer may be
 * NULL. */
typedef struct {
  int64_t* hcut_imb;
  double* seconds;
  double* flip_probability;
} gdi_trace_columns;

/* gdi_anneal_batch with the trace written as columns (out->trace and
 * out->counters are ignored): one conversion pass instead of records and a
 * second pass in the binding. */
int gdi_anneal_batch_columns(const gdi_graph* g, const gdi_params* p, const uint64_t* seeds, int32_t replicas,
                             gdi_outputs* out, const gdi_trace_columns* trace);

/* Fused exact evaluation (cut, imbalance, H) of R host spin vectors. */
int gdi_evaluate_batch(const gdi_graph* g, const int8_t* spins, int32_t replicas, int64_t a_num,
                       int64_t b_num, int64_t denom, gdi_score* scores);

/* The same on device-resident spins [R][n] (int8, device pointer), enqueued
 * on `stream` (a cudaStream_t; NULL = legacy stream) without synchronising:
 * d_cut_sum[2r] = cut, d_cut_sum[2r+1] = spin sum (device int64 [R][2]);
 * *d_bad (device uint32, may be NULL) becomes nonzero when a spin byte is
 * neither +1 nor -1. H = a*sum^2 + b*cut as in evaluate.cpp:25-32. The first
 * call on a graph builds its edge list (synchronous). */
int gdi_evaluate_device(const gdi_graph* g, const int8_t* d_spins, int32_t replicas, int64_t* d_cut_sum,
                        uint32_t* d_bad, void* stream);

/* Session API: keeps inputs and outputs resident in HBM between launches so
 * a caller can time the kernels alone. `stream` is a cudaStream_t (NULL: the
 * session creates its own). launch() is asynchronous on that stream. */
int gdi_session_create(const gdi_graph* g, const gdi_params* p, int32_t replicas, void* stream,
                       gdi_session** out);
int gdi_session_set_seeds(gdi_session* s, const uint64_t* seeds);
int gdi_session_launch(gdi_session* s);
int gdi_session_sync(gdi_session* s);
int gdi_session_fetch(gdi_session* s, gdi_outputs* out);
/* Kernel launches issued per gdi_session_launch (for launch accounting). */
int gdi_session_launch_count(const gdi_session* s, int32_t* count);
/* Name of the kernel variant the session selected (static string). */
const char* gdi_session_kernel(const gdi_session* s);
int gdi_session_destroy(gdi_session* s);

/* Vertex-partitioned anneal of ONE replica across W ranks (one device each;
 * SURVEY.md §8(e), the 1M-vertex config). Throughput mode only. Rank r owns
 * the chunks c = r (mod W) of the degree-binned order and keeps a full copy
 * of the spins (one bit per vertex); remote spins are refreshed once per
 * sweep (racy reads, reference SPEC.md concurrency contract). Per sweep the
 * caller runs, on `stream`:
 *   gdi_part_sweep(s, k, send)              sweep kernel: writes this rank's
 *                                           counter delta and its owned chunk
 *                                           spin words into `send`
 *   all-gather of the W send buffers        (e.g. ncclAllGather, same stream)
 *   gdi_part_finish(s, k, recv)             finishing kernel: global tail,
 *                                           this rank's cut share, counter,
 *                                           trace record
 * with send = gdi_part_exchange_bytes() bytes and recv = W times that
 * (rank-major): two kernel launches per sweep, no host work between them (the
 * sequence can be captured as one CUDA graph with the collectives). Trace cuts
 * and the final cut from gdi_part_fetch are this rank's share (the edges whose
 * lower endpoint in the visit order lies in a chunk this rank owns; rank 0
 * also counts the tail's); the sum over ranks is the cut. Imbalance, counters
 * and spins are global on every rank. W == 1 gives the single-device K4 path. */
typedef struct gdi_part gdi_part;
int gdi_part_create(const gdi_graph* g, const gdi_params* p, int32_t world, int32_t rank, uint64_t seed,
                    void* stream, gdi_part** out);
int gdi_part_exchange_bytes(const gdi_part* s, int64_t* bytes);
int gdi_part_init(gdi_part* s);
int gdi_part_sweep(gdi_part* s, int32_t sweep, void* send);
int gdi_part_finish(gdi_part* s, int32_t sweep, const void* recv);
int gdi_part_fetch(gdi_part* s, gdi_outputs* out);
int gdi_part_destroy(gdi_part* s);

/* Fused exchange (optional, before gdi_part_init): each rank's sweep kernel
 * stores every changed chunk spin word (32 vertices, 4 bytes) straight into
 * the other ranks' spin copies (peer memory, NVLink), so remote spins are
 * fresh during the sweep and the per-sweep collective shrinks to the counter
 * deltas (exchange bytes = 16). The ranks must not start sweep k+1 before
 * every rank has finished gdi_part_finish(k) (a barrier collective).
 * gdi_part_ipc_handle exports this rank's spin copy (GDI_IPC_HANDLE_BYTES
 * bytes); gdi_part_attach_peers takes every rank's handle, rank-major (the
 * caller all-gathers them); gdi_part_attach_local wires W partitions of one
 * process on one device (testing). At most 8 ranks. */
#define GDI_IPC_HANDLE_BYTES 64
int gdi_part_ipc_handle(const gdi_part* s, void* handle);
int gdi_part_attach_peers(gdi_part* s, const void* handles);
int gdi_part_attach_local(gdi_part* s, gdi_part* const* parts);
/* Teardown order for the fused exchange: every rank calls gdi_part_detach
 * (waits for its stream, closes the peers' IPC mappings), then the ranks
 * synchronise (a process-group barrier), then gdi_part_destroy frees this
 * rank's exported copy. Destroying an exporter while a peer still has its
 * copy open is undefined behaviour in CUDA. */
int gdi_part_detach(gdi_part* s);

/* Measurement utility (not a reference interface): sustained read bandwidth
 * in GB/s of an L2-resident buffer of `bytes` bytes re-read `iters` times on
 * `device`; the roofline denominator for cache-resident graphs. */
int gdi_probe_l2_bandwidth(int device, int64_t bytes, int32_t iters, double* gbs);

#ifdef __cplusplus
}
#endif
#endif
