// Shared device-side declarations of the sweep / evaluation kernels.
#pragma once

#include <cstdint>

namespace gdi {

// Device CSR (built from the reference layout by gdi_graph_create):
//   off[n+1] int32 row pointers, col[2m] int32 neighbours, w[2m] int32
//   weights (nullptr when every weight is +1). Row order = vertex order,
//   adjacency order = the reference's insertion order (sums are integer, so
//   order never changes a result).
struct DevCsr {
  const int32_t* off;
  const int32_t* col;
  const int32_t* w;
  int32_t n;
};

// Per-sweep trace record written by the device: exact cut, exact spin sum
// and the balance counter at the barrier (equal in exact mode).
struct DevTrace {
  long long cut;
  long long sum;
  long long counter;
};

struct ExactArgs {
  DevCsr g;
  const uint4* brow;      // k1_block rows variant: per vertex {maskp, maskn, 4 x 16-bit columns}
  int32_t n_pad;          // per-replica spin stride in shared memory
  int32_t sweeps;
  int32_t replicas;
  const uint64_t* seeds;  // [R]
  const long long* thr;   // [sweeps] flip threshold on (x >> 11); -1 = never
  const unsigned long long* tmask;  // [sweeps] thr*2^11 + 2047 (k1_block)
  long long a4;           // 4 * a_num
  long long b;            // b_num
  int8_t* spins_out;      // [R][n]
  DevTrace* trace;        // [R][sweeps] or nullptr
  unsigned long long* stamps;  // [R][sweeps+1] globaltimer or nullptr
  int8_t* snaps;          // [R][sweeps+1][n] or nullptr
  DevTrace* final_out;    // [R]
};

// k1_window (speculative visit windows, the exact kernel for graphs whose CSR
// does not fit k1_block's shared memory). win_pos/win_neg[i]: bit k-1 set
// when vertex (i-k) mod n is a +1 / -1 neighbour, k = 1..32.
struct PipeArgs {
  DevCsr g;                        // full CSR (initial cut only)
  const uint32_t* win_pos;
  const uint32_t* win_neg;
  const uint32_t* fwd_pos;         // k1_window: forward window masks (bit l: vertex v+1+l is a +1 neighbour)
  const uint32_t* fwd_neg;
  int32_t n_words;                 // spin words per CTA (>= n + 1)
  int8_t* gspins;                  // k1_window: [R][n_words] global int8 spins, or nullptr (shared memory)
  const int32_t* wsell;            // k1_window rows, SELL-32 over the natural order (layout.hpp)
  const int32_t* wsell_off;
  int32_t nprod;                   // k1_window: RNG producer warps
  int32_t rolemap;                 // k1_window: warp role layout (see k1_window.cu)
  int32_t kp;                      // k1_window: producer lanes per replica stream
  int32_t segl;                    // k1_window: draws per producer segment
  int32_t rounds;                  // k1_window: producer rounds buffered per replica (power of two)
  int32_t ring_n;                  // k1_window: draws per replica ring (power of two, multiple of 32)
  int32_t masks_smem;              // k1_window: window masks copied to shared memory
  int32_t jump_table2;             // k1_window: jump is the two-column table (xoshiro_jump2)
  const uint64_t* jump;            // k1_window: (kp-1)*segl-draw xoshiro jump matrix [256][4]
  int32_t sweeps;
  int32_t replicas;
  int32_t rc;                      // replicas (lanes) per CTA
  const uint64_t* seeds;
  const long long* thr;            // [sweeps] floor(pf*2^53), -1 = never
  const unsigned long long* tmask; // [sweeps] thr*2^11 + 2047 (saturated)
  int32_t a4;                      // 4*a_num (narrow)
  int32_t b;                       // b_num (narrow)
  int8_t* spins_out;
  DevTrace* trace;
  unsigned long long* stamps;
  int8_t* snaps;
  DevTrace* final_out;
  int* watchdog;                   // [8] zeroed; non-zero [0] = pipeline stalled
  unsigned long long* prof;        // [16] profiling counters (PROF builds)
  int32_t debug;                   // timing experiments only (GDI_PIPE_DEBUG); 0 in production
};

// k2_sweep (throughput / pooled mode): one CTA per replica.
struct ThruArgs {
  DevCsr g;
  const int32_t* order;            // [n] degree-binned visit order
  // SELL-32 over `order`: chunk c = order[32c .. 32c+31]; sell[sell_off[c] +
  // k*32 + lane] = neighbours 4k..4k+3 of the lane's vertex (index n = pad,
  // bit 31 set = weight -1 on +-1 graphs); sell_w likewise for general weights
  const int4* sell;
  const int32_t* sell_off;         // [chunks+1] in int4 units
  const int4* sell_w;              // nullptr unless general weights
  const int32_t* poff;             // k2_chains: the CSR in position space (row p = vertex order[p]),
  const int32_t* pcol;             //   neighbours as positions, bit 31 = weight -1 (+-1 graphs)
  const int32_t* ppos;             //   vertex -> position
  const int2* edges;               // [m] canonical (u < v) edge list
  const int32_t* edge_w;           // [m] or nullptr (unit)
  int64_t m;
  int32_t n_pad;                   // per-replica spin stride in shared memory
  int32_t sweeps;
  int32_t replicas;
  const uint64_t* seeds;
  const long long* thr;
  const unsigned long long* tmask;
  int32_t a4, b;                   // reduced by gcd (narrow)
  int8_t* spins_out;
  DevTrace* trace;
  unsigned long long* stamps;
  int8_t* snaps;
  DevTrace* final_out;
};

// k2_chains shape and shared-memory layout (byte offsets).
struct ChainCfg {
  int32_t rpc, chains, tail;  // replicas per CTA, chains (warps) per replica, tail chunks
  int32_t seg;                // chunks per segment (chain j visits segments j, j + chains, ...)
  int32_t lane_rows;          // max degree <= 16: changed lanes walk their own rows
  int32_t off_order, off_offs, off_cols, off_rep, rep_bytes, n_pad4, smem;
};

// k4 (vertex-partitioned throughput sweep for large graphs): the chunks of
// the SELL order are dealt round-robin to `world_chains` chains (chain J owns
// chunks J, J + world_chains, ...); this device runs the chains
// chain0 + i * chain_stride (i = warp index in the grid): one device has
// chain0 = 0, stride 1; rank r of W ranks has chain0 = r, stride W, so it owns
// the chunks c = r (mod W). Spins live in position space, one bit per vertex:
// bit l of word c is the spin of the vertex at position 32c + l of the visit
// order (+1 = set), so a chunk's 32 decisions are one word store.
struct PartArgs {
  DevCsr g;
  const int32_t* order;            // [n] position -> vertex (degree-binned visit order)
  const int4* psell;               // SELL-32 rows over positions (layout.hpp build_part_layout)
  const int32_t* pdeg;             // [n] degree of the vertex at each position
  const int2* pedges;              // [m] canonical edges in position space, sorted by the larger position
  const int32_t* pedge_w;          // [m] their weights (general graphs) or nullptr
  long long m_edges, m_main;       // edges; those between main vertices (a prefix of pedges)
  const int32_t* sell_off;         // [chunks+1] in int4 units
  const int4* sell_w;              // nullptr unless general weights
  int32_t nwp;                     // spin words per replica: chunks + 1 zero word, padded to 4
  int32_t chains;                  // chains per replica on this device
  int32_t world_chains, chain0, chain_stride;
  int32_t rank, world;             // vertex partition (1 device: 0, 1)
  int32_t sweeps;
  int32_t replicas;
  int32_t sweep;                   // set per launch
  const uint64_t* seeds;
  const long long* thr;
  const unsigned long long* tmask;
  int32_t a4, b;
  uint32_t* bits;                  // [R][nwp] live spin words
  long long* gsum;                 // [R] balance counter at the last barrier
  long long* gdelta;               // [R] sum of the chains' counter changes this sweep
  unsigned long long* acc;         // [R][2] cut / spin-sum accumulators
  unsigned int* done;              // [R] finishing blocks (ticket)
  unsigned int* finished;          // [R] sweep blocks (ticket, ranks > 1)
  // fused exchange (ranks > 1): every changed chunk word is also stored into
  // the other ranks' copies (peer memory over NVLink); the per-sweep
  // collective then only carries the counter deltas
  uint32_t* peer[7];
  int32_t npeer;
  // ranks > 1: this sweep's send buffer: [int64 delta][uint32 word of every
  // owned main chunk, c = rank + i * world] (the words only without peers)
  unsigned char* send;
  int32_t tail;                    // last chunks of the order, decided against the exact counter
  int32_t cta_tail;                // chains per CTA deferring their last chunk to the CTA tail
  int32_t refresh;                 // 1: the last warp of a CTA re-copies its shared spin copy (0: never)
  int32_t copy_parts;              // bulk copies in flight per refresh
  int32_t mcast;                   // sweep CTAs per cluster sharing the initial copy (1 or 2)
  int32_t debug;                   // timing experiments only (GDI_K4_DEBUG); 0 in production
  DevTrace* trace;
  unsigned long long* stamps;
  int8_t* snaps;
  DevTrace* final_out;
  int* watchdog;
};

struct EvalArgs {
  int32_t n;
  long long m, mpos;        // edges; +1 edges first ([0, mpos)) for +-1 weights
  bool narrow;              // edges as u | v << 16 words (else int2)
  bool aligned4;            // spin rows 4-byte aligned (set by eval_launch)
  const void* edges;        // canonical u < v edge list (EvalLayout)
  const int32_t* w;         // general weights per edge, or nullptr
  const int8_t* spins;      // [R][n]
  int32_t R;
  uint32_t* work;           // k3_pack words [R][nwp] (eval_work_words)
  int32_t nwp;
  unsigned long long* out;  // [R][2] = {cut, spin sum}, accumulated with atomics (zeroed)
  unsigned* bad;            // set when a spin byte is neither +1 nor -1 (zeroed)
};

} // namespace gdi
