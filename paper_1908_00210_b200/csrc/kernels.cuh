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
  int32_t n_pad;          // per-replica spin stride in shared memory
  int32_t sweeps;
  int32_t replicas;
  const uint64_t* seeds;  // [R]
  const long long* thr;   // [sweeps] flip threshold on (x >> 11); -1 = never
  long long a4;           // 4 * a_num
  long long b;            // b_num
  int8_t* spins_out;      // [R][n]
  DevTrace* trace;        // [R][sweeps] or nullptr
  unsigned long long* stamps;  // [R][sweeps+1] globaltimer or nullptr
  int8_t* snaps;          // [R][sweeps+1][n] or nullptr
  DevTrace* final_out;    // [R]
};

struct EvalArgs {
  DevCsr g;
  const int8_t* spins;    // [R][n]
  int32_t replicas;
  unsigned long long* out;  // [R][2] = {cut, sum} accumulated with atomics (zeroed)
};

} // namespace gdi
