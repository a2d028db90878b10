/* TEST INFRASTRUCTURE — CPU restatement of the reference algorithm for the
 * GDI hot path, used only as the parity checker by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg. Never linked
 * into, loaded by, or called from the product library.
 *
 * Parity pinned: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by the unmodified reference compiled from
 * /root/reference (oracle/_ref, tests/golden/make_golden.py) and against the
 * known answers of SURVEY.md §8(c).
 *
 * All arrays are caller-owned. Graphs use the reference CSR layout
 * (graph.hpp:66-67): int64 offsets[n+1], int32 neighbour[2m], int32 weight[2m],
 * adjacency in edge-insertion order (graph.cpp:67-77).
 */
#ifndef GDI_ORACLE_H
#define GDI_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint64_t s[4];
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed);
void orc_rng_stream(orc_rng* r, uint64_t seed, uint64_t stream_id);
uint64_t orc_rng_next(orc_rng* r);
uint64_t orc_rng_below(orc_rng* r, uint64_t bound);
/* Fill out[count] with consecutive raw draws of stream(seed, id). */
void orc_rng_draws(uint64_t seed, uint64_t stream_id, int64_t count, uint64_t* out);
void orc_rng_draws_seed(uint64_t seed, int64_t count, uint64_t* out);

/* Generators: edge lists in generation order. Return 0 or a negative code. */
int orc_gen_random(int32_t n, int64_t m, uint64_t seed, int32_t* eu, int32_t* ev, int32_t* ew);
int orc_gen_torus(int32_t rows, int32_t cols, uint64_t seed, int32_t* eu, int32_t* ev, int32_t* ew);
/* SURVEY §8(c) G81±1 recipe: torus edges in canonical order with coin weights. */
int orc_gen_torus_pm1(int32_t rows, int32_t cols, uint64_t seed, int32_t* eu, int32_t* ev, int32_t* ew);

/* CSR build (graph.cpp:46-79). Returns max degree (>=0) or a negative code:
 * -1 bad n, -2 endpoint out of range, -3 self-loop, -4 duplicate edge. */
int32_t orc_csr_from_edges(int32_t n, int64_t m, const int32_t* eu, const int32_t* ev,
                           const int32_t* ew, int64_t* offsets, int32_t* nbr, int32_t* w);

/* Canonical edge list (graph.cpp:141-151): ascending (min, max). */
int64_t orc_canonical_edges(int32_t n, const int64_t* offsets, const int32_t* nbr,
                            const int32_t* w, int32_t* eu, int32_t* ev, int32_t* ew);

int64_t orc_cut(int32_t n, const int64_t* offsets, const int32_t* nbr, const int32_t* w,
                const int8_t* spins);

/* Deterministic single-worker anneal (anneal.cpp:132-231, workers == 1):
 * spins_out[n]; trace_out[sweeps*3] = {h_scaled, cut, imbalance} per sweep;
 * counter_out[sweeps] (optional) = balance counter at each barrier;
 * pf_out[sweeps] (optional) = flip probability recorded per sweep;
 * stats_out[2] (optional) = {ties, draws}. Returns 0 or -1 on bad params. */
int orc_anneal_det(int32_t n, const int64_t* offsets, const int32_t* nbr, const int32_t* w,
                   int64_t a_num, int64_t b_num, int64_t denom, int32_t sweeps, double pf0,
                   double decay, uint64_t seed, int8_t* spins_out, int64_t* trace_out,
                   int64_t* counter_out, double* pf_out, int64_t* stats_out);

/* FNV-1a 64 (offset 1469598103934665603, prime 1099511628211) per row. */
void orc_fnv1a_rows(const uint8_t* data, int64_t count, int64_t len, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
