/* TEST INFRASTRUCTURE — see gdi_oracle.h. CPU restatement of the reference
 * GDI path; each function cites the reference file:line (paths relative to
 * /root/reference/proj) it restates. Plain C99, no dependency on the product. */
#include "gdi_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---- RNG: xoshiro256++ with splitmix64 seeding (include/ising/rng.hpp) ---- */

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:54-59 */
static uint64_t splitmix64(uint64_t* x) {
  uint64_t z = (*x += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:12-15 */
void orc_rng_seed(orc_rng* r, uint64_t seed) {
  uint64_t x = seed;
  for (int i = 0; i < 4; i++) r->s[i] = splitmix64(&x);
}

/* rng.hpp:19-21 */
void orc_rng_stream(orc_rng* r, uint64_t seed, uint64_t stream_id) {
  orc_rng_seed(r, seed ^ (0xd1b54a32d192ed03ULL * (stream_id + 1)));
}

/* rng.hpp:23-33 */
uint64_t orc_rng_next(orc_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

/* rng.hpp:41-51 (Lemire multiply-shift with the reference's rejection test) */
uint64_t orc_rng_below(orc_rng* r, uint64_t bound) {
  for (;;) {
    uint64_t x = orc_rng_next(r);
    __uint128_t m = (__uint128_t)x * bound;
    uint64_t lo = (uint64_t)m;
    if (lo >= bound || lo >= (uint64_t)(-bound) % bound) return (uint64_t)(m >> 64);
  }
}

void orc_rng_draws(uint64_t seed, uint64_t stream_id, int64_t count, uint64_t* out) {
  orc_rng r;
  orc_rng_stream(&r, seed, stream_id);
  for (int64_t i = 0; i < count; i++) out[i] = orc_rng_next(&r);
}

/* ---- open-addressing set of undirected pair keys (stands in for the
 *      std::unordered_set dedupe of gen.cpp:19-29 / graph.cpp:53-61) ---- */

typedef struct {
  uint64_t* slot;
  uint64_t mask;
} pairset;

static int pairset_init(pairset* ps, int64_t expect) {
  uint64_t cap = 16;
  while (cap < (uint64_t)expect * 2 + 16) cap <<= 1;
  ps->slot = (uint64_t*)malloc(cap * sizeof(uint64_t));
  if (!ps->slot) return -1;
  memset(ps->slot, 0xff, cap * sizeof(uint64_t));
  ps->mask = cap - 1;
  return 0;
}

/* returns 1 if newly inserted, 0 if already present */
static int pairset_insert(pairset* ps, uint64_t key) {
  uint64_t h = key * 0x9e3779b97f4a7c15ULL;
  uint64_t i = (h ^ (h >> 29)) & ps->mask;
  for (;;) {
    if (ps->slot[i] == UINT64_MAX) {
      ps->slot[i] = key;
      return 1;
    }
    if (ps->slot[i] == key) return 0;
    i = (i + 1) & ps->mask;
  }
}

static uint64_t pair_key(int32_t a, int32_t b) {
  if (a > b) {
    int32_t t = a;
    a = b;
    b = t;
  }
  return ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
}

/* ---- generators (src/gen.cpp) ---- */

/* gen.cpp:12-32: draw (u, v) with next_below(n) twice, drop self pairs,
 * order the pair, keep it if unseen. */
int orc_gen_random(int32_t n, int64_t m, uint64_t seed, int32_t* eu, int32_t* ev, int32_t* ew) {
  if (n < 2) return -1;
  if (m > (int64_t)n * (n - 1) / 2) return -2;
  orc_rng r;
  orc_rng_seed(&r, seed);
  pairset ps;
  if (pairset_init(&ps, m)) return -9;
  int64_t k = 0;
  while (k < m) {
    int32_t u = (int32_t)orc_rng_below(&r, (uint64_t)n);
    int32_t v = (int32_t)orc_rng_below(&r, (uint64_t)n);
    if (u == v) continue;
    if (u > v) {
      int32_t t = u;
      u = v;
      v = t;
    }
    if (pairset_insert(&ps, pair_key(u, v))) {
      eu[k] = u;
      ev[k] = v;
      ew[k] = 1;
      k++;
    }
  }
  free(ps.slot);
  return 0;
}

/* gen.cpp:34-54: Fisher-Yates label shuffle, then right and down edges. */
int orc_gen_torus(int32_t rows, int32_t cols, uint64_t seed, int32_t* eu, int32_t* ev, int32_t* ew) {
  if (rows < 3 || cols < 3) return -1;
  const int32_t n = rows * cols;
  int32_t* label = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  if (!label) return -9;
  for (int32_t i = 0; i < n; i++) label[i] = i;
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int32_t i = n - 1; i > 0; i--) {
    int32_t j = (int32_t)orc_rng_below(&r, (uint64_t)i + 1);
    int32_t t = label[i];
    label[i] = label[j];
    label[j] = t;
  }
  int64_t k = 0;
  for (int32_t rr = 0; rr < rows; rr++)
    for (int32_t c = 0; c < cols; c++) {
      int32_t u = rr * cols + c;
      eu[k] = label[u];
      ev[k] = label[rr * cols + (c + 1) % cols];
      ew[k++] = 1;
      eu[k] = label[u];
      ev[k] = label[((rr + 1) % rows) * cols + c];
      ew[k++] = 1;
    }
  free(label);
  return 0;
}

int orc_gen_torus_pm1(int32_t rows, int32_t cols, uint64_t seed, int32_t* eu, int32_t* ev, int32_t* ew) {
  const int32_t n = rows * cols;
  const int64_t m = 2 * (int64_t)n;
  int32_t *tu = malloc(m * 4), *tv = malloc(m * 4), *tw = malloc(m * 4), *nb = malloc(2 * m * 4),
          *w = malloc(2 * m * 4);
  int64_t* off = malloc((size_t)(n + 1) * 8);
  int rc = -9;
  if (!tu || !tv || !tw || !nb || !w || !off) goto done;
  rc = orc_gen_torus(rows, cols, seed, tu, tv, tw);
  if (rc) goto done;
  rc = orc_csr_from_edges(n, m, tu, tv, tw, off, nb, w);
  if (rc < 0) goto done;
  orc_canonical_edges(n, off, nb, w, eu, ev, ew);
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int64_t k = 0; k < m; k++) ew[k] = (orc_rng_next(&r) >> 63) ? 1 : -1;
  rc = 0;
done:
  free(tu);
  free(tv);
  free(tw);
  free(nb);
  free(w);
  free(off);
  return rc;
}

/* ---- CSR (src/graph.cpp) ---- */

/* graph.cpp:46-79: validate, degree count, prefix sum, fill in edge order. */
int32_t orc_csr_from_edges(int32_t n, int64_t m, const int32_t* eu, const int32_t* ev,
                           const int32_t* ew, int64_t* offsets, int32_t* nbr, int32_t* w) {
  if (n <= 0) return -1;
  pairset ps;
  if (pairset_init(&ps, m)) return -9;
  int32_t* deg = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  int64_t* pos = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  int32_t rc = 0;
  if (!deg || !pos) {
    rc = -9;
    goto done;
  }
  for (int64_t k = 0; k < m; k++) {
    if (eu[k] < 0 || eu[k] >= n || ev[k] < 0 || ev[k] >= n) { rc = -2; goto done; }
    if (eu[k] == ev[k]) { rc = -3; goto done; }
    if (!pairset_insert(&ps, pair_key(eu[k], ev[k]))) { rc = -4; goto done; }
    deg[eu[k]]++;
    deg[ev[k]]++;
  }
  offsets[0] = 0;
  for (int32_t i = 0; i < n; i++) {
    offsets[i + 1] = offsets[i] + deg[i];
    if (deg[i] > rc) rc = deg[i];
    pos[i] = offsets[i];
  }
  for (int64_t k = 0; k < m; k++) {
    nbr[pos[eu[k]]] = ev[k];
    w[pos[eu[k]]++] = ew[k];
    nbr[pos[ev[k]]] = eu[k];
    w[pos[ev[k]]++] = ew[k];
  }
done:
  free(ps.slot);
  free(deg);
  free(pos);
  return rc;
}

/* graph.cpp:141-151. Within one u the pairs come from one adjacency row, so
 * sorting (u, v) lexicographically reduces to sorting each row's v. */
static int cmp_pair(const void* a, const void* b) {
  const int32_t* x = (const int32_t*)a;
  const int32_t* y = (const int32_t*)b;
  if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
  return x[1] < y[1] ? -1 : (x[1] > y[1]);
}

int64_t orc_canonical_edges(int32_t n, const int64_t* offsets, const int32_t* nbr,
                            const int32_t* w, int32_t* eu, int32_t* ev, int32_t* ew) {
  int64_t m = offsets[n] / 2;
  int32_t* tmp = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * 3 * sizeof(int32_t));
  int64_t k = 0;
  for (int32_t u = 0; u < n; u++)
    for (int64_t e = offsets[u]; e < offsets[u + 1]; e++)
      if (u < nbr[e]) {
        tmp[3 * k] = u;
        tmp[3 * k + 1] = nbr[e];
        tmp[3 * k + 2] = w[e];
        k++;
      }
  qsort(tmp, (size_t)k, 3 * sizeof(int32_t), cmp_pair);
  for (int64_t i = 0; i < k; i++) {
    eu[i] = tmp[3 * i];
    ev[i] = tmp[3 * i + 1];
    ew[i] = tmp[3 * i + 2];
  }
  free(tmp);
  return k;
}

/* evaluate.cpp:10-18 (identical to anneal.cpp:64-70 cut_of) */
int64_t orc_cut(int32_t n, const int64_t* offsets, const int32_t* nbr, const int32_t* w,
                const int8_t* spins) {
  int64_t cut = 0;
  for (int32_t u = 0; u < n; u++)
    for (int64_t e = offsets[u]; e < offsets[u + 1]; e++)
      if (u < nbr[e] && spins[u] != spins[nbr[e]]) cut += w[e];
  return cut;
}

/* ---- deterministic GDI anneal (src/anneal.cpp) ---- */

int orc_anneal_det(int32_t n, const int64_t* offsets, const int32_t* nbr, const int32_t* w,
                   int64_t a_num, int64_t b_num, int64_t denom, int32_t sweeps, double pf0,
                   double decay, uint64_t seed, int8_t* spins_out, int64_t* trace_out,
                   int64_t* counter_out, double* pf_out, int64_t* stats_out) {
  (void)denom;
  /* anneal.cpp:24-37 validated() */
  if (sweeps < 1 || !(pf0 >= 0.0 && pf0 <= 1.0) || !(decay > 0.0 && decay < 1.0)) return -1;
  int8_t* s = spins_out;
  /* anneal.cpp:148-155: stream 0 coins initialise the spins, G = sum */
  orc_rng r0;
  orc_rng_stream(&r0, seed, 0);
  int64_t G = 0;
  for (int32_t i = 0; i < n; i++) {
    s[i] = (orc_rng_next(&r0) >> 63) ? 1 : -1;
    G += s[i];
  }
  /* anneal.cpp:189-202: single worker uses stream 1 */
  orc_rng r1;
  orc_rng_stream(&r1, seed, 1);
  double pf = pf0;
  int64_t ties = 0, draws = 0;
  for (int32_t k = 0; k < sweeps; k++) {
    for (int32_t i = 0; i < n; i++) {
      /* visit_node, anneal.cpp:86-128 */
      const int8_t own = s[i];
      int64_t field = 0;
      for (int64_t e = offsets[i]; e < offsets[i + 1]; e++) field += (int64_t)w[e] * s[nbr[e]];
      const int64_t excl = G - own;
      const int64_t diff = 4 * a_num * excl - b_num * field;
      int8_t chosen;
      if (diff < 0)
        chosen = 1;
      else if (diff > 0)
        chosen = -1;
      else {
        chosen = (orc_rng_next(&r1) >> 63) ? 1 : -1;
        ties++;
        draws++;
      }
      if (chosen != own) {
        s[i] = chosen;
        G += chosen - own;
      }
      const double u = (double)(orc_rng_next(&r1) >> 11) * 0x1.0p-53;
      draws++;
      if (pf > 0.0 && u <= pf) {
        const int8_t flipped = (int8_t)-chosen;
        s[i] = flipped;
        G += 2 * flipped;
      }
    }
    /* record_barrier, anneal.cpp:165-187 */
    int64_t bal = 0;
    for (int32_t i = 0; i < n; i++) bal += s[i];
    const int64_t cut = orc_cut(n, offsets, nbr, w, s);
    if (trace_out) {
      trace_out[3 * k] = a_num * bal * bal + b_num * cut;
      trace_out[3 * k + 1] = cut;
      trace_out[3 * k + 2] = bal < 0 ? -bal : bal;
    }
    if (counter_out) counter_out[k] = G;
    if (pf_out) pf_out[k] = pf;
    pf *= decay;
  }
  if (stats_out) {
    stats_out[0] = ties;
    stats_out[1] = draws;
  }
  return 0;
}

void orc_rng_draws_seed(uint64_t seed, int64_t count, uint64_t* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int64_t i = 0; i < count; i++) out[i] = orc_rng_next(&r);
}

/* FNV-1a 64 over `count` rows of `len` bytes (SURVEY §8(c) hashing). */
void orc_fnv1a_rows(const uint8_t* data, int64_t count, int64_t len, uint64_t* out) {
  for (int64_t r = 0; r < count; r++) {
    uint64_t h = 1469598103934665603ULL;
    const uint8_t* p = data + r * len;
    for (int64_t i = 0; i < len; i++) {
      h ^= p[i];
      h *= 1099511628211ULL;
    }
    out[r] = h;
  }
}
