// gdi-b200 — C++ solver API, source-compatible with the reference's public
// headers (reference proj/include/ising/{errors,rng,graph,model,evaluate,gen,
// anneal}.hpp). Callers written against the reference (its acceptance gate,
// tests/test_support.hpp, python/module.cpp-style bindings) compile against
// this header unchanged; the per-file headers next to it only forward here.
//
// What differs is underneath: `anneal` does not run a CPU worker pool. It is a
// thin wrapper over the C ABI in include/gdi.h, which uploads the graph to HBM
// once per (Graph, device) and runs the sm_100a sweep kernels. There is no CPU
// fallback: without a usable CUDA device `anneal` throws std::runtime_error.
#pragma once

#include <atomic>
#include <cstdint>
#include <functional>
#include <iosfwd>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace ising {

// ---------------------------------------------------------------- errors
// Taxonomy of reference errors.hpp:8-38. The C ABI reports the same four
// classes as negative status codes (GDI_ERR_*), mapped back to these types.

class parse_error : public std::runtime_error {
public:
  explicit parse_error(std::string msg, long line = 0)
      : std::runtime_error(line > 0 ? "line " + std::to_string(line) + ": " + msg : std::move(msg)),
        line_(line) {}
  long line() const { return line_; }

private:
  long line_;
};

class domain_error : public std::runtime_error {
public:
  using std::runtime_error::runtime_error;
};

class config_error : public std::runtime_error {
public:
  using std::runtime_error::runtime_error;
};

class capacity_error : public std::runtime_error {
public:
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- RNG
// xoshiro256++ seeded by four splitmix64 outputs; `stream(seed, id)` derives
// decorrelated streams (reference rng.hpp:10-65). The device kernels run the
// identical generator (paper_1908_00210_b200/csrc/device_rng.cuh); the
// deterministic mode is bit-exact only because these agree.
class Rng {
public:
  explicit Rng(std::uint64_t seed) {
    std::uint64_t x = seed;
    for (std::uint64_t& w : s_) w = mix(x);
  }
  static Rng stream(std::uint64_t seed, std::uint64_t stream_id) {
    return Rng(seed ^ (0xd1b54a32d192ed03ULL * (stream_id + 1)));
  }
  std::uint64_t next() {
    const std::uint64_t out = rot(s_[0] + s_[3], 23) + s_[0];
    const std::uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rot(s_[3], 45);
    return out;
  }
  double next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  bool coin() { return (next() >> 63) != 0; }
  // Uniform in [0, bound): 128-bit multiply-shift with exact rejection.
  std::uint64_t next_below(std::uint64_t bound) {
    const std::uint64_t reject_below = static_cast<std::uint64_t>(-bound) % bound;
    for (;;) {
      const __uint128_t prod = static_cast<__uint128_t>(next()) * bound;
      const auto low = static_cast<std::uint64_t>(prod);
      if (low >= bound || low >= reject_below) return static_cast<std::uint64_t>(prod >> 64);
    }
  }
  const std::uint64_t* state() const { return s_; }

private:
  static std::uint64_t mix(std::uint64_t& x) {
    std::uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  static std::uint64_t rot(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  std::uint64_t s_[4];
};

// ---------------------------------------------------------------- graph

struct Edge {
  std::int32_t u;
  std::int32_t v;
  std::int32_t weight;
};

struct Neighbor {
  std::int32_t node;
  std::int32_t weight;
};

namespace detail {
struct DeviceGraphCache; // per-(graph, device) HBM copy, see src anneal.cpp
}

class Graph;
namespace detail {
Graph parse_gset_text(std::string_view text);  // the G-set parser (graph.cpp)
}

// Immutable weighted undirected graph, CSR form: int64 offsets[n+1] and
// {node, weight} adjacency[2m] in edge-insertion order (reference
// graph.hpp:25-68). Copies share one lazily built device-resident copy.
class Graph {
public:
  Graph() = default;

  static Graph from_edges(std::int32_t num_nodes, std::span<const Edge> edges);
  static Graph parse_gset(std::istream& in);
  static Graph parse_gset(const std::string& text);
  static Graph parse_gset_file(const std::string& path);

  std::int32_t num_nodes() const { return n_; }
  std::int64_t num_edges() const { return m_; }
  std::int32_t max_degree() const { return max_deg_; }
  bool all_unit_weights() const { return unit_; }
  std::int32_t degree(std::int32_t v) const {
    return static_cast<std::int32_t>(offsets_[v + 1] - offsets_[v]);
  }
  std::span<const Neighbor> neighbors(std::int32_t v) const {
    return {adj_.data() + offsets_[v], adj_.data() + offsets_[v + 1]};
  }

  std::vector<Edge> edges() const; // canonical: ascending (min, max)
  std::string to_gset() const;      // canonical text; reparse is identity
  Graph with_unit_weights() const;

  // Raw CSR views (new; used by the device upload and the Python binding).
  const std::vector<std::int64_t>& csr_offsets() const { return offsets_; }
  const std::vector<Neighbor>& csr_adjacency() const { return adj_; }
  detail::DeviceGraphCache& device_cache() const;

private:
  friend Graph detail::parse_gset_text(std::string_view text);
  // CSR from an edge list; check: endpoint range, self-loop and duplicate
  // checks (from_edges); the parser has done them already
  static Graph build(std::int32_t num_nodes, std::span<const Edge> edges, bool check);

  std::int32_t n_ = 0;
  std::int64_t m_ = 0;
  std::int32_t max_deg_ = 0;
  bool unit_ = true;
  std::vector<std::int64_t> offsets_;
  std::vector<Neighbor> adj_;
  mutable std::shared_ptr<detail::DeviceGraphCache> dev_;
};

double density(const Graph& g); // 2m / (n(n-1)), n >= 2

// ---------------------------------------------------------------- model

using Spin = std::int8_t;
using SpinState = std::vector<Spin>;

void validate_spin_state(const SpinState& state, std::int32_t num_nodes);
std::int64_t spin_sum(const SpinState& state);

// A = a_num/denom, B = b_num/denom; energies are kept in integer units of
// 1/denom ("scaled") so every identity is exact.
struct Coefficients {
  std::int64_t a_num = 1;
  std::int64_t b_num = 1;
  std::int64_t denom = 1;
  double a() const { return static_cast<double>(a_num) / static_cast<double>(denom); }
  double b() const { return static_cast<double>(b_num) / static_cast<double>(denom); }
};

// G = sum sigma, relaxed atomic (reference model.hpp:39-49). On the device
// the counter lives in registers of the replica's lanes (exact mode) or in
// shared memory (throughput mode); this host type remains for API callers.
class BalanceCounter {
public:
  explicit BalanceCounter(std::int64_t initial = 0) : v_(initial) {}
  std::int64_t value() const { return v_.load(std::memory_order_relaxed); }
  void add(std::int64_t delta) { v_.fetch_add(delta, std::memory_order_relaxed); }
  void reset(std::int64_t value) { v_.store(value, std::memory_order_relaxed); }

private:
  std::atomic<std::int64_t> v_;
};

// Eq. 7 rule met with equality: B = b, A = b*min(2*maxdeg, N)/8.
Coefficients coefficients_for(const Graph& g, std::int64_t b_num = 1, std::int64_t b_den = 1);
// Solve-path default A=1, B=4 (reference model.cpp:46).
Coefficients solver_default_coefficients();

class MinCutProblem {
public:
  static MinCutProblem make(Graph graph, Coefficients coeffs,
                            std::vector<std::int64_t> external_field = {});
  static MinCutProblem make_unchecked(Graph graph, Coefficients coeffs,
                                      std::vector<std::int64_t> external_field = {});
  static MinCutProblem with_default_coefficients(Graph graph);

  const Graph& graph() const { return graph_; }
  const Coefficients& coefficients() const { return coeffs_; }
  std::int64_t external_field(std::int32_t i) const { return field_.empty() ? 0 : field_[i]; }
  bool satisfies_coefficient_rule() const;

private:
  MinCutProblem(Graph g, Coefficients c, std::vector<std::int64_t> f)
      : graph_(std::move(g)), coeffs_(c), field_(std::move(f)) {}
  Graph graph_;
  Coefficients coeffs_;
  std::vector<std::int64_t> field_;
};

double local_field(const MinCutProblem& problem, const SpinState& state, std::int32_t i);

struct CandidateEnergies {
  std::int64_t at_minus_scaled;
  std::int64_t at_plus_scaled;
  std::int64_t denom;
  double at_minus() const { return static_cast<double>(at_minus_scaled) / static_cast<double>(denom); }
  double at_plus() const { return static_cast<double>(at_plus_scaled) / static_cast<double>(denom); }
};

CandidateEnergies candidate_energies_mincut(const MinCutProblem& problem, const SpinState& state,
                                            std::int64_t balance_excl, std::int32_t i);
std::int64_t global_hamiltonian_scaled(const MinCutProblem& problem, const SpinState& state);
double global_hamiltonian(const MinCutProblem& problem, const SpinState& state);

// ---------------------------------------------------------------- evaluation

struct PartitionScore {
  std::int64_t cut;
  std::int64_t imbalance;
  std::int64_t hamiltonian_scaled;
  double hamiltonian;
};

std::int64_t cut_value(const Graph& g, const SpinState& state);
std::int64_t imbalance(const SpinState& state);
PartitionScore score(const MinCutProblem& problem, const SpinState& state);

struct OracleResult {
  std::int64_t cut;
  SpinState witness;
};
inline constexpr std::int32_t kOracleMaxNodes = 24;
// Exact balanced min cut by enumeration (host only, N <= 24).
OracleResult brute_force_balanced_mincut(const Graph& g, std::int64_t max_imbalance);

// ---------------------------------------------------------------- generators
// Seeded, bit-identical to the reference generators (gen.cpp:12-95).

Graph random_graph(std::int32_t n, std::int64_t m, std::uint64_t seed);
Graph torus_graph(std::int32_t rows, std::int32_t cols, std::uint64_t seed);
Graph random_tree(std::int32_t n, std::uint64_t seed);
Graph random_connected_gnp(std::int32_t n, double p, std::uint64_t seed);

// ---------------------------------------------------------------- annealing

enum class Strategy { standard, gdi };
const char* to_string(Strategy s);
Strategy strategy_from_string(const std::string& name);

struct AnnealParams {
  std::int32_t sweeps = 1000;
  double flip_fraction0 = 0.04;
  double decay_rate = 0.99;
  Strategy strategy = Strategy::gdi;
  std::int32_t workers = 0;
  std::uint64_t seed = 1;
  bool deterministic = false;
  AnnealParams validated() const; // throws config_error; resolves workers
};

double flip_probability(const AnnealParams& params, std::int32_t sweep_index);
AnnealParams default_params_for(Strategy strategy, const Graph& g);

struct TraceRecord {
  std::int64_t hamiltonian_scaled;
  double hamiltonian;
  std::int64_t cut;
  std::int64_t imbalance;
  double flip_probability;
  double seconds;
};

struct AnnealResult {
  SpinState state;
  std::vector<TraceRecord> trace;
  double seconds;
};

struct AnnealHooks {
  std::function<void(std::int32_t sweep, std::span<const Spin> spins, std::int64_t balance_counter)>
      on_sweep_end;
  std::function<void(std::int32_t node, std::span<const Spin> spins)> on_update;
};

// Drop-in for reference anneal.hpp:74-75. Resolved workers == 1 (or
// deterministic) runs the bit-exact kernel; otherwise the throughput kernel.
AnnealResult anneal(const MinCutProblem& problem, const AnnealParams& params,
                    const AnnealHooks* hooks = nullptr);

// ---- extensions (not in the reference): replica batching on the GPU

struct BatchResult {
  std::vector<AnnealResult> runs;       // one per seed, seed order
  std::vector<PartitionScore> scores;   // device-evaluated final scores
  double seconds = 0.0;                 // device time of the whole batch
};

// One launch for all seeds (same params otherwise). Equivalent, seed by
// seed, to calling anneal() with params.seed = seeds[r]. `with_trace` = false
// skips materialising TraceRecords on the host (scores are always returned).
BatchResult anneal_batch(const MinCutProblem& problem, const AnnealParams& params,
                         std::span<const std::uint64_t> seeds, bool with_trace = true);

// CUDA device used by anneal/anneal_batch in this process (default 0, or the
// GDI_DEVICE environment variable).
void set_device(int device);
int device();

} // namespace ising
