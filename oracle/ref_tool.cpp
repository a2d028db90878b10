// TEST INFRASTRUCTURE — never part of the product path.
//
// Driver around the *unmodified* reference CPU library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It is used
// (a) to generate the golden vectors under tests/golden/ and (b) as the
// reference arm / cpu_baseline of bench.py (bench.cpp:158-175 style replica
// pool of deterministic single-worker anneals).
//
// Subcommands (all output is one JSON document on stdout):
//   gset   <recipe...>                         canonical G-set text of a recipe graph
//   golden <recipe...> --seeds A B [params]    per-seed final score, spins, trace
//   bench  <recipe...> --replicas R --threads T [params]
//                                              replica-throughput timing
//   runbench <gset paths...> --replicas RUNS --seeds BASE _ --strategy gdi|standard|both
//            [--sweeps S]                      the reference's own run_benchmark rows
// Recipes: random N M SEED | torus R C SEED | torus_pm1 R C SEED | file PATH
//   torus_pm1 = SURVEY §8(c) G81±1 recipe: torus_graph(R,C,SEED), then over the
//   canonical edges() order w = Rng(SEED).coin() ? +1 : -1, rebuilt by from_edges.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ising/anneal.hpp"
#include "ising/bench.hpp"
#include "ising/evaluate.hpp"
#include "ising/gen.hpp"
#include "ising/graph.hpp"
#include "ising/model.hpp"
#include "ising/rng.hpp"

using namespace ising;

namespace {

std::uint64_t fnv1a(const void* data, std::size_t len,
                    std::uint64_t h = 1469598103934665603ULL) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (std::size_t i = 0; i < len; i++) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

struct Args {
  std::vector<std::string> pos;
  std::uint64_t seed_lo = 1, seed_hi = 1;
  std::int32_t sweeps = 1000;
  double pf0 = 0.04, decay = 0.99;
  std::int64_t a = 1, b = 4, denom = 1;
  std::int32_t replicas = 8, threads = 0;
  bool full_spins = false, full_trace = false;
  std::string strategy = "gdi";
};

Args parse(int argc, char** argv) {
  Args a;
  for (int i = 2; i < argc; i++) {
    std::string s = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) { std::fprintf(stderr, "missing value for %s\n", s.c_str()); std::exit(2); }
      return argv[++i];
    };
    if (s == "--seeds") { a.seed_lo = std::stoull(next()); a.seed_hi = std::stoull(next()); }
    else if (s == "--sweeps") a.sweeps = std::stoi(next());
    else if (s == "--pf0") a.pf0 = std::stod(next());
    else if (s == "--decay") a.decay = std::stod(next());
    else if (s == "--a") a.a = std::stoll(next());
    else if (s == "--b") a.b = std::stoll(next());
    else if (s == "--denom") a.denom = std::stoll(next());
    else if (s == "--replicas") a.replicas = std::stoi(next());
    else if (s == "--threads") a.threads = std::stoi(next());
    else if (s == "--strategy") a.strategy = next();
    else if (s == "--full-spins") a.full_spins = true;
    else if (s == "--full-trace") a.full_trace = true;
    else a.pos.push_back(s);
  }
  return a;
}

Graph recipe_graph(const std::vector<std::string>& p) {
  if (p.empty()) throw std::runtime_error("missing recipe");
  const std::string& kind = p[0];
  if (kind == "random") return random_graph(std::stoi(p.at(1)), std::stoll(p.at(2)), std::stoull(p.at(3)));
  if (kind == "torus") return torus_graph(std::stoi(p.at(1)), std::stoi(p.at(2)), std::stoull(p.at(3)));
  if (kind == "torus_pm1") {
    Graph t = torus_graph(std::stoi(p.at(1)), std::stoi(p.at(2)), std::stoull(p.at(3)));
    std::vector<Edge> edges = t.edges();
    Rng w(std::stoull(p.at(3)));
    for (Edge& e : edges) e.weight = w.coin() ? 1 : -1;
    return Graph::from_edges(t.num_nodes(), edges);
  }
  if (kind == "file") return Graph::parse_gset_file(p.at(1));
  throw std::runtime_error("unknown recipe " + kind);
}

AnnealParams make_params(const Args& a, std::uint64_t seed) {
  AnnealParams p;
  p.sweeps = a.sweeps;
  p.flip_fraction0 = a.pf0;
  p.decay_rate = a.decay;
  p.strategy = strategy_from_string(a.strategy);
  p.deterministic = true;
  p.seed = seed;
  return p;
}

int cmd_gset(const Args& a) {
  Graph g = recipe_graph(a.pos);
  std::string text = g.to_gset();
  std::fwrite(text.data(), 1, text.size(), stdout);
  return 0;
}

int cmd_golden(const Args& a) {
  Graph g = recipe_graph(a.pos);
  std::string text = g.to_gset();
  MinCutProblem prob = MinCutProblem::make_unchecked(g, {a.a, a.b, a.denom});
  std::printf("{\"n\": %d, \"m\": %lld, \"gset_fnv\": \"%016llx\", \"max_degree\": %d, \"runs\": [\n",
              g.num_nodes(), static_cast<long long>(g.num_edges()),
              static_cast<unsigned long long>(fnv1a(text.data(), text.size())), g.max_degree());
  bool first = true;
  for (std::uint64_t s = a.seed_lo; s <= a.seed_hi; s++) {
    AnnealResult r = anneal(prob, make_params(a, s));
    PartitionScore sc = score(prob, r.state);
    std::uint64_t tf = 1469598103934665603ULL;
    for (const TraceRecord& t : r.trace) {
      std::int64_t row[3] = {t.hamiltonian_scaled, t.cut, t.imbalance};
      tf = fnv1a(row, sizeof row, tf);
    }
    std::printf("%s{\"seed\": %llu, \"cut\": %lld, \"imbalance\": %lld, \"h_scaled\": %lld, "
                "\"spins_fnv\": \"%016llx\", \"trace_fnv\": \"%016llx\", \"last_pf\": %.17g",
                first ? "" : ",\n", static_cast<unsigned long long>(s),
                static_cast<long long>(sc.cut), static_cast<long long>(sc.imbalance),
                static_cast<long long>(sc.hamiltonian_scaled),
                static_cast<unsigned long long>(fnv1a(r.state.data(), r.state.size())),
                static_cast<unsigned long long>(tf), r.trace.back().flip_probability);
    if (a.full_spins) {
      std::printf(", \"spins\": \"");
      for (Spin v : r.state) std::putchar(v > 0 ? '1' : '0');
      std::printf("\"");
    }
    if (a.full_trace) {
      std::printf(", \"trace\": [");
      for (std::size_t k = 0; k < r.trace.size(); k++)
        std::printf("%s[%lld, %lld, %lld]", k ? ", " : "",
                    static_cast<long long>(r.trace[k].hamiltonian_scaled),
                    static_cast<long long>(r.trace[k].cut),
                    static_cast<long long>(r.trace[k].imbalance));
      std::printf("]");
    }
    std::printf("}");
    first = false;
  }
  std::printf("\n]}\n");
  return 0;
}

// Replica throughput exactly as the reference harness schedules it
// (bench.cpp:158-175): a pool of T threads pulling deterministic
// single-worker anneals (seeds seed_lo + r) off a shared counter.
int cmd_bench(const Args& a) {
  Graph g = recipe_graph(a.pos);
  MinCutProblem prob = MinCutProblem::make_unchecked(g, {a.a, a.b, a.denom});
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned threads = a.threads > 0 ? static_cast<unsigned>(a.threads) : hw;
  std::atomic<int> next{0};
  std::atomic<long long> cut_sum{0};
  auto t0 = std::chrono::steady_clock::now();
  {
    std::vector<std::jthread> pool;
    for (unsigned t = 0; t < threads; t++)
      pool.emplace_back([&]() {
        for (;;) {
          int r = next.fetch_add(1);
          if (r >= a.replicas) return;
          AnnealResult res = anneal(prob, make_params(a, a.seed_lo + static_cast<std::uint64_t>(r)));
          cut_sum.fetch_add(cut_value(g, res.state));
        }
      });
  }
  double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  double updates = static_cast<double>(a.replicas) * g.num_nodes() * a.sweeps;
  std::printf("{\"seconds\": %.6f, \"updates\": %.0f, \"updates_per_s\": %.6e, \"threads\": %u, "
              "\"replicas\": %d, \"n\": %d, \"sweeps\": %d, \"cut_sum\": %lld}\n",
              secs, updates, updates / secs, threads, a.replicas, g.num_nodes(), a.sweeps,
              cut_sum.load());
  return 0;
}

// The reference batched caller itself (bench.cpp:64-202): rows in its own
// order, JSON without the timing fields.
int cmd_runbench(const Args& a) {
  BenchConfig cfg;
  cfg.graph_paths = a.pos;
  cfg.runs_per_graph = a.replicas;
  cfg.base_seed = a.seed_lo;
  if (a.strategy == "both")
    cfg.strategies = {Strategy::gdi, Strategy::standard};
  else
    cfg.strategies = {a.strategy == "standard" ? Strategy::standard : Strategy::gdi};
  cfg.overrides.sweeps = a.sweeps;
  std::vector<RunReport> rows = run_benchmark(cfg);
  std::printf("[");
  for (std::size_t i = 0; i < rows.size(); i++) {
    const RunReport& r = rows[i];
    std::printf("%s\n{\"graph_id\": \"%s\", \"nodes\": %d, \"edges\": %lld, \"density\": %.17g, "
                "\"strategy\": \"%s\", \"best_cut\": %lld, \"best_imbalance\": %lld, \"cut_mean\": %.17g, "
                "\"cut_min\": %lld, \"cut_max\": %lld, \"seeds\": [",
                i ? "," : "", r.graph_id.c_str(), r.nodes, static_cast<long long>(r.edges), r.density,
                r.strategy == Strategy::gdi ? "gdi" : "standard", static_cast<long long>(r.best_cut),
                static_cast<long long>(r.best_imbalance), r.cut_mean, static_cast<long long>(r.cut_min),
                static_cast<long long>(r.cut_max));
    for (std::size_t k = 0; k < r.seeds.size(); k++)
      std::printf("%s%llu", k ? ", " : "", static_cast<unsigned long long>(r.seeds[k]));
    std::printf("], \"error\": %s}", r.error.empty() ? "\"\"" : "\"unreadable\"");
  }
  std::printf("\n]\n");
  return 0;
}

} // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_tool gset|golden|bench <recipe> [options]\n");
    return 2;
  }
  try {
    Args a = parse(argc, argv);
    std::string cmd = argv[1];
    if (cmd == "gset") return cmd_gset(a);
    if (cmd == "golden") return cmd_golden(a);
    if (cmd == "bench") return cmd_bench(a);
    if (cmd == "runbench") return cmd_runbench(a);
    std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
