// Batched callers of the annealer (include/ising/bench.hpp): the reference's
// run_benchmark job loop (bench.cpp:64-202) and solve --runs selection
// (ising_cli.cpp:148-166), each row / solve as one anneal_batch launch.
#include "ising/bench.hpp"

#include <algorithm>
#include <exception>
#include <limits>
#include <numeric>

namespace ising {

namespace {

std::string path_stem(const std::string& path) {  // bench.cpp graph_id rule
  const auto slash = path.find_last_of("/\\");
  std::string name = slash == std::string::npos ? path : path.substr(slash + 1);
  const auto dot = name.find_last_of('.');
  if (dot != std::string::npos && dot > 0) name = name.substr(0, dot);
  return name;
}

}  // namespace

std::vector<RunReport> run_benchmark(const BenchConfig& config) {
  if (config.runs_per_graph < 1) throw config_error("runs_per_graph must be >= 1");
  if (config.strategies.empty()) throw config_error("at least one strategy must be selected");
  std::vector<RunReport> reports;
  std::vector<std::uint64_t> seeds(static_cast<std::size_t>(config.runs_per_graph));
  for (std::size_t r = 0; r < seeds.size(); r++) seeds[r] = config.base_seed + r;

  for (const std::string& path : config.graph_paths) {
    Graph graph;
    try {
      graph = Graph::parse_gset_file(path);
    } catch (const std::exception& e) {  // per-graph error row, the run continues
      RunReport row;
      row.graph_id = path_stem(path);
      row.strategy = config.strategies.front();
      row.error = e.what();
      reports.push_back(std::move(row));
      continue;
    }
    if (config.unit_weights) graph = graph.with_unit_weights();
    for (Strategy strategy : config.strategies) {
      RunReport row;
      row.graph_id = path_stem(path);
      row.nodes = graph.num_nodes();
      row.edges = graph.num_edges();
      row.density = graph.num_nodes() >= 2 ? density(graph) : 0.0;
      row.strategy = strategy;
      AnnealParams params = default_params_for(strategy, graph);
      const ParamOverrides& o = config.overrides;
      if (o.sweeps) params.sweeps = *o.sweeps;
      if (o.flip_fraction0) params.flip_fraction0 = *o.flip_fraction0;
      if (o.decay_rate) params.decay_rate = *o.decay_rate;
      if (o.workers)
        params.workers = *o.workers;
      else
        params.deterministic = true;  // reproducible rows; parallelism is across runs (here: replicas)
      const Coefficients coeffs = o.coefficients ? *o.coefficients : solver_default_coefficients();
      const MinCutProblem problem = MinCutProblem::make_unchecked(graph, coeffs);
      const BatchResult b = anneal_batch(problem, params, seeds, /*with_trace=*/true);
      row.seeds = seeds;
      row.best_cut = std::numeric_limits<std::int64_t>::max();
      row.best_imbalance = std::numeric_limits<std::int64_t>::max();
      row.cut_min = std::numeric_limits<std::int64_t>::max();
      row.cut_max = std::numeric_limits<std::int64_t>::min();
      double sum = 0.0;
      for (std::size_t r = 0; r < seeds.size(); r++) {
        const PartitionScore& sc = b.scores[r];
        row.best_cut = std::min(row.best_cut, sc.cut);
        row.best_imbalance = std::min(row.best_imbalance, sc.imbalance);
        row.cut_min = std::min(row.cut_min, sc.cut);
        row.cut_max = std::max(row.cut_max, sc.cut);
        sum += static_cast<double>(sc.cut);
        row.run_seconds.push_back(b.runs[r].seconds);
      }
      row.cut_mean = sum / static_cast<double>(seeds.size());
      reports.push_back(std::move(row));
    }
  }
  // bench.cpp:196-201: valid rows first, then by density
  std::stable_sort(reports.begin(), reports.end(), [](const RunReport& a, const RunReport& b) {
    if (a.error.empty() != b.error.empty()) return a.error.empty();
    return a.density < b.density;
  });
  return reports;
}

BestOfRuns anneal_best_of(const MinCutProblem& problem, const AnnealParams& params, std::int32_t runs) {
  if (runs < 1) throw config_error("--runs must be >= 1");
  std::vector<std::uint64_t> seeds(static_cast<std::size_t>(runs));
  for (std::size_t r = 0; r < seeds.size(); r++) seeds[r] = params.seed + r;
  BatchResult b = anneal_batch(problem, params, seeds, /*with_trace=*/true);
  std::size_t best = 0;
  for (std::size_t r = 1; r < seeds.size(); r++)
    if (b.scores[r].hamiltonian_scaled < b.scores[best].hamiltonian_scaled) best = r;  // first seed wins ties
  BestOfRuns out;
  out.best = std::move(b.runs[best]);
  out.score = b.scores[best];
  out.seed = seeds[best];
  out.scores = std::move(b.scores);
  return out;
}

}  // namespace ising
