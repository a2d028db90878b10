// ising::anneal — drop-in for reference proj/src/anneal.cpp:132-231, as a
// thin C++ wrapper over the C ABI (include/gdi.h). No CPU annealing code
// exists here: the sweeps run in the sm_100a kernels of libgdi; a missing or
// non-Blackwell device is an error (std::runtime_error), never a fallback.
//
// Mapping of the reference's execution modes (anneal.cpp:189-225):
//   resolved workers == 1 (or deterministic) -> GDI_MODE_EXACT: bit-exact
//     replay of the single-worker path, any strategy (standard and gdi
//     coincide there, acceptance.cpp:311-336);
//   workers > 1 -> GDI_MODE_THROUGHPUT: the racy pooled contract.
// Hooks (anneal.hpp:54-63) are served from per-sweep device snapshots:
// on_sweep_end gets the spins and the device balance counter at every
// barrier; on_update (single worker only, as in the reference) is replayed
// exactly, because visit i of sweep k is the last write of spin i in that
// sweep: the state after visit i is snapshot[k+1][0..i] ++ snapshot[k][i+1..].
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <thread>

#include "abi_util.hpp"
#include "gdi.h"
#include "ising/ising.hpp"

namespace ising {

// ---------------------------------------------------------------- device cache

namespace detail {

struct DeviceGraphCache {
  std::mutex mu;
  std::vector<gdi_graph*> per_device;
  ~DeviceGraphCache() {
    for (gdi_graph* g : per_device)
      if (g) gdi_graph_destroy(g);
  }
};

} // namespace detail

namespace {

std::mutex g_cache_create_mu;

std::atomic<int>& device_slot() {
  static std::atomic<int> dev{[] {
    const char* e = std::getenv("GDI_DEVICE");
    return e ? std::atoi(e) : 0;
  }()};
  return dev;
}

[[noreturn]] void raise(int rc) {
  const std::string msg = gdi_last_error();
  switch (rc) {
    case GDI_ERR_CONFIG: throw config_error(msg);
    case GDI_ERR_DOMAIN: throw domain_error(msg);
    case GDI_ERR_CAPACITY: throw capacity_error(msg);
    default: throw std::runtime_error("gdi: " + msg);
  }
}

void check(int rc) {
  if (rc != GDI_OK) raise(rc);
}

const gdi_graph* device_graph(const Graph& g, int dev) {
  detail::DeviceGraphCache& cache = g.device_cache();
  std::lock_guard<std::mutex> lock(cache.mu);
  if (static_cast<int>(cache.per_device.size()) <= dev) cache.per_device.resize(dev + 1, nullptr);
  if (!cache.per_device[dev]) {
    const std::int32_t n = g.num_nodes();
    gdi_graph* h = nullptr;
    check(gdi_graph_create_pairs(dev, n, g.csr_offsets().data(), adjacency_pairs(g), &h));
    cache.per_device[dev] = h;
  }
  return cache.per_device[dev];
}

gdi_params to_abi(const MinCutProblem& problem, const AnnealParams& p) {
  gdi_params q{};
  q.sweeps = p.sweeps;
  q.strategy = p.strategy == Strategy::standard ? GDI_STRATEGY_STANDARD : GDI_STRATEGY_GDI;
  q.mode = p.workers == 1 ? GDI_MODE_EXACT : GDI_MODE_THROUGHPUT;
  q.flags = 0;
  q.flip_fraction0 = p.flip_fraction0;
  q.decay_rate = p.decay_rate;
  q.a_num = problem.coefficients().a_num;
  q.b_num = problem.coefficients().b_num;
  q.denom = problem.coefficients().denom;
  return q;
}

TraceRecord to_record(const gdi_trace_rec& t) {
  return TraceRecord{t.hamiltonian_scaled, t.hamiltonian, t.cut, t.imbalance, t.flip_probability, t.seconds};
}

} // namespace

detail::DeviceGraphCache& Graph::device_cache() const {
  std::lock_guard<std::mutex> lock(g_cache_create_mu);
  if (!dev_) dev_ = std::make_shared<detail::DeviceGraphCache>();
  return *dev_;
}

void set_device(int device) { device_slot().store(device); }
int device() { return device_slot().load(); }

// ---------------------------------------------------------------- params

const char* to_string(Strategy s) { return s == Strategy::standard ? "standard" : "gdi"; }

Strategy strategy_from_string(const std::string& name) {
  if (name == "gdi") return Strategy::gdi;
  if (name == "standard") return Strategy::standard;
  throw config_error("unknown strategy \"" + name + "\" (standard|gdi)");
}

// anneal.cpp:24-37
AnnealParams AnnealParams::validated() const {
  AnnealParams p = *this;
  if (p.sweeps < 1) throw config_error("sweeps must be >= 1");
  if (!(p.flip_fraction0 >= 0.0 && p.flip_fraction0 <= 1.0)) throw config_error("flip_fraction0 must be in [0, 1]");
  if (!(p.decay_rate > 0.0 && p.decay_rate < 1.0)) throw config_error("decay_rate must be in (0, 1)");
  if (p.workers < 0) throw config_error("workers must be >= 0");
  if (p.deterministic)
    p.workers = 1;
  else if (p.workers == 0)
    p.workers = static_cast<std::int32_t>(std::max(1u, std::thread::hardware_concurrency()));
  return p;
}

// anneal.cpp:39-45 — iterated product, not pow(), so the values match the
// trace bit for bit.
double flip_probability(const AnnealParams& params, std::int32_t sweep_index) {
  if (sweep_index < 0 || sweep_index >= params.sweeps) throw config_error("sweep index out of range");
  double pf = params.flip_fraction0;
  for (std::int32_t k = 0; k < sweep_index; k++) pf *= params.decay_rate;
  return pf;
}

// anneal.cpp:47-58 (standard needs 5x the flip fraction, paper §V-D)
AnnealParams default_params_for(Strategy strategy, const Graph&) {
  AnnealParams p;
  p.strategy = strategy;
  p.flip_fraction0 = strategy == Strategy::standard ? 0.20 : 0.04;
  p.decay_rate = 0.99;
  p.sweeps = 1000;
  p.workers = 0;
  return p;
}

// ---------------------------------------------------------------- anneal

AnnealResult anneal(const MinCutProblem& problem, const AnnealParams& params_in, const AnnealHooks* hooks) {
  const AnnealParams params = params_in.validated();
  const Graph& g = problem.graph();
  const std::int32_t n = g.num_nodes();
  const std::size_t S = static_cast<std::size_t>(params.sweeps);
  const int dev = device();
  const gdi_graph* dg = device_graph(g, dev);

  const bool want_sweep_hook = hooks && hooks->on_sweep_end;
  const bool want_update_hook = hooks && hooks->on_update && params.workers == 1;

  gdi_params q = to_abi(problem, params);
  AnnealResult res;
  res.state.resize(static_cast<std::size_t>(n));
  std::vector<gdi_trace_rec> trace(S);
  std::vector<std::int64_t> counters(S);
  std::vector<std::int8_t> snaps;
  gdi_score sc{};
  gdi_outputs out{};
  out.spins = res.state.data();
  out.trace = trace.data();
  out.scores = &sc;
  out.counters = counters.data();
  if (want_sweep_hook || want_update_hook) {
    snaps.resize((S + 1) * static_cast<std::size_t>(n));
    out.snapshots = snaps.data();
  }
  const std::uint64_t seed = params.seed;
  check(gdi_anneal_batch(dg, &q, &seed, 1, &out));

  res.trace.reserve(S);
  res.seconds = 0.0;
  for (const gdi_trace_rec& t : trace) {
    res.trace.push_back(to_record(t));
    res.seconds += t.seconds;
  }

  if (want_sweep_hook || want_update_hook) {
    SpinState live(snaps.begin(), snaps.begin() + n);
    for (std::size_t k = 0; k < S; k++) {
      const std::int8_t* after = snaps.data() + (k + 1) * static_cast<std::size_t>(n);
      if (want_update_hook) {
        for (std::int32_t i = 0; i < n; i++) {
          live[i] = after[i];
          hooks->on_update(i, std::span<const Spin>(live));
        }
      } else {
        std::copy(after, after + n, live.begin());
      }
      if (want_sweep_hook) hooks->on_sweep_end(static_cast<std::int32_t>(k), std::span<const Spin>(live), counters[k]);
    }
  }
  return res;
}

BatchResult anneal_batch(const MinCutProblem& problem, const AnnealParams& params_in,
                         std::span<const std::uint64_t> seeds, bool with_trace) {
  const AnnealParams params = params_in.validated();
  if (seeds.empty()) return BatchResult{};
  const Graph& g = problem.graph();
  const std::size_t n = static_cast<std::size_t>(g.num_nodes());
  const std::size_t S = static_cast<std::size_t>(params.sweeps);
  const std::size_t R = seeds.size();
  const gdi_graph* dg = device_graph(g, device());

  gdi_params q = to_abi(problem, params);
  std::vector<std::int8_t> spins(R * n);
  std::vector<gdi_trace_rec> trace(with_trace ? R * S : 0);
  std::vector<gdi_score> sc(R);
  gdi_outputs out{};
  out.spins = spins.data();
  out.trace = with_trace ? trace.data() : nullptr;
  out.scores = sc.data();
  check(gdi_anneal_batch(dg, &q, seeds.data(), static_cast<std::int32_t>(R), &out));

  BatchResult b;
  b.seconds = out.seconds;
  b.runs.resize(R);
  b.scores.resize(R);
  for (std::size_t r = 0; r < R; r++) {
    AnnealResult& a = b.runs[r];
    a.state.assign(spins.begin() + r * n, spins.begin() + (r + 1) * n);
    a.seconds = 0.0;
    if (with_trace) {
      a.trace.reserve(S);
      for (std::size_t k = 0; k < S; k++) {
        a.trace.push_back(to_record(trace[r * S + k]));
        a.seconds += trace[r * S + k].seconds;
      }
    }
    b.scores[r] = PartitionScore{sc[r].cut, sc[r].imbalance, sc[r].hamiltonian_scaled, sc[r].hamiltonian};
  }
  return b;
}

} // namespace ising
