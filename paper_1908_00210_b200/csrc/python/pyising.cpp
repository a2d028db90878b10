// pyising — Python binding of the gdi-b200 solver API.
//
// Same module name, class names, attribute names and exception classes as
// the reference binding (reference proj/python/module.cpp:15-183), so its
// Python callers (proj/python/tests/test_smoke.py) run unchanged; `anneal`
// releases the GIL like the reference (module.cpp:177-183). Extensions:
// optional hooks on anneal(), the batched replica call anneal_batch()
// (numpy outputs), numpy CSR views, and Session — the device-resident C-ABI
// session used by bench.py to time the kernels with inputs already in HBM.
#include <pybind11/functional.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <memory>

#include "../host/abi_util.hpp"
#include "../host/parallel.hpp"
#include "gdi.h"
#include "ising/bench.hpp"
#include "ising/ising.hpp"

namespace py = pybind11;
using namespace ising;

namespace {

template <typename T>
py::array_t<T> to_numpy(std::vector<T>&& v, std::vector<py::ssize_t> shape) {
  auto* heap = new std::vector<T>(std::move(v));
  py::capsule owner(heap, [](void* p) { delete static_cast<std::vector<T>*>(p); });
  return py::array_t<T>(shape, heap->data(), owner);
}

[[noreturn]] void raise_abi(int rc) {
  const std::string msg = gdi_last_error();
  if (rc == GDI_ERR_CONFIG) throw config_error(msg);
  if (rc == GDI_ERR_DOMAIN) throw domain_error(msg);
  if (rc == GDI_ERR_CAPACITY) throw capacity_error(msg);
  throw std::runtime_error("gdi: " + msg);
}

void check_abi(int rc) {
  if (rc != GDI_OK) raise_abi(rc);
}

// Per-thread scratch for C-ABI trace records: reused across calls so a batch
// of R x S records does not page-fault ~50 MB of fresh memory every call.
gdi_trace_rec* trace_scratch(std::size_t count) {
  thread_local std::vector<gdi_trace_rec> buf;
  if (buf.size() < count) buf.resize(count);
  return buf.data();
}

// Device-resident session over the C ABI: graph + buffers stay in HBM; the
// caller times launch() on the stream it passes in.
class Evaluator {
public:
  Evaluator(const MinCutProblem& problem, int dev) : n_(problem.graph().num_nodes()), c_(problem.coefficients()) {
    const Graph& g = problem.graph();
    check_abi(gdi_graph_create_pairs(dev, n_, g.csr_offsets().data(), adjacency_pairs(g), &graph_));
  }
  ~Evaluator() {
    if (graph_) gdi_graph_destroy(graph_);
  }
  py::dict evaluate(py::array_t<std::int8_t, py::array::c_style | py::array::forcecast> spins);
  void evaluate_device(std::uintptr_t spins, int replicas, std::uintptr_t cut_sum, std::uintptr_t bad,
                       std::uintptr_t stream) {
    check_abi(gdi_evaluate_device(graph_, reinterpret_cast<const std::int8_t*>(spins), replicas,
                                  reinterpret_cast<std::int64_t*>(cut_sum), reinterpret_cast<std::uint32_t*>(bad),
                                  reinterpret_cast<void*>(stream)));
  }

private:
  std::int32_t n_;
  Coefficients c_;
  gdi_graph* graph_ = nullptr;
};

class Session {
public:
  Session(const MinCutProblem& problem, const AnnealParams& params_in, int replicas, std::uintptr_t stream,
          bool trace, int dev)
      : n_(problem.graph().num_nodes()), replicas_(replicas) {
    const AnnealParams params = params_in.validated();
    const Graph& g = problem.graph();
    check_abi(gdi_graph_create_pairs(dev, n_, g.csr_offsets().data(), adjacency_pairs(g), &graph_));
    gdi_params q{};
    q.sweeps = params.sweeps;
    q.strategy = params.strategy == Strategy::standard ? GDI_STRATEGY_STANDARD : GDI_STRATEGY_GDI;
    q.mode = params.workers == 1 ? GDI_MODE_EXACT : GDI_MODE_THROUGHPUT;
    q.flags = trace ? GDI_FLAG_TRACE : 0u;
    q.flip_fraction0 = params.flip_fraction0;
    q.decay_rate = params.decay_rate;
    q.a_num = problem.coefficients().a_num;
    q.b_num = problem.coefficients().b_num;
    q.denom = problem.coefficients().denom;
    sweeps_ = q.sweeps;
    trace_ = trace;
    check_abi(gdi_session_create(graph_, &q, replicas, reinterpret_cast<void*>(stream), &sess_));
  }
  ~Session() {
    if (sess_) gdi_session_destroy(sess_);
    if (graph_) gdi_graph_destroy(graph_);
  }
  void set_seeds(py::array_t<std::uint64_t, py::array::c_style | py::array::forcecast> seeds) {
    if (seeds.size() != replicas_) throw config_error("need one seed per replica");
    check_abi(gdi_session_set_seeds(sess_, seeds.data()));
  }
  void launch() { check_abi(gdi_session_launch(sess_)); }
  void sync() {
    py::gil_scoped_release nogil;
    check_abi(gdi_session_sync(sess_));
  }
  py::dict fetch(bool spins, bool trace) {
    const std::size_t R = replicas_, n = n_, S = sweeps_;
    std::vector<std::int8_t> sp(spins ? R * n : 0);
    std::vector<gdi_score> sc(R);
    gdi_trace_rec* tr = trace ? trace_scratch(R * S) : nullptr;
    gdi_outputs out{};
    out.spins = spins ? sp.data() : nullptr;
    out.scores = sc.data();
    out.trace = tr;
    std::vector<std::int64_t> ctr(trace ? R * S : 0);
    out.counters = trace ? ctr.data() : nullptr;
    {
      py::gil_scoped_release nogil;
      check_abi(gdi_session_fetch(sess_, &out));
    }
    py::dict d = pack(std::move(sp), sc, tr, R, n, S, out.seconds, spins, trace);
    // signed balance counter at every barrier (acceptance criterion 4 checks)
    if (trace) d["counters"] = to_numpy(std::move(ctr), {static_cast<py::ssize_t>(R), static_cast<py::ssize_t>(S)});
    return d;
  }
  int launch_count() const {
    std::int32_t c = 0;
    check_abi(gdi_session_launch_count(sess_, &c));
    return c;
  }
  std::string kernel() const { return gdi_session_kernel(sess_); }

  static py::dict pack(std::vector<std::int8_t>&& sp, const std::vector<gdi_score>& sc, const gdi_trace_rec* tr,
                       std::size_t R, std::size_t n, std::size_t S, double seconds, bool spins, bool trace) {
    py::dict d;
    std::vector<std::int64_t> cut(R), imb(R), h(R), ctr(R);
    for (std::size_t r = 0; r < R; r++) {
      cut[r] = sc[r].cut;
      imb[r] = sc[r].imbalance;
      h[r] = sc[r].hamiltonian_scaled;
      ctr[r] = sc[r].balance_counter;
    }
    d["cut"] = to_numpy(std::move(cut), {static_cast<py::ssize_t>(R)});
    d["imbalance"] = to_numpy(std::move(imb), {static_cast<py::ssize_t>(R)});
    d["hamiltonian_scaled"] = to_numpy(std::move(h), {static_cast<py::ssize_t>(R)});
    d["balance_counter"] = to_numpy(std::move(ctr), {static_cast<py::ssize_t>(R)});
    d["seconds"] = seconds;
    if (spins) d["spins"] = to_numpy(std::move(sp), {static_cast<py::ssize_t>(R), static_cast<py::ssize_t>(n)});
    if (trace) {
      // (R, S, 3) int64 = {hamiltonian_scaled, cut, imbalance}; (R, S) seconds;
      // filled row-parallel without the GIL (first touch of ~30 MB of fresh
      // pages dominates a single-threaded fill)
      py::array_t<std::int64_t> t3({static_cast<py::ssize_t>(R), static_cast<py::ssize_t>(S), py::ssize_t{3}});
      py::array_t<double> secs({static_cast<py::ssize_t>(R), static_cast<py::ssize_t>(S)});
      std::vector<double> pf(S);
      std::int64_t* t3p = t3.mutable_data();
      double* sp_ = secs.mutable_data();
      {
        py::gil_scoped_release nogil;
        gdi::parallel_rows(R * S, 64 * 1024, [&](std::size_t lo, std::size_t hi) {
          for (std::size_t i = lo; i < hi; i++) {
            t3p[3 * i] = tr[i].hamiltonian_scaled;
            t3p[3 * i + 1] = tr[i].cut;
            t3p[3 * i + 2] = tr[i].imbalance;
            sp_[i] = tr[i].seconds;
          }
        });
      }
      for (std::size_t k = 0; k < S; k++) pf[k] = tr[k].flip_probability;
      d["trace"] = t3;
      d["trace_seconds"] = secs;
      d["flip_probability"] = to_numpy(std::move(pf), {static_cast<py::ssize_t>(S)});
    }
    return d;
  }

private:
  gdi_graph* graph_ = nullptr;
  gdi_session* sess_ = nullptr;
  std::int32_t n_ = 0;
  int replicas_ = 0;
  int sweeps_ = 0;
  bool trace_ = false;
};

std::vector<Edge> edges_from(const py::iterable& it) {
  std::vector<Edge> out;
  for (py::handle h : it) {
    if (py::isinstance<Edge>(h)) {
      out.push_back(h.cast<Edge>());
    } else {
      auto t = h.cast<py::tuple>();
      out.push_back(Edge{t[0].cast<std::int32_t>(), t[1].cast<std::int32_t>(),
                         t.size() > 2 ? t[2].cast<std::int32_t>() : 1});
    }
  }
  return out;
}

} // namespace

// One rank of a vertex-partitioned anneal (gdi_part_*): the caller moves the
// exchange buffers between ranks (NCCL all-gather, or copies when emulating
// the ranks on one device); buffers are passed as device addresses.
class PartSession {
public:
  PartSession(const MinCutProblem& problem, const AnnealParams& params_in, int world, int rank, std::uint64_t seed,
              std::uintptr_t stream, int dev)
      : n_(problem.graph().num_nodes()) {
    const AnnealParams params = params_in.validated();
    const Graph& g = problem.graph();
    check_abi(gdi_graph_create_pairs(dev, n_, g.csr_offsets().data(), adjacency_pairs(g), &graph_));
    gdi_params q{};
    q.sweeps = params.sweeps;
    q.strategy = params.strategy == Strategy::standard ? GDI_STRATEGY_STANDARD : GDI_STRATEGY_GDI;
    q.mode = GDI_MODE_THROUGHPUT;
    q.flip_fraction0 = params.flip_fraction0;
    q.decay_rate = params.decay_rate;
    q.a_num = problem.coefficients().a_num;
    q.b_num = problem.coefficients().b_num;
    q.denom = problem.coefficients().denom;
    sweeps_ = q.sweeps;
    check_abi(gdi_part_create(graph_, &q, world, rank, seed, reinterpret_cast<void*>(stream), &sess_));
  }
  ~PartSession() {
    if (sess_) gdi_part_destroy(sess_);
    if (graph_) gdi_graph_destroy(graph_);
  }
  std::int64_t exchange_bytes() const {
    std::int64_t b = 0;
    check_abi(gdi_part_exchange_bytes(sess_, &b));
    return b;
  }
  void init() { check_abi(gdi_part_init(sess_)); }
  py::bytes ipc_handle() const {
    char h[GDI_IPC_HANDLE_BYTES];
    check_abi(gdi_part_ipc_handle(sess_, h));
    return py::bytes(h, sizeof h);
  }
  void attach_peers(const py::bytes& handles) {
    const std::string hs = handles;
    check_abi(gdi_part_attach_peers(sess_, hs.data()));
  }
  void detach() { check_abi(gdi_part_detach(sess_)); }
  void attach_local(const std::vector<PartSession*>& parts) {
    std::vector<gdi_part*> ps;
    for (PartSession* q : parts) ps.push_back(q->sess_);
    check_abi(gdi_part_attach_local(sess_, ps.data()));
  }
  void sweep(int k, std::uintptr_t send) { check_abi(gdi_part_sweep(sess_, k, reinterpret_cast<void*>(send))); }
  void finish(int k, std::uintptr_t recv) {
    check_abi(gdi_part_finish(sess_, k, reinterpret_cast<const void*>(recv)));
  }
  py::dict fetch() {
    const std::size_t n = n_, S = sweeps_;
    std::vector<std::int8_t> sp(n);
    std::vector<gdi_score> sc(1);
    std::vector<gdi_trace_rec> tr(S);
    std::vector<std::int64_t> ctr(S);
    gdi_outputs out{};
    out.spins = sp.data();
    out.scores = sc.data();
    out.trace = tr.data();
    out.counters = ctr.data();
    {
      py::gil_scoped_release nogil;
      check_abi(gdi_part_fetch(sess_, &out));
    }
    std::vector<std::int64_t> tcut(S), timb(S);
    for (std::size_t k = 0; k < S; k++) {
      tcut[k] = tr[k].cut;
      timb[k] = tr[k].imbalance;
    }
    py::dict d;
    d["spins"] = to_numpy(std::move(sp), {static_cast<py::ssize_t>(n)});
    d["cut_part"] = sc[0].cut;
    d["imbalance"] = sc[0].imbalance;
    d["balance_counter"] = sc[0].balance_counter;
    d["trace_cut_part"] = to_numpy(std::move(tcut), {static_cast<py::ssize_t>(S)});
    d["trace_imbalance"] = to_numpy(std::move(timb), {static_cast<py::ssize_t>(S)});
    d["counters"] = to_numpy(std::move(ctr), {static_cast<py::ssize_t>(S)});
    d["seconds"] = out.seconds;
    return d;
  }

private:
  gdi_graph* graph_ = nullptr;
  gdi_part* sess_ = nullptr;
  std::int32_t n_ = 0;
  int sweeps_ = 0;
};

py::dict Evaluator::evaluate(py::array_t<std::int8_t, py::array::c_style | py::array::forcecast> spins) {
  if (spins.ndim() != 2 || spins.shape(1) != n_) throw domain_error("spins must have shape (replicas, num_nodes)");
  const auto R = static_cast<std::int32_t>(spins.shape(0));
  std::vector<gdi_score> sc(static_cast<std::size_t>(R));
  {
    py::gil_scoped_release nogil;
    check_abi(gdi_evaluate_batch(graph_, spins.data(), R, c_.a_num, c_.b_num, c_.denom, sc.data()));
  }
  return Session::pack({}, sc, {}, static_cast<std::size_t>(R), 0, 0, 0.0, false, false);
}

PYBIND11_MODULE(pyising, m) {
  m.doc() = "gdi-b200: GDI Ising annealing for balanced min-cut on NVIDIA B200 (sm_100a)";

  py::register_exception<parse_error>(m, "ParseError", PyExc_ValueError);
  py::register_exception<domain_error>(m, "DomainError", PyExc_ValueError);
  py::register_exception<config_error>(m, "ConfigError", PyExc_ValueError);
  py::register_exception<capacity_error>(m, "CapacityError", PyExc_ValueError);

  // ---- graph
  py::class_<Edge>(m, "Edge")
      .def(py::init([](std::int32_t u, std::int32_t v, std::int32_t w) { return Edge{u, v, w}; }),
           py::arg("u"), py::arg("v"), py::arg("weight") = 1)
      .def_readwrite("u", &Edge::u)
      .def_readwrite("v", &Edge::v)
      .def_readwrite("weight", &Edge::weight)
      .def("__repr__", [](const Edge& e) {
        return "Edge(" + std::to_string(e.u) + ", " + std::to_string(e.v) + ", " + std::to_string(e.weight) + ")";
      });

  py::class_<Graph>(m, "Graph")
      .def_static("parse_gset", [](const std::string& text) { return Graph::parse_gset(text); }, py::arg("text"))
      .def_static("parse_gset_file", &Graph::parse_gset_file, py::arg("path"))
      .def_static("from_edges",
                  [](std::int32_t n, const py::iterable& edges) { return Graph::from_edges(n, edges_from(edges)); },
                  py::arg("num_nodes"), py::arg("edges"))
      .def_property_readonly("num_nodes", &Graph::num_nodes)
      .def_property_readonly("num_edges", &Graph::num_edges)
      .def_property_readonly("max_degree", &Graph::max_degree)
      .def_property_readonly("all_unit_weights", &Graph::all_unit_weights)
      .def("degree", &Graph::degree, py::arg("node"))
      .def("neighbors",
           [](const Graph& g, std::int32_t v) {
             if (v < 0 || v >= g.num_nodes()) throw domain_error("node index out of range");
             std::vector<std::pair<std::int32_t, std::int32_t>> out;
             for (const Neighbor& nb : g.neighbors(v)) out.emplace_back(nb.node, nb.weight);
             return out;
           },
           py::arg("node"))
      .def("edges", &Graph::edges)
      .def("to_gset", &Graph::to_gset)
      .def("with_unit_weights", &Graph::with_unit_weights)
      .def("csr",
           [](const Graph& g) {
             std::vector<std::int64_t> off = g.csr_offsets();
             std::vector<std::int32_t> nbr, w;
             for (const Neighbor& nb : g.csr_adjacency()) {
               nbr.push_back(nb.node);
               w.push_back(nb.weight);
             }
             const auto nn = static_cast<py::ssize_t>(nbr.size());
             return py::make_tuple(to_numpy(std::move(off), {static_cast<py::ssize_t>(g.num_nodes()) + 1}),
                                   to_numpy(std::move(nbr), {nn}), to_numpy(std::move(w), {nn}));
           },
           "CSR arrays (offsets int64[n+1], neighbour int32[2m], weight int32[2m])")
      .def("__repr__", [](const Graph& g) {
        return "Graph(num_nodes=" + std::to_string(g.num_nodes()) + ", num_edges=" + std::to_string(g.num_edges()) + ")";
      });

  m.def("density", &density, py::arg("graph"));

  py::class_<Rng>(m, "Rng", "xoshiro256++ (reference rng.hpp), exposed for recipe scripts")
      .def(py::init<std::uint64_t>(), py::arg("seed"))
      .def_static("stream", &Rng::stream, py::arg("seed"), py::arg("stream_id"))
      .def("next", &Rng::next)
      .def("next_unit", &Rng::next_unit)
      .def("coin", &Rng::coin)
      .def("next_below", &Rng::next_below, py::arg("bound"));
  m.def("random_graph", &random_graph, py::arg("n"), py::arg("m"), py::arg("seed"));
  m.def("torus_graph", &torus_graph, py::arg("rows"), py::arg("cols"), py::arg("seed"));
  m.def("random_tree", &random_tree, py::arg("n"), py::arg("seed"));
  m.def("random_connected_gnp", &random_connected_gnp, py::arg("n"), py::arg("p"), py::arg("seed"));

  // ---- model
  py::class_<Coefficients>(m, "Coefficients")
      .def(py::init([](std::int64_t a, std::int64_t b, std::int64_t d) { return Coefficients{a, b, d}; }),
           py::arg("a_num") = 1, py::arg("b_num") = 1, py::arg("denom") = 1)
      .def_readwrite("a_num", &Coefficients::a_num)
      .def_readwrite("b_num", &Coefficients::b_num)
      .def_readwrite("denom", &Coefficients::denom)
      .def_property_readonly("a", &Coefficients::a)
      .def_property_readonly("b", &Coefficients::b)
      .def("__repr__", [](const Coefficients& c) {
        return "Coefficients(a=" + std::to_string(c.a()) + ", b=" + std::to_string(c.b()) + ")";
      });
  m.def("coefficients_for", &coefficients_for, py::arg("graph"), py::arg("b_num") = 1, py::arg("b_den") = 1);
  m.def("solver_default_coefficients", &solver_default_coefficients);

  py::class_<MinCutProblem>(m, "MinCutProblem")
      .def_static("make", &MinCutProblem::make, py::arg("graph"), py::arg("coefficients"),
                  py::arg("external_field") = std::vector<std::int64_t>{})
      .def_static("make_unchecked", &MinCutProblem::make_unchecked, py::arg("graph"), py::arg("coefficients"),
                  py::arg("external_field") = std::vector<std::int64_t>{})
      .def_static("with_default_coefficients", &MinCutProblem::with_default_coefficients, py::arg("graph"))
      .def_property_readonly("graph", &MinCutProblem::graph, py::return_value_policy::reference_internal)
      .def_property_readonly("coefficients", &MinCutProblem::coefficients)
      .def("satisfies_coefficient_rule", &MinCutProblem::satisfies_coefficient_rule);

  m.def("local_field", &local_field, py::arg("problem"), py::arg("state"), py::arg("node"));
  py::class_<CandidateEnergies>(m, "CandidateEnergies")
      .def_readonly("at_minus_scaled", &CandidateEnergies::at_minus_scaled)
      .def_readonly("at_plus_scaled", &CandidateEnergies::at_plus_scaled)
      .def_readonly("denom", &CandidateEnergies::denom)
      .def_property_readonly("at_minus", &CandidateEnergies::at_minus)
      .def_property_readonly("at_plus", &CandidateEnergies::at_plus);
  m.def("candidate_energies_mincut", &candidate_energies_mincut, py::arg("problem"), py::arg("state"),
        py::arg("balance_excl"), py::arg("node"));
  m.def("global_hamiltonian", &global_hamiltonian, py::arg("problem"), py::arg("state"));
  m.def("global_hamiltonian_scaled", &global_hamiltonian_scaled, py::arg("problem"), py::arg("state"));

  // ---- evaluation
  m.def("cut_value", &cut_value, py::arg("graph"), py::arg("state"));
  m.def("imbalance", &imbalance, py::arg("state"));
  py::class_<PartitionScore>(m, "PartitionScore")
      .def_readonly("cut", &PartitionScore::cut)
      .def_readonly("imbalance", &PartitionScore::imbalance)
      .def_readonly("hamiltonian_scaled", &PartitionScore::hamiltonian_scaled)
      .def_readonly("hamiltonian", &PartitionScore::hamiltonian)
      .def("__repr__", [](const PartitionScore& s) {
        return "PartitionScore(cut=" + std::to_string(s.cut) + ", imbalance=" + std::to_string(s.imbalance) + ")";
      });
  m.def("score", &score, py::arg("problem"), py::arg("state"));
  py::class_<OracleResult>(m, "OracleResult")
      .def_readonly("cut", &OracleResult::cut)
      .def_readonly("witness", &OracleResult::witness);
  m.def("brute_force_balanced_mincut", &brute_force_balanced_mincut, py::arg("graph"), py::arg("max_imbalance"));
  m.attr("ORACLE_MAX_NODES") = kOracleMaxNodes;

  // ---- annealing
  py::enum_<Strategy>(m, "Strategy").value("standard", Strategy::standard).value("gdi", Strategy::gdi);
  py::class_<AnnealParams>(m, "AnnealParams")
      .def(py::init<>())
      .def_readwrite("sweeps", &AnnealParams::sweeps)
      .def_readwrite("flip_fraction0", &AnnealParams::flip_fraction0)
      .def_readwrite("decay_rate", &AnnealParams::decay_rate)
      .def_readwrite("strategy", &AnnealParams::strategy)
      .def_readwrite("workers", &AnnealParams::workers)
      .def_readwrite("seed", &AnnealParams::seed)
      .def_readwrite("deterministic", &AnnealParams::deterministic)
      .def("validated", &AnnealParams::validated);
  m.def("default_params_for", &default_params_for, py::arg("strategy"), py::arg("graph"));
  m.def("flip_probability", &flip_probability, py::arg("params"), py::arg("sweep_index"));
  m.def("strategy_from_string", &strategy_from_string, py::arg("name"));

  py::class_<TraceRecord>(m, "TraceRecord")
      .def_readonly("hamiltonian_scaled", &TraceRecord::hamiltonian_scaled)
      .def_readonly("hamiltonian", &TraceRecord::hamiltonian)
      .def_readonly("cut", &TraceRecord::cut)
      .def_readonly("imbalance", &TraceRecord::imbalance)
      .def_readonly("flip_probability", &TraceRecord::flip_probability)
      .def_readonly("seconds", &TraceRecord::seconds);
  py::class_<AnnealResult>(m, "AnnealResult")
      .def_readonly("state", &AnnealResult::state)
      .def_readonly("trace", &AnnealResult::trace)
      .def_readonly("seconds", &AnnealResult::seconds);

  m.def(
      "anneal",
      [](const MinCutProblem& problem, const AnnealParams& params, py::object on_sweep_end, py::object on_update) {
        AnnealHooks hooks;
        const bool any = !on_sweep_end.is_none() || !on_update.is_none();
        if (!on_sweep_end.is_none())
          hooks.on_sweep_end = [on_sweep_end](std::int32_t k, std::span<const Spin> s, std::int64_t c) {
            py::gil_scoped_acquire gil;
            on_sweep_end(k, std::vector<Spin>(s.begin(), s.end()), c);
          };
        if (!on_update.is_none())
          hooks.on_update = [on_update](std::int32_t i, std::span<const Spin> s) {
            py::gil_scoped_acquire gil;
            on_update(i, std::vector<Spin>(s.begin(), s.end()));
          };
        py::gil_scoped_release nogil;
        return anneal(problem, params, any ? &hooks : nullptr);
      },
      py::arg("problem"), py::arg("params"), py::arg("on_sweep_end") = py::none(), py::arg("on_update") = py::none());

  m.def(
      "anneal_batch",
      [](const MinCutProblem& problem, const AnnealParams& params,
         py::array_t<std::uint64_t, py::array::c_style | py::array::forcecast> seeds, bool trace) {
        std::vector<std::uint64_t> sd(seeds.data(), seeds.data() + seeds.size());
        BatchResult b;
        {
          py::gil_scoped_release nogil;
          b = anneal_batch(problem, params, sd, trace);
        }
        const std::size_t R = b.runs.size(), n = static_cast<std::size_t>(problem.graph().num_nodes());
        const std::size_t S = trace ? static_cast<std::size_t>(params.sweeps) : 0;
        std::vector<std::int8_t> sp(R * n);
        std::vector<gdi_score> sc(R);
        gdi_trace_rec* tr = trace_scratch(R * S);
        for (std::size_t r = 0; r < R; r++) {
          std::copy(b.runs[r].state.begin(), b.runs[r].state.end(), sp.begin() + r * n);
          const PartitionScore& p = b.scores[r];
          sc[r] = gdi_score{p.cut, p.imbalance, p.hamiltonian_scaled, p.hamiltonian, 0};
          for (std::size_t k = 0; k < S; k++) {
            const TraceRecord& t = b.runs[r].trace[k];
            tr[r * S + k] = gdi_trace_rec{t.hamiltonian_scaled, t.hamiltonian, t.cut, t.imbalance, t.flip_probability, t.seconds};
          }
        }
        return Session::pack(std::move(sp), sc, tr, R, n, S, b.seconds, true, trace);
      },
      py::arg("problem"), py::arg("params"), py::arg("seeds"), py::arg("trace") = false,
      "One device launch for len(seeds) replicas; returns numpy spins/scores (and trace).");

  m.def(
      "anneal_batch_fresh",
      [](const MinCutProblem& problem, const AnnealParams& params_in,
         py::array_t<std::uint64_t, py::array::c_style | py::array::forcecast> seeds, bool trace) {
        // End-to-end C-ABI path with host buffers and no device caching:
        // CSR upload (gdi_graph_create), seeds H2D, kernel, spins + scores
        // (+ trace) D2H, device buffers released — every call. The trace is
        // written by the library straight into the returned numpy columns
        // (gdi_anneal_batch_columns: one conversion pass).
        const AnnealParams params = params_in.validated();
        const Graph& g = problem.graph();
        const std::size_t R = static_cast<std::size_t>(seeds.size());
        const std::size_t n = static_cast<std::size_t>(g.num_nodes()), S = static_cast<std::size_t>(params.sweeps);
        std::vector<std::int8_t> sp(R * n);
        std::vector<gdi_score> sc(R);
        py::array_t<std::int64_t> t3;
        py::array_t<double> secs_a, pf_a;
        gdi_trace_columns cols{};
        if (trace) {
          t3 = py::array_t<std::int64_t>({static_cast<py::ssize_t>(R), static_cast<py::ssize_t>(S), py::ssize_t{3}});
          secs_a = py::array_t<double>({static_cast<py::ssize_t>(R), static_cast<py::ssize_t>(S)});
          pf_a = py::array_t<double>({static_cast<py::ssize_t>(S)});
          cols.hcut_imb = t3.mutable_data();
          cols.seconds = secs_a.mutable_data();
          cols.flip_probability = pf_a.mutable_data();
        }
        double secs = 0.0;
        std::vector<std::uint64_t> sd(seeds.data(), seeds.data() + R);
        {
          py::gil_scoped_release nogil;
          gdi_graph* dg = nullptr;
          check_abi(gdi_graph_create_pairs(device(), g.num_nodes(), g.csr_offsets().data(), adjacency_pairs(g), &dg));
          gdi_params q{};
          q.sweeps = params.sweeps;
          q.strategy = params.strategy == Strategy::standard ? GDI_STRATEGY_STANDARD : GDI_STRATEGY_GDI;
          q.mode = params.workers == 1 ? GDI_MODE_EXACT : GDI_MODE_THROUGHPUT;
          q.flip_fraction0 = params.flip_fraction0;
          q.decay_rate = params.decay_rate;
          q.a_num = problem.coefficients().a_num;
          q.b_num = problem.coefficients().b_num;
          q.denom = problem.coefficients().denom;
          gdi_outputs out{};
          out.spins = sp.data();
          out.scores = sc.data();
          const int rc = gdi_anneal_batch_columns(dg, &q, sd.data(), static_cast<std::int32_t>(R), &out,
                                                  trace ? &cols : nullptr);
          gdi_graph_destroy(dg);
          check_abi(rc);
          secs = out.seconds;
        }
        py::dict d = Session::pack(std::move(sp), sc, nullptr, R, n, 0, secs, true, false);
        if (trace) {
          d["trace"] = t3;
          d["trace_seconds"] = secs_a;
          d["flip_probability"] = pf_a;
        }
        return d;
      },
      py::arg("problem"), py::arg("params"), py::arg("seeds"), py::arg("trace") = true);

  m.def(
      "evaluate_batch",
      [](const MinCutProblem& problem, py::array_t<std::int8_t, py::array::c_style | py::array::forcecast> spins) {
        const Graph& g = problem.graph();
        if (spins.ndim() != 2 || spins.shape(1) != g.num_nodes())
          throw domain_error("spins must have shape (replicas, num_nodes)");
        const auto R = static_cast<std::int32_t>(spins.shape(0));
        std::vector<gdi_score> sc(static_cast<std::size_t>(R));
        const Coefficients& c = problem.coefficients();
        {
          py::gil_scoped_release nogil;
          gdi_graph* dg = nullptr;
          check_abi(gdi_graph_create_pairs(device(), g.num_nodes(), g.csr_offsets().data(), adjacency_pairs(g), &dg));
          const int rc = gdi_evaluate_batch(dg, spins.data(), R, c.a_num, c.b_num, c.denom, sc.data());
          gdi_graph_destroy(dg);
          check_abi(rc);
        }
        return Session::pack({}, sc, {}, static_cast<std::size_t>(R), 0, 0, 0.0, false, false);
      },
      py::arg("problem"), py::arg("spins"), "K3 fused exact cut/imbalance/H of (R, n) spin rows on the device.");

  // a device graph kept for repeated K3 evaluations (gdi_evaluate_batch on
  // host spins, gdi_evaluate_device on device pointers)
  py::class_<Evaluator>(m, "Evaluator")
      .def(py::init<const MinCutProblem&, int>(), py::arg("problem"), py::arg("device") = 0)
      .def("evaluate", &Evaluator::evaluate, py::arg("spins"))
      .def("evaluate_device", &Evaluator::evaluate_device, py::arg("spins_ptr"), py::arg("replicas"),
           py::arg("cut_sum_ptr"), py::arg("bad_ptr") = 0, py::arg("stream") = 0,
           "Enqueue K3 on device int8 spins [R][n]; writes int64 {cut, sum} per replica to cut_sum_ptr.");

  py::class_<Session>(m, "Session")
      .def(py::init<const MinCutProblem&, const AnnealParams&, int, std::uintptr_t, bool, int>(), py::arg("problem"),
           py::arg("params"), py::arg("replicas"), py::arg("stream") = 0, py::arg("trace") = false,
           py::arg("device") = 0)
      .def("set_seeds", &Session::set_seeds, py::arg("seeds"))
      .def("launch", &Session::launch)
      .def("sync", &Session::sync)
      .def("fetch", &Session::fetch, py::arg("spins") = true, py::arg("trace") = false)
      .def_property_readonly("launch_count", &Session::launch_count)
      .def_property_readonly("kernel", &Session::kernel);

  // batched callers (include/ising/bench.hpp; reference bench.hpp run_benchmark)
  py::class_<BenchConfig>(m, "BenchConfig")
      .def(py::init<>())
      .def_readwrite("graph_paths", &BenchConfig::graph_paths)
      .def_readwrite("strategies", &BenchConfig::strategies)
      .def_readwrite("runs_per_graph", &BenchConfig::runs_per_graph)
      .def_readwrite("base_seed", &BenchConfig::base_seed)
      .def_readwrite("unit_weights", &BenchConfig::unit_weights)
      .def_property(
          "sweeps", [](const BenchConfig& c) { return c.overrides.sweeps; },
          [](BenchConfig& c, std::optional<std::int32_t> v) { c.overrides.sweeps = v; })
      .def_property(
          "flip_fraction0", [](const BenchConfig& c) { return c.overrides.flip_fraction0; },
          [](BenchConfig& c, std::optional<double> v) { c.overrides.flip_fraction0 = v; })
      .def_property(
          "workers", [](const BenchConfig& c) { return c.overrides.workers; },
          [](BenchConfig& c, std::optional<std::int32_t> v) { c.overrides.workers = v; });
  py::class_<RunReport>(m, "RunReport")
      .def_readonly("graph_id", &RunReport::graph_id)
      .def_readonly("nodes", &RunReport::nodes)
      .def_readonly("edges", &RunReport::edges)
      .def_readonly("density", &RunReport::density)
      .def_readonly("strategy", &RunReport::strategy)
      .def_readonly("best_cut", &RunReport::best_cut)
      .def_readonly("best_imbalance", &RunReport::best_imbalance)
      .def_readonly("cut_mean", &RunReport::cut_mean)
      .def_readonly("cut_min", &RunReport::cut_min)
      .def_readonly("cut_max", &RunReport::cut_max)
      .def_readonly("run_seconds", &RunReport::run_seconds)
      .def_readonly("seeds", &RunReport::seeds)
      .def_readonly("error", &RunReport::error);
  m.def(
      "run_benchmark",
      [](const BenchConfig& c) {
        py::gil_scoped_release nogil;
        return run_benchmark(c);
      },
      py::arg("config"), "Reference run_benchmark rows, one device launch per (graph, strategy) row.");
  py::class_<BestOfRuns>(m, "BestOfRuns")
      .def_readonly("best", &BestOfRuns::best)
      .def_readonly("score", &BestOfRuns::score)
      .def_readonly("seed", &BestOfRuns::seed)
      .def_readonly("scores", &BestOfRuns::scores);
  m.def(
      "anneal_best_of",
      [](const MinCutProblem& p, const AnnealParams& params, int runs) {
        py::gil_scoped_release nogil;
        return anneal_best_of(p, params, runs);
      },
      py::arg("problem"), py::arg("params"), py::arg("runs"),
      "solve --runs as one launch: lowest H, first seed on ties (ising_cli.cpp:148-166).");

  py::class_<PartSession>(m, "PartSession",
                          "One rank of a vertex-partitioned throughput-mode anneal (C ABI gdi_part_*).")
      .def(py::init<const MinCutProblem&, const AnnealParams&, int, int, std::uint64_t, std::uintptr_t, int>(),
           py::arg("problem"), py::arg("params"), py::arg("world"), py::arg("rank"), py::arg("seed"),
           py::arg("stream") = 0, py::arg("device") = 0)
      .def_property_readonly("exchange_bytes", &PartSession::exchange_bytes)
      .def("init", &PartSession::init)
      .def("ipc_handle", &PartSession::ipc_handle, "this rank's spin copy as a CUDA IPC handle (bytes)")
      .def("attach_peers", &PartSession::attach_peers, py::arg("handles"),
           "fused exchange: every rank's ipc_handle(), rank-major, concatenated")
      .def("detach", &PartSession::detach,
           "close the peers' IPC mappings (call on every rank, then barrier, before dropping the session)")
      .def("attach_local", &PartSession::attach_local, py::arg("parts"),
           "fused exchange between partitions of this process on one device (testing)")
      .def("sweep", &PartSession::sweep, py::arg("k"), py::arg("send"))
      .def("finish", &PartSession::finish, py::arg("k"), py::arg("recv"))
      .def("fetch", &PartSession::fetch);

  m.def(
      "probe_l2_bandwidth",
      [](std::int64_t bytes, int iters) {
        double gbs = 0.0;
        check_abi(gdi_probe_l2_bandwidth(device(), bytes, iters, &gbs));
        return gbs;
      },
      py::arg("bytes") = 48LL << 20, py::arg("iters") = 50,
      "Sustained read GB/s of an L2-resident buffer on the current device (roofline denominator).");
  m.def("set_device", &set_device, py::arg("device"));
  m.def("device", &device);
  m.def("device_count", []() {
    int c = 0;
    gdi_device_count(&c);
    return c;
  });
  m.attr("ABI_VERSION") = gdi_abi_version();
}
