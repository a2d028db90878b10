// Graph construction, G-set text I/O and canonical serialisation.
// Behaviour (accepted syntax, error classes, line numbers, canonical order)
// follows reference proj/src/graph.cpp:46-174; the implementation scans the
// whole input buffer once instead of getline + std::unordered_set.
#include <algorithm>
#include <charconv>
#include <fstream>
#include <istream>
#include <iterator>
#include <limits>
#include <sstream>

#include "ising/ising.hpp"
#include "pairset.hpp"

namespace ising {

namespace {

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r'; }

// Blank or comment ('%' / '#' first non-blank) lines are skipped
// (graph.cpp:22-28).
bool skippable(std::string_view line) {
  for (char c : line) {
    if (is_space(c)) continue;
    return c == '%' || c == '#';
  }
  return true;
}

// Exactly `count` integers separated by blanks and nothing else
// (graph.cpp:31-42: std::from_chars semantics, no leading '+').
bool read_ints(std::string_view line, long long* out, int count) {
  const char* p = line.data();
  const char* end = p + line.size();
  for (int k = 0; k < count; k++) {
    while (p < end && is_space(*p)) p++;
    auto [q, ec] = std::from_chars(p, end, out[k]);
    if (ec != std::errc{} || q == p) return false;
    p = q;
  }
  while (p < end && is_space(*p)) p++;
  return p == end;
}

// Splits text into getline-equivalent lines: '\n' separated, no trailing
// empty line after a final newline.
class LineReader {
public:
  explicit LineReader(std::string_view text) : text_(text) {}
  bool next(std::string_view& line) {
    if (pos_ >= text_.size()) return false;
    std::size_t nl = text_.find('\n', pos_);
    if (nl == std::string_view::npos) nl = text_.size();
    line = text_.substr(pos_, nl - pos_);
    pos_ = nl + 1;
    number_++;
    return true;
  }
  long number() const { return number_; }

private:
  std::string_view text_;
  std::size_t pos_ = 0;
  long number_ = 0;
};

Graph parse_text(std::string_view text) {
  LineReader rd(text);
  std::string_view line;
  long long head[2];
  for (;;) {
    if (!rd.next(line)) throw parse_error("missing header line", rd.number());
    if (skippable(line)) continue;
    if (!read_ints(line, head, 2)) throw parse_error("header must be two integers \"N M\"", rd.number());
    break;
  }
  const long long n = head[0], m = head[1];
  const long head_line = rd.number();
  if (n <= 0) throw parse_error("node count must be positive", head_line);
  if (m < 0) throw parse_error("edge count must be non-negative", head_line);
  if (n > std::numeric_limits<std::int32_t>::max()) throw parse_error("node count too large", head_line);

  std::vector<Edge> edges;
  edges.reserve(static_cast<std::size_t>(std::min<long long>(m, 1LL << 26)));
  detail::PairSet seen(static_cast<std::size_t>(std::min<long long>(m, 1LL << 26)));
  while (rd.next(line)) {
    if (skippable(line)) continue;
    long long t[3];
    if (!read_ints(line, t, 3)) throw parse_error("edge line must be \"u v w\"", rd.number());
    if (t[0] < 1 || t[0] > n || t[1] < 1 || t[1] > n)
      throw parse_error("endpoint out of range [1, " + std::to_string(n) + "]", rd.number());
    if (t[0] == t[1]) throw parse_error("self-loop", rd.number());
    if (t[2] < std::numeric_limits<std::int32_t>::min() || t[2] > std::numeric_limits<std::int32_t>::max())
      throw parse_error("weight out of range", rd.number());
    const auto u = static_cast<std::int32_t>(t[0] - 1), v = static_cast<std::int32_t>(t[1] - 1);
    if (!seen.insert(detail::PairSet::key(u, v))) throw parse_error("duplicate edge", rd.number());
    edges.push_back({u, v, static_cast<std::int32_t>(t[2])});
  }
  if (static_cast<long long>(edges.size()) != m)
    throw parse_error("header announces " + std::to_string(m) + " edges, found " +
                      std::to_string(edges.size()));
  return Graph::from_edges(static_cast<std::int32_t>(n), edges);
}

} // namespace

Graph Graph::from_edges(std::int32_t num_nodes, std::span<const Edge> edges) {
  if (num_nodes <= 0) throw domain_error("graph needs a positive node count");
  Graph g;
  g.n_ = num_nodes;
  g.m_ = static_cast<std::int64_t>(edges.size());
  std::vector<std::int64_t> deg(static_cast<std::size_t>(num_nodes) + 1, 0);
  detail::PairSet seen(edges.size());
  for (const Edge& e : edges) {
    if (e.u < 0 || e.u >= num_nodes || e.v < 0 || e.v >= num_nodes)
      throw domain_error("edge endpoint out of range");
    if (e.u == e.v) throw domain_error("self-loop");
    if (!seen.insert(detail::PairSet::key(e.u, e.v))) throw domain_error("duplicate edge");
    deg[e.u + 1]++;
    deg[e.v + 1]++;
    g.unit_ = g.unit_ && e.weight == 1;
  }
  // Prefix sum -> offsets; rows filled in edge order (graph.cpp:67-77).
  for (std::int32_t i = 0; i < num_nodes; i++) {
    g.max_deg_ = std::max(g.max_deg_, static_cast<std::int32_t>(deg[i + 1]));
    deg[i + 1] += deg[i];
  }
  g.offsets_ = deg;
  g.adj_.resize(2 * edges.size());
  std::vector<std::int64_t> cursor(g.offsets_.begin(), g.offsets_.end() - 1);
  for (const Edge& e : edges) {
    g.adj_[cursor[e.u]++] = Neighbor{e.v, e.weight};
    g.adj_[cursor[e.v]++] = Neighbor{e.u, e.weight};
  }
  return g;
}

Graph Graph::parse_gset(std::istream& in) {
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return parse_text(text);
}

Graph Graph::parse_gset(const std::string& text) { return parse_text(text); }

Graph Graph::parse_gset_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw parse_error("cannot open " + path);
  return parse_gset(in);
}

std::vector<Edge> Graph::edges() const {
  std::vector<Edge> out;
  out.reserve(static_cast<std::size_t>(m_));
  std::vector<Neighbor> row;
  for (std::int32_t u = 0; u < n_; u++) {
    row.clear();
    for (const Neighbor& nb : neighbors(u))
      if (nb.node > u) row.push_back(nb);
    std::sort(row.begin(), row.end(), [](const Neighbor& a, const Neighbor& b) { return a.node < b.node; });
    for (const Neighbor& nb : row) out.push_back(Edge{u, nb.node, nb.weight});
  }
  return out;
}

std::string Graph::to_gset() const {
  std::string s;
  s.reserve(static_cast<std::size_t>(m_) * 16 + 32);
  char buf[64];
  auto put = [&](long long v, char sep) {
    auto [p, ec] = std::to_chars(buf, buf + sizeof buf, v);
    (void)ec;
    s.append(buf, p);
    s.push_back(sep);
  };
  put(n_, ' ');
  put(m_, '\n');
  for (const Edge& e : edges()) {
    put(e.u + 1LL, ' ');
    put(e.v + 1LL, ' ');
    put(e.weight, '\n');
  }
  return s;
}

Graph Graph::with_unit_weights() const {
  Graph g = *this;
  for (Neighbor& nb : g.adj_) nb.weight = 1;
  g.unit_ = true;
  g.dev_.reset(); // different weights: never share the device copy
  return g;
}

double density(const Graph& g) {
  if (g.num_nodes() < 2) throw domain_error("density needs at least 2 nodes");
  const double n = g.num_nodes();
  return 2.0 * static_cast<double>(g.num_edges()) / (n * (n - 1.0));
}

} // namespace ising
