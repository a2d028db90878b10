// Graph construction, G-set text I/O and canonical serialisation.
// Behaviour (accepted syntax, error classes, line numbers, canonical order)
// follows reference proj/src/graph.cpp:46-174; the implementation parses the
// input buffer in parallel (one piece of whole lines per host thread) and
// checks duplicates by hash-partitioned buckets, instead of getline +
// std::unordered_set.
#include <algorithm>
#include <charconv>
#include <fstream>
#include <istream>
#include <iterator>
#include <limits>
#include <sstream>
#include <thread>

#include "ising/ising.hpp"
#include "pairset.hpp"
#include "parallel.hpp"

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

// One piece of the body (whole lines): its edges, its line count and its
// first malformed line (local line number, message).
struct Piece {
  std::vector<Edge> edges;
  long lines = 0;
  long err_line = 0;  // 0: none
  std::string err;
};

void parse_piece(std::string_view text, long long n, Piece& out) {
  LineReader rd(text);
  std::string_view line;
  while (rd.next(line)) {
    if (skippable(line)) continue;
    long long t[3];
    const char* msg = nullptr;
    std::string range_msg;
    if (!read_ints(line, t, 3)) {
      msg = "edge line must be \"u v w\"";
    } else if (t[0] < 1 || t[0] > n || t[1] < 1 || t[1] > n) {
      range_msg = "endpoint out of range [1, " + std::to_string(n) + "]";
    } else if (t[0] == t[1]) {
      msg = "self-loop";
    } else if (t[2] < std::numeric_limits<std::int32_t>::min() || t[2] > std::numeric_limits<std::int32_t>::max()) {
      msg = "weight out of range";
    }
    if (msg != nullptr || !range_msg.empty()) {
      out.err_line = rd.number();
      out.err = msg != nullptr ? std::string(msg) : range_msg;
      out.lines = rd.number();
      return;
    }
    out.edges.push_back({static_cast<std::int32_t>(t[0] - 1), static_cast<std::int32_t>(t[1] - 1),
                         static_cast<std::int32_t>(t[2])});
  }
  out.lines = rd.number();
}

// Local line number of the k-th edge line of a piece (error path only).
long edge_line(std::string_view text, std::size_t k) {
  LineReader rd(text);
  std::string_view line;
  std::size_t seen = 0;
  while (rd.next(line)) {
    if (skippable(line)) continue;
    if (seen++ == k) return rd.number();
  }
  return rd.number();
}

} // namespace

namespace detail {

// The body is cut at newlines into one piece per host thread and parsed in
// parallel; the duplicate check partitions the edges by key hash (one bucket
// per thread, each bucket scanned in file order). The error reported is the
// reference's: the first offending line in file order, with its line number.
Graph parse_gset_text(std::string_view text) {
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
  const std::size_t body0 = static_cast<std::size_t>(line.data() + line.size() - text.data()) + 1;
  const std::string_view body = body0 < text.size() ? text.substr(body0) : std::string_view{};

  // pieces: [cut[t], cut[t+1]), each starting at a line start
  unsigned T = std::thread::hardware_concurrency();
  T = T < 1 ? 1 : T > 16 ? 16 : T;
  if (body.size() < (1u << 20)) T = 1;
  std::vector<std::size_t> cut(T + 1, body.size());
  cut[0] = 0;
  for (unsigned t = 1; t < T; t++) {
    std::size_t p = std::max(cut[t - 1], body.size() * t / T);
    while (p < body.size() && p > 0 && body[p - 1] != '\n') p++;
    cut[t] = p;
  }
  std::vector<Piece> pieces(T);
  gdi::parallel_rows(T, 2, [&](std::size_t t0, std::size_t t1) {
    for (std::size_t t = t0; t < t1; t++) parse_piece(body.substr(cut[t], cut[t + 1] - cut[t]), n, pieces[t]);
  });
  // the first malformed line in file order (pieces after it are not used)
  long base = head_line;
  unsigned used = T;
  long syntax_line = 0;
  std::string syntax_msg;
  std::vector<long> first_line(T);
  for (unsigned t = 0; t < T; t++) {
    first_line[t] = base;
    if (pieces[t].err_line != 0) {
      syntax_line = base + pieces[t].err_line;
      syntax_msg = pieces[t].err;
      used = t + 1;
      break;
    }
    base += pieces[t].lines;
  }
  std::vector<std::size_t> eoff(used + 1, 0);
  for (unsigned t = 0; t < used; t++) eoff[t + 1] = eoff[t] + pieces[t].edges.size();
  const std::size_t ne = eoff[used];
  std::vector<Edge> edges(ne);
  gdi::parallel_rows(used, 2, [&](std::size_t t0, std::size_t t1) {
    for (std::size_t t = t0; t < t1; t++) std::copy(pieces[t].edges.begin(), pieces[t].edges.end(), edges.begin() + eoff[t]);
  });

  // duplicates: (key, index) scattered into per-bucket runs, in file order
  // within a bucket; bucket b is then checked by one thread
  const unsigned B = T;
  auto bucket = [B](std::uint64_t k) {
    const std::uint64_t h = k * 0x9e3779b97f4a7c15ULL;
    return static_cast<unsigned>((h >> 32) % B);
  };
  std::size_t dup = ne;  // index of the first edge repeating an earlier one
  if (ne > 1) {
    std::vector<std::size_t> cnt(static_cast<std::size_t>(T) * B, 0);
    gdi::parallel_rows(T, 2, [&](std::size_t t0, std::size_t t1) {
      for (std::size_t t = t0; t < t1; t++)
        for (std::size_t i = ne * t / T; i < ne * (t + 1) / T; i++)
          cnt[t * B + bucket(PairSet::key(edges[i].u, edges[i].v))]++;
    });
    std::vector<std::size_t> start(static_cast<std::size_t>(T) * B);
    std::vector<std::size_t> bstart(B + 1, 0);
    std::size_t acc = 0;
    for (unsigned b = 0; b < B; b++) {
      bstart[b] = acc;
      for (unsigned t = 0; t < T; t++) {
        start[t * B + b] = acc;
        acc += cnt[t * B + b];
      }
    }
    bstart[B] = acc;
    std::vector<std::pair<std::uint64_t, std::size_t>> keyed(ne);
    gdi::parallel_rows(T, 2, [&](std::size_t t0, std::size_t t1) {
      for (std::size_t t = t0; t < t1; t++) {
        std::vector<std::size_t> pos(start.begin() + t * B, start.begin() + (t + 1) * B);
        for (std::size_t i = ne * t / T; i < ne * (t + 1) / T; i++) {
          const std::uint64_t k = PairSet::key(edges[i].u, edges[i].v);
          keyed[pos[bucket(k)]++] = {k, i};
        }
      }
    });
    std::vector<std::size_t> first_dup(B, ne);
    gdi::parallel_rows(B, 2, [&](std::size_t b0, std::size_t b1) {
      for (std::size_t b = b0; b < b1; b++) {
        PairSet seen(bstart[b + 1] - bstart[b]);
        for (std::size_t i = bstart[b]; i < bstart[b + 1]; i++)
          if (!seen.insert(keyed[i].first)) {
            first_dup[b] = keyed[i].second;
            break;
          }
      }
    });
    dup = *std::min_element(first_dup.begin(), first_dup.end());
  }
  if (dup < ne) {
    unsigned t = 0;
    while (eoff[t + 1] <= dup) t++;
    const long dup_line = first_line[t] + edge_line(body.substr(cut[t], cut[t + 1] - cut[t]), dup - eoff[t]);
    if (syntax_line == 0 || dup_line < syntax_line) throw parse_error("duplicate edge", dup_line);
  }
  if (syntax_line != 0) throw parse_error(syntax_msg, syntax_line);
  if (static_cast<long long>(ne) != m)
    throw parse_error("header announces " + std::to_string(m) + " edges, found " + std::to_string(ne));
  return Graph::build(static_cast<std::int32_t>(n), edges, false);
}

}  // namespace detail

Graph Graph::from_edges(std::int32_t num_nodes, std::span<const Edge> edges) {
  return build(num_nodes, edges, true);
}

Graph Graph::build(std::int32_t num_nodes, std::span<const Edge> edges, bool check) {
  if (num_nodes <= 0) throw domain_error("graph needs a positive node count");
  Graph g;
  g.n_ = num_nodes;
  g.m_ = static_cast<std::int64_t>(edges.size());
  std::vector<std::int64_t> deg(static_cast<std::size_t>(num_nodes) + 1, 0);
  if (check) {
    detail::PairSet seen(edges.size());
    for (const Edge& e : edges) {
      if (e.u < 0 || e.u >= num_nodes || e.v < 0 || e.v >= num_nodes)
        throw domain_error("edge endpoint out of range");
      if (e.u == e.v) throw domain_error("self-loop");
      if (!seen.insert(detail::PairSet::key(e.u, e.v))) throw domain_error("duplicate edge");
    }
  }
  for (const Edge& e : edges) {
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
  return detail::parse_gset_text(text);
}

Graph Graph::parse_gset(const std::string& text) { return detail::parse_gset_text(text); }

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
