// Graph ingestion (see include/mgg/graph.hpp for the contract).
#include "mgg/graph.hpp"

#include <algorithm>
#include <atomic>
#include <bit>
#include <cmath>
#include <cstring>
#include <istream>
#include <iterator>
#include <ostream>
#include <string>

#include "mgg/errors.hpp"
#include "mgg/rng.hpp"
#include "parallel.hpp"

namespace mgg {

using detail::parallel_for;

std::uint64_t CsrGraph::max_degree() const {
  std::uint64_t m = 0;
  for (std::uint64_t v = 0; v < num_nodes; ++v) m = std::max(m, degree(v));
  return m;
}

void validate_csr(const CsrGraph& g) {
  if (g.row_ptr.size() != g.num_nodes + 1)
    throw InputError("csr: row_ptr length must be num_nodes + 1");
  if (g.row_ptr.front() != 0) throw InputError("csr: row_ptr[0] must be 0");
  if (g.row_ptr.back() != g.col_idx.size())
    throw InputError("csr: row_ptr[num_nodes] must equal num_edges");
  std::atomic<int> bad{0};
  parallel_for(g.num_nodes, 1 << 16, [&](std::uint64_t b, std::uint64_t e) {
    for (std::uint64_t i = b; i < e; ++i)
      if (g.row_ptr[i + 1] < g.row_ptr[i]) bad |= 1;
  });
  if (bad) throw InputError("csr: row_ptr must be non-decreasing");
  parallel_for(g.col_idx.size(), 1 << 20, [&](std::uint64_t b, std::uint64_t e) {
    for (std::uint64_t i = b; i < e; ++i)
      if (g.col_idx[i] >= g.num_nodes) bad |= 2;
  });
  if (bad) throw InputError("csr: col_idx entry out of range");
}

namespace {

// Sort every row of a CSR whose row_ptr is final (rows in parallel).
void sort_rows(CsrGraph& g) {
  parallel_for(g.num_nodes, 4096, [&](std::uint64_t b, std::uint64_t e) {
    for (std::uint64_t v = b; v < e; ++v)
      std::sort(g.col_idx.begin() + static_cast<std::ptrdiff_t>(g.row_ptr[v]),
                g.col_idx.begin() + static_cast<std::ptrdiff_t>(g.row_ptr[v + 1]));
  });
}

void exclusive_scan_inplace(std::vector<std::uint64_t>& a) {
  std::uint64_t run = 0;
  for (auto& x : a) {
    const std::uint64_t d = x;
    x = run;
    run += d;
  }
}

}  // namespace

CsrGraph from_edges(std::uint64_t num_nodes,
                    std::span<const std::pair<NodeId, NodeId>> edges) {
  // Range check first so the error names the offending id like the
  // reference does (R:proj/src/graph.cpp:57-62) — first bad edge in order.
  for (const auto& [s, d] : edges)
    if (s >= num_nodes || d >= num_nodes)
      throw InputError("from_edges: node id " + std::to_string(std::max(s, d)) +
                       " out of range (num_nodes=" + std::to_string(num_nodes) +
                       ")");

  CsrGraph g;
  g.num_nodes = num_nodes;
  // Counting sort by source with atomic cursors; rows are sorted afterwards,
  // so scatter order inside a row is irrelevant to the result.
  std::vector<std::uint64_t> cnt(num_nodes + 1, 0);
  {
    auto* c = cnt.data();
    parallel_for(edges.size(), 1 << 18, [&](std::uint64_t b, std::uint64_t e) {
      for (std::uint64_t i = b; i < e; ++i)
        std::atomic_ref<std::uint64_t>(c[edges[i].first]).fetch_add(
            1, std::memory_order_relaxed);
    });
  }
  exclusive_scan_inplace(cnt);  // cnt[v] = first slot of row v, cnt[N] = E
  g.row_ptr = cnt;
  g.col_idx.resize(edges.size());
  {
    auto* cur = cnt.data();
    auto* out = g.col_idx.data();
    parallel_for(edges.size(), 1 << 18, [&](std::uint64_t b, std::uint64_t e) {
      for (std::uint64_t i = b; i < e; ++i) {
        const std::uint64_t slot =
            std::atomic_ref<std::uint64_t>(cur[edges[i].first])
                .fetch_add(1, std::memory_order_relaxed);
        out[slot] = edges[i].second;
      }
    });
  }
  sort_rows(g);
  return g;
}

namespace {

bool skip_line(const char* b, const char* e) {
  for (; b != e; ++b) {
    if (*b == ' ' || *b == '\t' || *b == '\r') continue;
    return *b == '#' || *b == '%';
  }
  return true;
}

bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' ||
         c == '\f';
}

}  // namespace

CsrGraph load_edge_list(std::istream& in) {
  const std::string text((std::istreambuf_iterator<char>(in)),
                         std::istreambuf_iterator<char>());
  std::vector<std::pair<NodeId, NodeId>> edges;
  NodeId max_id = 0;
  std::size_t line_no = 0;
  const char* p = text.data();
  const char* const end = p + text.size();
  while (p < end) {
    const char* eol = static_cast<const char*>(std::memchr(p, '\n', end - p));
    if (!eol) eol = end;
    ++line_no;
    if (!skip_line(p, eol)) {
      NodeId ids[2];
      int n = 0;
      const char* q = p;
      while (true) {
        while (q < eol && is_space(*q)) ++q;
        if (q >= eol) break;
        const char* t0 = q;
        while (q < eol && !is_space(*q)) ++q;
        if (n == 2)
          throw ParseError("edge list: expected 'src dst', found extra token",
                           line_no);
        NodeId v = 0;
        bool ok = (q > t0);
        for (const char* c = t0; c < q && ok; ++c) {
          if (*c < '0' || *c > '9') {
            ok = false;
            break;
          }
          const NodeId digit = static_cast<NodeId>(*c - '0');
          if (v > (~0ull - digit) / 10) ok = false;  // u64 overflow
          v = v * 10 + digit;
        }
        if (!ok)
          throw ParseError("edge list: expected integer node id, got '" +
                               std::string(t0, q) + "'",
                           line_no);
        ids[n++] = v;
      }
      if (n != 2) throw ParseError("edge list: expected 'src dst'", line_no);
      max_id = std::max({max_id, ids[0], ids[1]});
      edges.emplace_back(ids[0], ids[1]);
    }
    p = eol + 1;
  }
  if (edges.empty())
    throw ParseError("edge list: no edges found, node count unknown", 0);
  return from_edges(max_id + 1, edges);
}

CsrGraph gen_synthetic(SyntheticKind kind, std::uint64_t num_nodes,
                       double avg_degree, std::uint64_t seed) {
  if (num_nodes < 1) throw InputError("gen_synthetic: num_nodes must be >= 1");
  if (avg_degree < 0) throw InputError("gen_synthetic: avg_degree must be >= 0");

  // The reference draws, node after node, one degree and then that many
  // uniform neighbors from a single stream (R:proj/src/graph.cpp:148-174).
  // Edges therefore arrive grouped by ascending source, so the CSR is the
  // draw order itself plus a per-row sort — no edge list, no counting sort.
  Rng rng(seed);
  CsrGraph g;
  g.num_nodes = num_nodes;
  g.row_ptr.resize(num_nodes + 1);
  g.row_ptr[0] = 0;
  g.col_idx.reserve(static_cast<std::size_t>(avg_degree * num_nodes) + num_nodes);

  const std::uint64_t whole = static_cast<std::uint64_t>(avg_degree);
  const double frac = avg_degree - static_cast<double>(whole);
  // powerlaw constants, same expressions as the reference so the doubles
  // round identically (R:proj/src/graph.cpp:161-168).
  const double alpha = 1.6;
  const double x_min = std::max(0.5, avg_degree * (alpha - 1.0) / alpha);
  const double neg_inv_alpha = -1.0 / alpha;
  const double cap = num_nodes == 1 ? 1.0 : static_cast<double>(num_nodes - 1);
  const double hi = std::max(cap, 1.0);

  for (std::uint64_t v = 0; v < num_nodes; ++v) {
    std::uint64_t deg;
    if (kind == SyntheticKind::uniform) {
      deg = whole + (rng.next_unit() < frac ? 1 : 0);
    } else {
      const double u = rng.next_unit();
      const double x = x_min * std::pow(1.0 - u, neg_inv_alpha);
      deg = static_cast<std::uint64_t>(std::clamp(std::floor(x), 1.0, hi));
    }
    for (std::uint64_t k = 0; k < deg; ++k)
      g.col_idx.push_back(rng.next_below(num_nodes));
    g.row_ptr[v + 1] = g.col_idx.size();
  }
  sort_rows(g);
  return g;
}

CsrGraph gen_rmat(std::uint64_t num_nodes, std::uint64_t num_edges,
                  std::uint64_t seed, RmatParams p) {
  if (num_nodes < 1) throw InputError("gen_rmat: num_nodes must be >= 1");
  if (p.a < 0 || p.b < 0 || p.c < 0 || p.a + p.b + p.c > 1.0)
    throw InputError("gen_rmat: quadrant probabilities must be in [0,1]");
  const unsigned scale =
      num_nodes <= 1 ? 0u : static_cast<unsigned>(std::bit_width(num_nodes - 1));
  const double ab = p.a + p.b, abc = p.a + p.b + p.c;
  constexpr std::uint64_t kBlock = 1u << 16;
  const std::uint64_t blocks = (num_edges + kBlock - 1) / kBlock;
  std::vector<std::pair<NodeId, NodeId>> edges(num_edges);
  parallel_for(blocks, 1, [&](std::uint64_t b0, std::uint64_t b1) {
    for (std::uint64_t blk = b0; blk < b1; ++blk) {
      Rng rng(seed ^ (0xD1B54A32D192ED03ull * (blk + 1)));
      const std::uint64_t lo = blk * kBlock;
      const std::uint64_t hi = std::min(num_edges, lo + kBlock);
      for (std::uint64_t i = lo; i < hi; ++i) {
        std::uint64_t s, d;
        do {
          s = d = 0;
          for (unsigned l = 0; l < scale; ++l) {
            const double r = rng.next_unit();
            const unsigned q = r < p.a ? 0u : r < ab ? 1u : r < abc ? 2u : 3u;
            s = (s << 1) | (q >> 1);
            d = (d << 1) | (q & 1u);
          }
        } while (s >= num_nodes || d >= num_nodes);
        edges[i] = {s, d};
      }
    }
  });
  return from_edges(num_nodes, edges);
}

DegreeStats degree_stats(const CsrGraph& g) {
  DegreeStats s;
  if (g.num_nodes == 0) return s;
  s.min_degree = g.degree(0);
  for (std::uint64_t v = 0; v < g.num_nodes; ++v) {
    s.min_degree = std::min(s.min_degree, g.degree(v));
    s.max_degree = std::max(s.max_degree, g.degree(v));
  }
  s.mean_degree =
      static_cast<double>(g.num_edges()) / static_cast<double>(g.num_nodes);
  s.histogram.assign(s.max_degree + 1, 0);
  for (std::uint64_t v = 0; v < g.num_nodes; ++v) ++s.histogram[g.degree(v)];
  return s;
}

namespace {

static_assert(std::endian::native == std::endian::little,
              "binary CSR dump assumes a little-endian host");

void write_u64s(std::ostream& out, const std::uint64_t* p, std::size_t n) {
  out.write(reinterpret_cast<const char*>(p),
            static_cast<std::streamsize>(n * sizeof(std::uint64_t)));
}

void read_u64s(std::istream& in, std::uint64_t* p, std::size_t n) {
  const auto want = static_cast<std::streamsize>(n * sizeof(std::uint64_t));
  in.read(reinterpret_cast<char*>(p), want);
  if (in.gcount() != want) throw ParseError("csr dump: truncated stream", 0);
}

}  // namespace

void save_csr(const CsrGraph& g, std::ostream& out) {
  const std::uint64_t hdr[2] = {g.num_nodes, g.num_edges()};
  write_u64s(out, hdr, 2);
  write_u64s(out, g.row_ptr.data(), g.row_ptr.size());
  write_u64s(out, g.col_idx.data(), g.col_idx.size());
}

CsrGraph load_csr(std::istream& in) {
  std::uint64_t hdr[2];
  read_u64s(in, hdr, 2);
  CsrGraph g;
  g.num_nodes = hdr[0];
  // Guard absurd headers before allocating (a corrupt dump must fail as a
  // ParseError, not as bad_alloc).
  if (hdr[0] > (1ull << 40) || hdr[1] > (1ull << 42))
    throw ParseError("csr dump: implausible header", 0);
  g.row_ptr.resize(hdr[0] + 1);
  read_u64s(in, g.row_ptr.data(), g.row_ptr.size());
  g.col_idx.resize(hdr[1]);
  read_u64s(in, g.col_idx.data(), g.col_idx.size());
  validate_csr(g);
  return g;
}

}  // namespace mgg
