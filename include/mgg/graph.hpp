// Graph ingestion: the input contract of the hot path.
//
// Same value type and semantics as the reference (R:proj/include/pipeshard/
// graph.hpp:25-85): a directed CSR whose row v lists the neighbors whose
// embeddings node v aggregates (R:SPEC.md:105-111); rows sorted ascending,
// duplicates and self-loops kept. The builders here are multi-threaded (the
// reference is single-threaded, 1.5-3.9 s at 62-117M edges) but produce the
// identical CSR for the same input, and gen_synthetic reproduces the
// reference's SplitMix64 streams draw for draw.
#pragma once

#include <cstdint>
#include <iosfwd>
#include <span>
#include <utility>
#include <vector>

namespace mgg {

using NodeId = std::uint64_t;
using EdgeOffset = std::uint64_t;

struct CsrGraph {
  std::uint64_t num_nodes = 0;
  std::vector<EdgeOffset> row_ptr;  // num_nodes + 1
  std::vector<NodeId> col_idx;      // num_edges

  std::uint64_t num_edges() const { return col_idx.size(); }
  std::uint64_t degree(NodeId v) const { return row_ptr[v + 1] - row_ptr[v]; }
  std::span<const NodeId> neighbors(NodeId v) const {
    return {col_idx.data() + row_ptr[v], row_ptr[v + 1] - row_ptr[v]};
  }
  std::uint64_t max_degree() const;
};

struct DegreeStats {
  std::uint64_t min_degree = 0;
  std::uint64_t max_degree = 0;
  double mean_degree = 0.0;
  std::vector<std::uint64_t> histogram;  // histogram[d] = #nodes of degree d
};

/// uniform / powerlaw are the reference generators (R:proj/src/graph.cpp:
/// 139-176); rmat is added for the locality-bearing configs.
enum class SyntheticKind { uniform, powerlaw };

/// Throws InputError when the CSR invariants fail (R:proj/src/graph.cpp:38-49).
void validate_csr(const CsrGraph& g);

/// CSR from an arbitrary edge list; rows grouped by source and sorted, ids >=
/// num_nodes raise InputError (R:proj/src/graph.cpp:51-76).
CsrGraph from_edges(std::uint64_t num_nodes,
                    std::span<const std::pair<NodeId, NodeId>> edges);

/// "src dst" text; '#'/'%' comment lines; ParseError with the 1-based line;
/// empty input is a ParseError (R:proj/src/graph.cpp:99-137).
CsrGraph load_edge_list(std::istream& in);

/// Bit-identical to the reference's gen_synthetic for the same arguments.
CsrGraph gen_synthetic(SyntheticKind kind, std::uint64_t num_nodes,
                       double avg_degree, std::uint64_t seed);

/// R-MAT (Chakrabarti et al. 2004) on 2^ceil(log2 N) ids with quadrant
/// probabilities (a, b, c, 1-a-b-c); endpoints >= N are rejected and redrawn
/// until num_edges edges exist. Ids are NOT shuffled, so low ids form the
/// dense core (locality-bearing graphs). Deterministic per seed: edges are
/// drawn in fixed 1<<16-edge blocks, block k from SplitMix64(seed ^ f(k)).
struct RmatParams {
  double a = 0.57, b = 0.19, c = 0.19;
};
CsrGraph gen_rmat(std::uint64_t num_nodes, std::uint64_t num_edges,
                  std::uint64_t seed, RmatParams p = {});

DegreeStats degree_stats(const CsrGraph& g);

/// Binary dump: LE u64 num_nodes, num_edges, row_ptr[], col_idx[]
/// (R:proj/src/graph.cpp:216-233).
void save_csr(const CsrGraph& g, std::ostream& out);
CsrGraph load_csr(std::istream& in);

}  // namespace mgg
