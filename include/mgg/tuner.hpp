// Heuristic runtime tuner over (ps, dist, wpb) — R:PAPER.md:471-482 — with
// the reference's exact search semantics (R:proj/include/pipeshard/
// tuner.hpp:28-81, R:proj/src/tuner.cpp:40-243): greedy ascent ps -> dist ->
// wpb from (1,1,1), the ps retreat, the "last three behind the third best"
// stop rule, the 15-evaluation budget and the lookup table. On B200 the
// SimulateFn plug is the measured aggregation-kernel latency
// (Engine::time_aggregate, ns) instead of the reference's DES cycles.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "mgg/costmodel.hpp"

namespace mgg {

using SimulateFn = std::function<std::uint64_t(const KernelConfig&)>;

struct TuneEntry {
  KernelConfig cfg;
  std::uint64_t cycles = 0;
};

struct TuneTrace {
  std::vector<TuneEntry> entries;
  KernelConfig best;
  std::uint64_t best_cycles = 0;
  std::size_t iterations() const { return entries.size(); }
};

enum class RetreatRule : std::uint8_t { latency_rank, value_rank };

struct TuneOptions {
  std::vector<std::uint32_t> ps_steps = {1, 2, 4, 8, 16, 32};
  std::vector<std::uint32_t> dist_steps = {1, 2, 4, 8, 16};
  std::vector<std::uint32_t> wpb_steps = {1, 2, 4, 8, 16};
  std::size_t max_evaluations = 15;
  RetreatRule retreat = RetreatRule::latency_rank;
};

TuneTrace optimize(const SimulateFn& simulate, const HardwareProfile& hw,
                   std::uint64_t dim, const TuneOptions& opts = {});

struct ExhaustiveResult {
  std::vector<TuneEntry> table;  // by cycles, ties by (ps, dist, wpb)
  KernelConfig best;
  std::uint64_t best_cycles = 0;
};

ExhaustiveResult exhaustive(const SimulateFn& simulate, const HardwareProfile& hw,
                            std::uint64_t dim, const TuneOptions& grid = {});

/// "ps,dist,wpb,cycles,rank" rows; rank 1 = lowest latency, ties kept in
/// evaluation order.
std::string trace_to_csv(const TuneTrace& trace);

}  // namespace mgg
