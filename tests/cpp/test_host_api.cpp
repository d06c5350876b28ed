// The host C++ API used the way the reference's own unit tests use theirs
// (R:proj/tests/test_graph.cpp, test_placement.cpp, test_workload.cpp,
// test_costmodel.cpp, test_tuner.cpp): same calls, same expectations, against
// namespace mgg. Built and run by tests/test_cpp_api.py (no GPU needed).
#include <cmath>
#include <cstdio>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "mgg/costmodel.hpp"
#include "mgg/errors.hpp"
#include "mgg/graph.hpp"
#include "mgg/placement.hpp"
#include "mgg/rng.hpp"
#include "mgg/tuner.hpp"
#include "mgg/workload.hpp"

using namespace mgg;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                          \
  do {                                                                    \
    ++g_checks;                                                           \
    if (!(c)) {                                                           \
      ++g_fail;                                                           \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
    }                                                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, T)       \
  do {                                 \
    bool ok = false;                   \
    try {                              \
      (void)(expr);                    \
    } catch (const T&) {               \
      ok = true;                       \
    } catch (...) {                    \
    }                                  \
    CHECK(ok && "throws " #T);         \
  } while (0)

static CsrGraph degrees(const std::vector<uint64_t>& d) {
  std::vector<std::pair<NodeId, NodeId>> e;
  for (NodeId v = 0; v < d.size(); ++v)
    for (uint64_t k = 0; k < d[v]; ++k) e.emplace_back(v, 0);
  return from_edges(d.size(), e);
}

static CsrGraph rows(const std::vector<std::vector<NodeId>>& r, uint64_t n) {
  std::vector<std::pair<NodeId, NodeId>> e;
  for (NodeId v = 0; v < r.size(); ++v)
    for (NodeId u : r[v]) e.emplace_back(v, u);
  return from_edges(n, e);
}

static void graph_tests() {
  CsrGraph g = from_edges(3, std::vector<std::pair<NodeId, NodeId>>{{0, 1}, {0, 2}, {1, 2}});
  CHECK((g.row_ptr == std::vector<EdgeOffset>{0, 2, 3, 3}));
  CHECK((g.col_idx == std::vector<NodeId>{1, 2, 2}));
  CHECK_THROWS_AS(from_edges(3, std::vector<std::pair<NodeId, NodeId>>{{0, 5}}), InputError);
  std::istringstream in("# c\n2 0\n");
  CHECK(load_edge_list(in).num_nodes == 3);
  std::istringstream bad("0 1\n1 x\n");
  try {
    load_edge_list(bad);
    CHECK(false);
  } catch (const ParseError& e) {
    CHECK(e.line() == 2);
  }
  CsrGraph a = gen_synthetic(SyntheticKind::uniform, 100, 8, 42);
  CHECK(a.num_edges() == 800);
  CsrGraph p = gen_synthetic(SyntheticKind::powerlaw, 1000, 10, 7);
  DegreeStats s = degree_stats(p);
  CHECK(s.max_degree > 3 * s.mean_degree && s.min_degree >= 1);
  std::stringstream buf(std::ios::in | std::ios::out | std::ios::binary);
  save_csr(p, buf);
  CsrGraph q = load_csr(buf);
  CHECK(q.row_ptr == p.row_ptr && q.col_idx == p.col_idx);
}

static void placement_tests() {
  CHECK((split_by_edges(degrees({2, 2, 2, 2}), 2).split_points == std::vector<NodeId>{2}));
  WorkloadSplit s = split_by_edges(degrees({5, 1, 1, 1}), 2);
  CHECK((s.split_points == std::vector<NodeId>{1}));
  CHECK(s.chunk_edges(degrees({5, 1, 1, 1}), 0) == 5);
  CHECK_THROWS_AS(split_by_edges(degrees({1}), 0), InputError);
  CsrGraph g10 = from_edges(10, {});
  NePlacement p = plan_ne_placement(g10, 4, PlacementMode::equal_nodes, 8);
  CHECK((p.ranges == std::vector<NodeRange>{{0, 3}, {3, 6}, {6, 9}, {9, 10}}));
  CsrGraph g6 = from_edges(6, {});
  NePlacement p6 = plan_ne_placement(g6, 2, PlacementMode::equal_nodes, 4);
  CHECK((translate(p6, 4) == Owner{1, 1}));
  CHECK_THROWS_AS(translate(p6, 6), InputError);
  CHECK_THROWS_AS(plan_ne_placement(g6, 2, PlacementMode::follow_split, 4), InputError);
  WorkloadSplit s2 = split_from_json(split_to_json(split_by_edges(degrees({3, 1, 4, 1, 5}), 3)));
  CHECK(s2.split_points.size() == 2);
}

static void workload_tests() {
  CsrGraph csr = rows({{1, 2, 3, 4, 5}, {1, 2}}, 6);
  auto parts = partition_neighbors(csr, 0, PartKind::local, 2);
  std::vector<uint64_t> sizes;
  for (auto& x : parts) sizes.push_back(x.size());
  CHECK((sizes == std::vector<uint64_t>{2, 2, 1, 2}));
  CHECK_THROWS_AS(partition_neighbors(csr, 0, PartKind::local, 33), ConfigError);
  std::vector<NeighborPartition> l(4), r(4);
  for (auto& x : l) x.neighbors = {0};
  for (auto& x : r) x = {0, PartKind::remote, {0}};
  auto w = interleave(l, r, 2);
  CHECK(w.size() == 2 && w[0].tasks.size() == 4);
  CHECK((w[1].tasks[2] == WarpTask{PartKind::remote, 2}));
  CHECK_THROWS_AS(interleave(l, {}, 17), ConfigError);
  auto five = std::vector<NeighborPartition>(5, NeighborPartition{0, PartKind::local, {0}});
  KernelLaunchPlan plan = map_to_blocks(five, {}, interleave(five, {}, 1), {16, 1, 2}, 16);
  CHECK(plan.blocks.size() == 3 && plan.blocks[2].warp_count == 1);
  CHECK(plan.smem_bytes_per_block == 384);
  // the device form expands to the same plan build_launch_plan makes
  CsrGraph g = gen_synthetic(SyntheticKind::powerlaw, 500, 6, 1);
  WorkloadSplit sp = split_by_edges(g, 3);
  NePlacement ne = plan_ne_placement(g, 3, PlacementMode::follow_split, 8, &sp);
  for (uint32_t gpu = 0; gpu < 3; ++gpu) {
    KernelLaunchPlan ref = build_launch_plan(split_local_remote(g, sp, ne, gpu), {4, 3, 2}, 8);
    FlatPlan fp = build_flat_plan(g, sp, ne, gpu, {4, 3, 2}, 8);
    CHECK(plan_to_json(fp.expand()) == plan_to_json(ref));
    validate_plan(ref);
    KernelLaunchPlan back = plan_from_json(plan_to_json(ref));
    CHECK(back.warps.size() == ref.warps.size());
  }
  // halo plan: distinct remote rows, (owner, offset)-sorted, columns map back
  for (uint32_t gpu = 0; gpu < 3; ++gpu) {
    FlatPlan fp = build_flat_plan(g, sp, ne, gpu, {4, 3, 2}, 8);
    HaloPlan h = build_halo_plan(fp);
    CHECK(h.cols.size() == fp.remote.cols.size());
    for (size_t i = 1; i < h.rows.size(); ++i) CHECK(h.rows[i - 1] < h.rows[i]);
    bool back = true;
    for (size_t i = 0; i < h.cols.size(); ++i) back &= h.rows[h.cols[i]] == fp.remote.cols[i];
    CHECK(back);
    CHECK(h.rows.empty() || h.dedup_ratio() >= 1.0);
  }
  KernelLaunchPlan broken = plan;
  broken.warps[1].tasks[0].index = 0;
  CHECK_THROWS_AS(validate_plan(broken), IntegrityError);
}

static void costmodel_tuner_tests() {
  CHECK(wpw({16, 2, 1}, 602) == 38528);
  CHECK(smem({32, 1, 16}, 602) == 79104);
  HardwareProfile a100 = builtin_profile("a100");
  CHECK(launch_geometry(4, 4, {1, 2, 1}, a100).num_warps == 2);
  CHECK(validate({33, 1, 1}, a100, 16).size() == 1);
  CHECK_THROWS_AS(builtin_profile("h100"), ConfigError);
  HardwareProfile b200 = builtin_profile("b200");
  CHECK(b200.num_sms == 148 && b200.smem_per_sm_bytes == 228 * 1024);
  CHECK(profile_from_json(profile_to_json(b200)).lat.remote_get_base == b200.lat.remote_get_base);
  auto convex = [](const KernelConfig& c) -> uint64_t {
    const double d = 30.0 * std::pow(std::log2(double(c.ps)) - 2.0, 2) +
                     20.0 * std::pow(std::log2(double(c.dist)) - 1.0, 2) +
                     10.0 * std::pow(std::log2(double(c.wpb)) - 1.0, 2);
    return 1000 + static_cast<uint64_t>(std::lround(d));
  };
  TuneTrace t = optimize(convex, a100, 16);
  CHECK((t.best == KernelConfig{4, 2, 2}) && t.best_cycles == 1000 && t.iterations() <= 15);
  ExhaustiveResult full = exhaustive(convex, a100, 16);
  CHECK(full.best_cycles <= t.best_cycles);
  CHECK(trace_to_csv(t).rfind("ps,dist,wpb,cycles,rank\n", 0) == 0);
  try {
    optimize([](const KernelConfig& c) -> uint64_t {
      if (c.ps == 2) throw std::runtime_error("boom");
      return 100;
    }, a100, 16);
    CHECK(false);
  } catch (const std::runtime_error& e) {
    CHECK(std::string(e.what()).find("ps=2") != std::string::npos);
  }
}

int main() {
  graph_tests();
  placement_tests();
  workload_tests();
  costmodel_tuner_tests();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
