// TEST INFRASTRUCTURE ONLY — part of the parity oracle, never shipped.
//
// C shim over the UNMODIFIED reference library (pipeshard, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It flattens
// the reference's value types into plain arrays so pytest (ctypes) can compare
// them bit-for-bit with the product's metadata builder. Only tests/, the
// smoke() checker and bench.py's cpu_baseline / --impl reference leg load it.
//
// Every entry point forwards to exactly one reference function:
//   ref_graph_gen        -> gen_synthetic          (R:proj/src/graph.cpp:139)
//   ref_graph_from_edges -> from_edges             (R:proj/src/graph.cpp:51)
//   ref_graph_from_csr   -> validate_csr           (R:proj/src/graph.cpp:38)
//   ref_split            -> split_by_edges         (R:proj/src/placement.cpp:44)
//   ref_placement        -> plan_ne_placement      (R:proj/src/placement.cpp:73)
//   ref_translate        -> translate              (R:proj/src/placement.cpp:108)
//   ref_footprint        -> memory_footprint       (R:proj/src/placement.cpp:121)
//   ref_lr_split         -> split_local_remote     (R:proj/src/workload.cpp:26)
//   ref_plan_build       -> build_launch_plan      (R:proj/src/workload.cpp:174)
//   ref_wpw/ref_smem/... -> costmodel              (R:proj/src/costmodel.cpp:27-77)
//   ref_optimize         -> optimize               (R:proj/src/tuner.cpp:129)
//   ref_exhaustive       -> exhaustive             (R:proj/src/tuner.cpp:186)
//   ref_multi_gpu_cycles -> multi_gpu_run          (R:proj/src/sim.cpp:597)
//   ref_plan_json        -> to_json(KernelLaunchPlan) (R:proj/src/workload.cpp:276)
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "pipeshard/costmodel.hpp"
#include "pipeshard/errors.hpp"
#include "pipeshard/graph.hpp"
#include "pipeshard/placement.hpp"
#include "pipeshard/sim.hpp"
#include "pipeshard/tuner.hpp"
#include "pipeshard/workload.hpp"

using namespace pipeshard;

namespace {
thread_local std::string g_err;

// 0 ok, 1 input, 2 parse, 3 config, 4 integrity, 9 other
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ParseError& e) {
    g_err = e.what();
    return 2;
  } catch (const InputError& e) {
    g_err = e.what();
    return 1;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 3;
  } catch (const IntegrityError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

struct RefPlan {
  KernelLaunchPlan plan;
  std::string json;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_graph_free(void* g) { delete static_cast<CsrGraph*>(g); }

int ref_graph_gen(int kind, uint64_t n, double avg, uint64_t seed, void** out) {
  return guard([&] {
    *out = new CsrGraph(gen_synthetic(kind == 0 ? SyntheticKind::uniform
                                                : SyntheticKind::powerlaw,
                                      n, avg, seed));
  });
}

int ref_graph_from_edges(uint64_t n, uint64_t m, const uint64_t* src,
                         const uint64_t* dst, void** out) {
  return guard([&] {
    std::vector<std::pair<NodeId, NodeId>> e(m);
    for (uint64_t i = 0; i < m; ++i) e[i] = {src[i], dst[i]};
    *out = new CsrGraph(from_edges(n, e));
  });
}

int ref_graph_from_csr(uint64_t n, uint64_t m, const uint64_t* row_ptr,
                       const uint64_t* col, void** out) {
  return guard([&] {
    auto* g = new CsrGraph();
    g->num_nodes = n;
    g->row_ptr.assign(row_ptr, row_ptr + n + 1);
    g->col_idx.assign(col, col + m);
    try {
      validate_csr(*g);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

void ref_graph_dims(void* gp, uint64_t* n, uint64_t* m) {
  auto* g = static_cast<CsrGraph*>(gp);
  *n = g->num_nodes;
  *m = g->num_edges();
}

void ref_graph_copy(void* gp, uint64_t* row_ptr, uint64_t* col) {
  auto* g = static_cast<CsrGraph*>(gp);
  std::memcpy(row_ptr, g->row_ptr.data(), g->row_ptr.size() * 8);
  std::memcpy(col, g->col_idx.data(), g->col_idx.size() * 8);
}

// split_points: num_gpus-1 entries
int ref_split(void* gp, uint32_t num_gpus, uint64_t* split_points) {
  return guard([&] {
    WorkloadSplit s = split_by_edges(*static_cast<CsrGraph*>(gp), num_gpus);
    for (size_t i = 0; i < s.split_points.size(); ++i)
      split_points[i] = s.split_points[i];
  });
}

// ranges: 2*num_gpus entries (lb, ub) ; mode 0 equal_nodes 1 follow_split
int ref_placement(void* gp, uint32_t num_gpus, int mode, uint64_t dim,
                  uint64_t* ranges) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(gp);
    WorkloadSplit s = split_by_edges(g, num_gpus);
    NePlacement p = plan_ne_placement(
        g, num_gpus, mode == 0 ? PlacementMode::equal_nodes
                               : PlacementMode::follow_split,
        dim, &s);
    for (uint32_t i = 0; i < num_gpus; ++i) {
      ranges[2 * i] = p.ranges[i].lb;
      ranges[2 * i + 1] = p.ranges[i].ub;
    }
  });
}

int ref_translate(void* gp, uint32_t num_gpus, int mode, uint64_t count,
                  const uint64_t* ids, uint32_t* gpu, uint64_t* off) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(gp);
    WorkloadSplit s = split_by_edges(g, num_gpus);
    NePlacement p = plan_ne_placement(
        g, num_gpus, mode == 0 ? PlacementMode::equal_nodes
                               : PlacementMode::follow_split,
        4, &s);
    for (uint64_t i = 0; i < count; ++i) {
      Owner o = translate(p, ids[i]);
      gpu[i] = o.gpu;
      off[i] = o.offset;
    }
  });
}

// per_gpu: 2*num_gpus (ne_bytes, gp_bytes); returns fits in *fits
int ref_footprint(void* gp, uint32_t num_gpus, int mode, uint64_t dim,
                  uint64_t device_mem, uint64_t* per_gpu, int* fits) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(gp);
    WorkloadSplit s = split_by_edges(g, num_gpus);
    NePlacement p = plan_ne_placement(
        g, num_gpus, mode == 0 ? PlacementMode::equal_nodes
                               : PlacementMode::follow_split,
        dim, &s);
    HardwareProfile hw = builtin_profile("a100");
    hw.device_mem_bytes = device_mem;
    FootprintReport r = memory_footprint(g, p, s, hw);
    for (uint32_t i = 0; i < r.per_gpu.size(); ++i) {
      per_gpu[2 * i] = r.per_gpu[i].ne_bytes;
      per_gpu[2 * i + 1] = r.per_gpu[i].gp_bytes;
    }
    *fits = r.fits ? 1 : 0;
  });
}

// Local/remote split for one gpu. Two-phase: sizes then copy.
// sizes: [rows, local_edges, remote_edges, first_target]
int ref_lr_split(void* gp, uint32_t num_gpus, int mode, uint32_t gpu,
                 uint64_t* sizes, uint64_t* l_row, uint64_t* l_col,
                 uint64_t* r_row, uint64_t* r_col) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(gp);
    WorkloadSplit s = split_by_edges(g, num_gpus);
    NePlacement p = plan_ne_placement(
        g, num_gpus, mode == 0 ? PlacementMode::equal_nodes
                               : PlacementMode::follow_split,
        4, &s);
    LocalRemoteSplit lr = split_local_remote(g, s, p, gpu);
    sizes[0] = lr.local_csr.num_nodes;
    sizes[1] = lr.local_csr.num_edges();
    sizes[2] = lr.remote_csr.num_edges();
    sizes[3] = lr.first_target;
    if (l_row) {
      std::memcpy(l_row, lr.local_csr.row_ptr.data(), (sizes[0] + 1) * 8);
      std::memcpy(l_col, lr.local_csr.col_idx.data(), sizes[1] * 8);
      std::memcpy(r_row, lr.remote_csr.row_ptr.data(), (sizes[0] + 1) * 8);
      std::memcpy(r_col, lr.remote_csr.col_idx.data(), sizes[2] * 8);
    }
  });
}

// Builds a reference KernelLaunchPlan for one gpu (multi_gpu_run's recipe,
// R:proj/src/sim.cpp:603-611). mapping 0 interleaved 1 segregated;
// granularity 0 partitioned 1 whole_list.
int ref_plan_build(void* gp, uint32_t num_gpus, int mode, uint32_t gpu,
                   uint32_t ps, uint32_t dist, uint32_t wpb, uint64_t dim,
                   int mapping, int granularity, void** out) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(gp);
    WorkloadSplit s = split_by_edges(g, num_gpus);
    NePlacement p = plan_ne_placement(
        g, num_gpus, mode == 0 ? PlacementMode::equal_nodes
                               : PlacementMode::follow_split,
        dim, &s);
    LocalRemoteSplit lr = split_local_remote(g, s, p, gpu);
    auto* rp = new RefPlan();
    rp->plan = build_launch_plan(
        lr, KernelConfig{ps, dist, wpb}, dim,
        mapping == 0 ? MappingMode::interleaved : MappingMode::segregated,
        granularity == 0 ? Granularity::partitioned : Granularity::whole_list);
    *out = rp;
  });
}

void ref_plan_free(void* p) { delete static_cast<RefPlan*>(p); }

// counts: [n_local_parts, n_remote_parts, local_nbrs, remote_nbrs, n_warps,
//          n_tasks, n_blocks, smem_bytes_per_block]
void ref_plan_counts(void* pp, uint64_t* c) {
  const KernelLaunchPlan& p = static_cast<RefPlan*>(pp)->plan;
  c[0] = p.local_parts.size();
  c[1] = p.remote_parts.size();
  uint64_t ln = 0, rn = 0, tasks = 0;
  for (auto& x : p.local_parts) ln += x.size();
  for (auto& x : p.remote_parts) rn += x.size();
  for (auto& w : p.warps) tasks += w.tasks.size();
  c[2] = ln;
  c[3] = rn;
  c[4] = p.warps.size();
  c[5] = tasks;
  c[6] = p.blocks.size();
  c[7] = p.smem_bytes_per_block;
}

// kind 0 local 1 remote; target[n_parts], size[n_parts], nbrs[total]
void ref_plan_parts(void* pp, int kind, uint64_t* target, uint64_t* size,
                    uint64_t* nbrs) {
  const KernelLaunchPlan& p = static_cast<RefPlan*>(pp)->plan;
  const auto& parts = kind == 0 ? p.local_parts : p.remote_parts;
  uint64_t k = 0;
  for (size_t i = 0; i < parts.size(); ++i) {
    target[i] = parts[i].target;
    size[i] = parts[i].size();
    for (NodeId v : parts[i].neighbors) nbrs[k++] = v;
  }
}

// warp_off[n_warps+1] (task offsets), task_kind[n_tasks], task_idx[n_tasks],
// warp_id[n_warps], block_first[n_blocks], block_count[n_blocks]
void ref_plan_warps(void* pp, uint64_t* warp_off, uint32_t* warp_id,
                    uint8_t* task_kind, uint32_t* task_idx,
                    uint32_t* block_first, uint32_t* block_count) {
  const KernelLaunchPlan& p = static_cast<RefPlan*>(pp)->plan;
  uint64_t k = 0;
  for (size_t w = 0; w < p.warps.size(); ++w) {
    warp_off[w] = k;
    warp_id[w] = p.warps[w].warp_id;
    for (const WarpTask& t : p.warps[w].tasks) {
      task_kind[k] = t.kind == PartKind::local ? 0 : 1;
      task_idx[k] = t.index;
      ++k;
    }
  }
  warp_off[p.warps.size()] = k;
  for (size_t b = 0; b < p.blocks.size(); ++b) {
    block_first[b] = p.blocks[b].first_warp;
    block_count[b] = p.blocks[b].warp_count;
  }
}

// Canonical JSON (R:proj/src/workload.cpp:276-305). Returned pointer valid
// until ref_plan_free.
const char* ref_plan_json(void* pp) {
  auto* rp = static_cast<RefPlan*>(pp);
  nlohmann::json j = rp->plan;
  rp->json = j.dump();
  return rp->json.c_str();
}

uint64_t ref_wpw(uint32_t ps, uint32_t dist, uint32_t wpb, uint64_t dim) {
  return wpw(KernelConfig{ps, dist, wpb}, dim);
}
uint64_t ref_smem(uint32_t ps, uint32_t dist, uint32_t wpb, uint64_t dim) {
  return smem(KernelConfig{ps, dist, wpb}, dim);
}
// geometry: [num_warps, num_blocks]; blocks_per_sm in *bps
int ref_launch_geometry(uint64_t nl, uint64_t nr, uint32_t ps, uint32_t dist,
                        uint32_t wpb, const char* profile, uint64_t* geom,
                        double* bps) {
  return guard([&] {
    LaunchGeometry g = launch_geometry(nl, nr, KernelConfig{ps, dist, wpb},
                                       builtin_profile(profile));
    geom[0] = g.num_warps;
    geom[1] = g.num_blocks;
    *bps = g.blocks_per_sm;
  });
}

// Returns the number of violations; names joined by ';' into buf.
int ref_validate(uint32_t ps, uint32_t dist, uint32_t wpb, uint64_t dim,
                 uint32_t num_sms, uint32_t max_warps, uint64_t smem_per_sm,
                 char* buf, size_t buflen) {
  HardwareProfile hw;
  hw.num_sms = num_sms;
  hw.max_warps_per_sm = max_warps;
  hw.smem_per_sm_bytes = smem_per_sm;
  auto v = validate(KernelConfig{ps, dist, wpb}, hw, dim);
  std::string s;
  for (auto& x : v) s += x.constraint + ";";
  if (buf && buflen) {
    std::strncpy(buf, s.c_str(), buflen - 1);
    buf[buflen - 1] = 0;
  }
  return static_cast<int>(v.size());
}

typedef uint64_t (*ref_measure_fn)(uint32_t ps, uint32_t dist, uint32_t wpb,
                                   void* user);

// trace out: up to cap entries of (ps,dist,wpb,cycles); returns count in *n.
// best in best[4]. retreat 0 latency_rank 1 value_rank.
int ref_optimize(ref_measure_fn fn, void* user, uint32_t num_sms,
                 uint32_t max_warps, uint64_t smem_per_sm, uint64_t dim,
                 int retreat, uint64_t max_evals, uint64_t* trace, size_t cap,
                 size_t* n, uint64_t* best) {
  return guard([&] {
    HardwareProfile hw;
    hw.num_sms = num_sms;
    hw.max_warps_per_sm = max_warps;
    hw.smem_per_sm_bytes = smem_per_sm;
    TuneOptions o;
    o.retreat = retreat == 0 ? RetreatRule::latency_rank
                             : RetreatRule::value_rank;
    o.max_evaluations = max_evals;
    TuneTrace t = optimize(
        [&](const KernelConfig& c) { return fn(c.ps, c.dist, c.wpb, user); },
        hw, dim, o);
    *n = t.entries.size();
    for (size_t i = 0; i < t.entries.size() && i < cap; ++i) {
      trace[4 * i] = t.entries[i].cfg.ps;
      trace[4 * i + 1] = t.entries[i].cfg.dist;
      trace[4 * i + 2] = t.entries[i].cfg.wpb;
      trace[4 * i + 3] = t.entries[i].cycles;
    }
    best[0] = t.best.ps;
    best[1] = t.best.dist;
    best[2] = t.best.wpb;
    best[3] = t.best_cycles;
  });
}

int ref_exhaustive(ref_measure_fn fn, void* user, uint32_t num_sms,
                   uint32_t max_warps, uint64_t smem_per_sm, uint64_t dim,
                   uint64_t* table, size_t cap, size_t* n) {
  return guard([&] {
    HardwareProfile hw;
    hw.num_sms = num_sms;
    hw.max_warps_per_sm = max_warps;
    hw.smem_per_sm_bytes = smem_per_sm;
    ExhaustiveResult r = exhaustive(
        [&](const KernelConfig& c) { return fn(c.ps, c.dist, c.wpb, user); },
        hw, dim);
    *n = r.table.size();
    for (size_t i = 0; i < r.table.size() && i < cap; ++i) {
      table[4 * i] = r.table[i].cfg.ps;
      table[4 * i + 1] = r.table[i].cfg.dist;
      table[4 * i + 2] = r.table[i].cfg.wpb;
      table[4 * i + 3] = r.table[i].cycles;
    }
  });
}

// Modelled cycles of the reference DES for one config (the reference's
// stand-in for the kernel). Used only as a CPU-side comparison.
int ref_multi_gpu_cycles(void* gp, uint32_t num_gpus, uint32_t ps,
                         uint32_t dist, uint32_t wpb, uint64_t dim,
                         const char* profile, uint64_t* cycles) {
  return guard([&] {
    MultiGpuReport r =
        multi_gpu_run(*static_cast<CsrGraph*>(gp), num_gpus,
                      KernelConfig{ps, dist, wpb}, builtin_profile(profile),
                      dim, ScheduleMode{});
    *cycles = r.total_cycles;
  });
}

// Times the reference metadata path for all gpus (split -> place -> per-gpu
// LR split + build_launch_plan), i.e. multi_gpu_run minus the DES.
// Returns seconds.
int ref_time_metadata(void* gp, uint32_t num_gpus, uint32_t ps, uint32_t dist,
                      uint32_t wpb, uint64_t dim, double* seconds,
                      uint64_t* n_parts) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(gp);
    auto t0 = std::chrono::steady_clock::now();
    WorkloadSplit s = split_by_edges(g, num_gpus);
    NePlacement p =
        plan_ne_placement(g, num_gpus, PlacementMode::follow_split, dim, &s);
    uint64_t parts = 0;
    for (uint32_t gpu = 0; gpu < num_gpus; ++gpu) {
      LocalRemoteSplit lr = split_local_remote(g, s, p, gpu);
      KernelLaunchPlan plan =
          build_launch_plan(lr, KernelConfig{ps, dist, wpb}, dim);
      parts += plan.local_parts.size() + plan.remote_parts.size();
    }
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    *n_parts = parts;
  });
}

}  // extern "C"
