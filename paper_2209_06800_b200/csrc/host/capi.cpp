// C-ABI layer B (include/mgg.h): host facade over the C++ API. Exceptions
// never cross this boundary; they become status codes + mgg_last_error().
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>

#include "mgg.h"
#include "mgg/costmodel.hpp"
#include "mgg/engine.hpp"
#include "mgg/errors.hpp"
#include "mgg/graph.hpp"
#include "mgg/placement.hpp"
#include "mgg/tuner.hpp"
#include "mgg/workload.hpp"

namespace mgg::dev {
std::string& last_error();  // runtime.cu
}

struct mgg_graph {
  mgg::CsrGraph g;
};
struct mgg_flat_plan {
  mgg::FlatPlan p;
};
struct mgg_engine {
  std::unique_ptr<mgg::Engine> e;
};

namespace {

using namespace mgg;

template <class F>
int guard(F&& f) {
  try {
    f();
    return MGG_OK;
  } catch (const ParseError& e) {
    dev::last_error() = e.what();
    return MGG_E_PARSE;
  } catch (const InputError& e) {
    dev::last_error() = e.what();
    return MGG_E_INPUT;
  } catch (const ConfigError& e) {
    dev::last_error() = e.what();
    return MGG_E_CONFIG;
  } catch (const IntegrityError& e) {
    dev::last_error() = e.what();
    return MGG_E_INTEGRITY;
  } catch (const CudaError& e) {
    dev::last_error() = e.what();
    return MGG_E_CUDA;
  } catch (const std::bad_alloc&) {
    dev::last_error() = "host out of memory";
    return MGG_E_INPUT;
  } catch (const std::exception& e) {
    dev::last_error() = e.what();
    return MGG_E_INPUT;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw InputError(std::string(what) + ": null argument");
}

char* dup(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  if (!out) throw std::bad_alloc();
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

PlacementMode mode_of(int m) {
  return m == 0 ? PlacementMode::equal_nodes : PlacementMode::follow_split;
}

HardwareProfile hw_of(uint32_t num_sms, uint32_t max_warps, uint64_t smem_per_sm) {
  HardwareProfile hw;
  hw.num_sms = num_sms;
  hw.max_warps_per_sm = max_warps;
  hw.smem_per_sm_bytes = smem_per_sm;
  return hw;
}

SimulateFn wrap(mgg_measure_fn fn, void* user) {
  return [fn, user](const KernelConfig& c) -> std::uint64_t {
    int err = 0;
    const std::uint64_t v = fn(c.ps, c.dist, c.wpb, user, &err);
    if (err) throw std::runtime_error("callback reported error " + std::to_string(err));
    return v;
  };
}

}  // namespace

extern "C" {

const char* mgg_version(void) { return "mgg-b200 0.1 (sm_100a)"; }

void mgg_free(void* p) { std::free(p); }

int mgg_graph_from_csr(uint64_t n, uint64_t m, const uint64_t* row_ptr,
                       const uint64_t* col, mgg_graph** out) {
  return guard([&] {
    need(row_ptr, "graph_from_csr");
    need(out, "graph_from_csr");
    auto h = std::make_unique<mgg_graph>();
    h->g.num_nodes = n;
    h->g.row_ptr.assign(row_ptr, row_ptr + n + 1);
    if (m) {
      need(col, "graph_from_csr");
      h->g.col_idx.assign(col, col + m);
    }
    validate_csr(h->g);
    *out = h.release();
  });
}

int mgg_graph_from_edges(uint64_t n, uint64_t m, const uint64_t* src,
                         const uint64_t* dst, mgg_graph** out) {
  return guard([&] {
    need(out, "graph_from_edges");
    std::vector<std::pair<NodeId, NodeId>> e(m);
    for (uint64_t i = 0; i < m; ++i) e[i] = {src[i], dst[i]};
    auto h = std::make_unique<mgg_graph>();
    h->g = from_edges(n, e);
    *out = h.release();
  });
}

int mgg_graph_generate(int kind, uint64_t n, double avg, uint64_t seed, mgg_graph** out) {
  return guard([&] {
    need(out, "graph_generate");
    auto h = std::make_unique<mgg_graph>();
    if (kind == 0 || kind == 1)
      h->g = gen_synthetic(kind == 0 ? SyntheticKind::uniform : SyntheticKind::powerlaw,
                           n, avg, seed);
    else if (kind == 2)
      h->g = gen_rmat(n, static_cast<std::uint64_t>(avg), seed);
    else
      throw InputError("graph_generate: unknown kind");
    *out = h.release();
  });
}

int mgg_graph_load_edge_list(const char* path, mgg_graph** out) {
  return guard([&] {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw InputError(std::string("cannot open '") + path + "'");
    auto h = std::make_unique<mgg_graph>();
    h->g = load_edge_list(in);
    *out = h.release();
  });
}

int mgg_graph_load_csr(const char* path, mgg_graph** out) {
  return guard([&] {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw InputError(std::string("cannot open '") + path + "'");
    auto h = std::make_unique<mgg_graph>();
    h->g = load_csr(in);
    *out = h.release();
  });
}

int mgg_graph_save_csr(const mgg_graph* g, const char* path) {
  return guard([&] {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw InputError(std::string("cannot open '") + path + "'");
    save_csr(g->g, out);
  });
}

int mgg_graph_dims(const mgg_graph* g, uint64_t* n, uint64_t* m) {
  if (!g) return MGG_E_INPUT;
  if (n) *n = g->g.num_nodes;
  if (m) *m = g->g.num_edges();
  return MGG_OK;
}

const uint64_t* mgg_graph_row_ptr(const mgg_graph* g) { return g->g.row_ptr.data(); }
const uint64_t* mgg_graph_col_idx(const mgg_graph* g) { return g->g.col_idx.data(); }

int mgg_graph_destroy(mgg_graph* g) {
  delete g;
  return MGG_OK;
}

int mgg_split_by_edges(const mgg_graph* g, uint32_t num_gpus, uint64_t* pts) {
  return guard([&] {
    const WorkloadSplit s = split_by_edges(g->g, num_gpus);
    std::copy(s.split_points.begin(), s.split_points.end(), pts);
  });
}

int mgg_plan_ne_placement(const mgg_graph* g, uint32_t num_gpus, int mode, uint64_t dim,
                          uint64_t* ranges) {
  return guard([&] {
    const WorkloadSplit s = split_by_edges(g->g, num_gpus);
    const NePlacement p = plan_ne_placement(g->g, num_gpus, mode_of(mode), dim, &s);
    for (uint32_t i = 0; i < num_gpus; ++i) {
      ranges[2 * i] = p.ranges[i].lb;
      ranges[2 * i + 1] = p.ranges[i].ub;
    }
  });
}

int mgg_translate(const mgg_graph* g, uint32_t num_gpus, int mode, uint64_t count,
                  const uint64_t* ids, uint32_t* gpu, uint64_t* off) {
  return guard([&] {
    const WorkloadSplit s = split_by_edges(g->g, num_gpus);
    const NePlacement p = plan_ne_placement(g->g, num_gpus, mode_of(mode), 4, &s);
    for (uint64_t i = 0; i < count; ++i) {
      const Owner o = translate(p, ids[i]);
      gpu[i] = o.gpu;
      off[i] = o.offset;
    }
  });
}

int mgg_memory_footprint(const mgg_graph* g, uint32_t num_gpus, int mode, uint64_t dim,
                         uint64_t device_mem, uint64_t* per_gpu, int* fits) {
  return guard([&] {
    const WorkloadSplit s = split_by_edges(g->g, num_gpus);
    const NePlacement p = plan_ne_placement(g->g, num_gpus, mode_of(mode), dim, &s);
    HardwareProfile hw;
    hw.device_mem_bytes = device_mem;
    const FootprintReport r = memory_footprint(g->g, p, s, hw);
    for (std::size_t i = 0; i < r.per_gpu.size(); ++i) {
      per_gpu[2 * i] = r.per_gpu[i].ne_bytes;
      per_gpu[2 * i + 1] = r.per_gpu[i].gp_bytes;
    }
    *fits = r.fits ? 1 : 0;
  });
}

int mgg_flat_plan_build(const mgg_graph* g, uint32_t num_gpus, int placement_mode,
                        uint32_t gpu, uint32_t ps, uint32_t dist, uint32_t wpb,
                        uint64_t dim, int mapping, int granularity, mgg_flat_plan** out) {
  return guard([&] {
    need(g, "flat_plan_build");
    const WorkloadSplit s = split_by_edges(g->g, num_gpus);
    const NePlacement p = plan_ne_placement(g->g, num_gpus, mode_of(placement_mode), dim, &s);
    auto h = std::make_unique<mgg_flat_plan>();
    h->p = build_flat_plan(g->g, s, p, gpu, KernelConfig{ps, dist, wpb}, dim,
                           mapping == 0 ? MappingMode::interleaved : MappingMode::segregated,
                           granularity == 0 ? Granularity::partitioned
                                            : Granularity::whole_list);
    *out = h.release();
  });
}

int mgg_flat_plan_info(const mgg_flat_plan* h, uint64_t* info) {
  if (!h || !info) return MGG_E_INPUT;
  const FlatPlan& p = h->p;
  info[0] = p.local.num_parts();
  info[1] = p.remote.num_parts();
  info[2] = p.local.cols.size();
  info[3] = p.remote.cols.size();
  info[4] = p.num_warps();
  info[5] = p.num_blocks();
  info[6] = p.first_target;
  info[7] = p.rows;
  info[8] = smem(p.cfg, p.dim);
  info[9] = launch_smem(p.cfg, p.dim);
  return MGG_OK;
}

const int32_t* mgg_flat_plan_meta(const mgg_flat_plan* h, int kind) {
  return kind == 0 ? h->p.local.meta.data() : h->p.remote.meta.data();
}
const uint32_t* mgg_flat_plan_cols(const mgg_flat_plan* h, int kind) {
  return kind == 0 ? h->p.local.cols.data() : h->p.remote.cols.data();
}

int mgg_flat_plan_json(const mgg_flat_plan* h, char** json) {
  return guard([&] { *json = dup(plan_to_json(h->p.expand())); });
}

int mgg_flat_plan_tasks(const mgg_flat_plan* h, uint64_t* warp_off, uint8_t* kind,
                        uint32_t* idx) {
  return guard([&] {
    const KernelLaunchPlan kp = h->p.expand();
    uint64_t k = 0;
    for (std::size_t w = 0; w < kp.warps.size(); ++w) {
      warp_off[w] = k;
      for (const WarpTask& t : kp.warps[w].tasks) {
        kind[k] = t.kind == PartKind::local ? 0 : 1;
        idx[k++] = t.index;
      }
    }
    warp_off[kp.warps.size()] = k;
  });
}

int mgg_flat_plan_destroy(mgg_flat_plan* h) {
  delete h;
  return MGG_OK;
}

uint64_t mgg_wpw(uint32_t ps, uint32_t dist, uint32_t wpb, uint64_t dim) {
  return wpw(KernelConfig{ps, dist, wpb}, dim);
}
uint64_t mgg_smem(uint32_t ps, uint32_t dist, uint32_t wpb, uint64_t dim) {
  return smem(KernelConfig{ps, dist, wpb}, dim);
}

int mgg_launch_geometry(uint64_t nl, uint64_t nr, uint32_t ps, uint32_t dist, uint32_t wpb,
                        const char* profile, uint64_t* wb, double* bps) {
  return guard([&] {
    const LaunchGeometry g =
        launch_geometry(nl, nr, KernelConfig{ps, dist, wpb}, builtin_profile(profile));
    wb[0] = g.num_warps;
    wb[1] = g.num_blocks;
    *bps = g.blocks_per_sm;
  });
}

int mgg_validate(uint32_t ps, uint32_t dist, uint32_t wpb, uint64_t dim, uint32_t num_sms,
                 uint32_t max_warps, uint64_t smem_per_sm, char* buf, size_t buflen) {
  const auto v = validate(KernelConfig{ps, dist, wpb}, hw_of(num_sms, max_warps, smem_per_sm), dim);
  std::string s;
  for (const auto& x : v) s += x.constraint + ";";
  if (buf && buflen) {
    std::strncpy(buf, s.c_str(), buflen - 1);
    buf[buflen - 1] = 0;
  }
  return static_cast<int>(v.size());
}

int mgg_profile_json(const char* name_or_path, char** json) {
  return guard([&] { *json = dup(profile_to_json(resolve_profile(name_or_path))); });
}

int mgg_optimize(mgg_measure_fn fn, void* user, uint32_t num_sms, uint32_t max_warps,
                 uint64_t smem_per_sm, uint64_t dim, int retreat_value_rank,
                 uint64_t max_evals, uint64_t* trace, size_t cap, size_t* n, uint64_t* best) {
  return guard([&] {
    TuneOptions o;
    o.retreat = retreat_value_rank ? RetreatRule::value_rank : RetreatRule::latency_rank;
    o.max_evaluations = max_evals;
    const TuneTrace t = optimize(wrap(fn, user), hw_of(num_sms, max_warps, smem_per_sm), dim, o);
    *n = t.entries.size();
    for (std::size_t i = 0; i < t.entries.size() && i < cap; ++i) {
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

int mgg_exhaustive(mgg_measure_fn fn, void* user, uint32_t num_sms, uint32_t max_warps,
                   uint64_t smem_per_sm, uint64_t dim, uint64_t* table, size_t cap,
                   size_t* n) {
  return guard([&] {
    const ExhaustiveResult r =
        exhaustive(wrap(fn, user), hw_of(num_sms, max_warps, smem_per_sm), dim);
    *n = r.table.size();
    for (std::size_t i = 0; i < r.table.size() && i < cap; ++i) {
      table[4 * i] = r.table[i].cfg.ps;
      table[4 * i + 1] = r.table[i].cfg.dist;
      table[4 * i + 2] = r.table[i].cfg.wpb;
      table[4 * i + 3] = r.table[i].cycles;
    }
  });
}

int mgg_engine_create(const mgg_graph* g, uint32_t num_parts, const int32_t* part_device,
                      uint32_t ps, uint32_t dist, uint32_t wpb, const mgg_model_desc* m,
                      mgg_engine** out) {
  return guard([&] {
    need(g, "engine_create");
    need(m, "engine_create");
    need(part_device, "engine_create");
    ModelSpec spec;
    spec.kind = m->kind == 0 ? ModelSpec::Kind::gcn : ModelSpec::Kind::gin;
    spec.layers = m->layers;
    spec.in_dim = m->in_dim;
    spec.hidden = m->hidden;
    spec.out_dim = m->out_dim;
    spec.eps = m->eps;
    spec.norm = m->norm != 0;
    if (spec.kind == ModelSpec::Kind::gcn) {
      need(m->w1, "engine_create w1");
      const std::size_t n =
          std::size_t(m->in_dim) * m->hidden + std::size_t(m->hidden) * m->out_dim;
      spec.w1.assign(m->w1, m->w1 + n);
    } else {
      std::size_t n1 = 0, nb1 = 0, n2 = 0, nb2 = 0;
      std::uint32_t d = m->in_dim;
      for (std::uint32_t l = 0; l < m->layers; ++l) {
        const std::uint32_t b = l + 1 == m->layers ? m->out_dim : m->hidden;
        n1 += std::size_t(d) * m->hidden;
        nb1 += m->hidden;
        n2 += std::size_t(m->hidden) * b;
        nb2 += b;
        d = b;
      }
      need(m->w1, "engine_create w1");
      need(m->b1, "engine_create b1");
      need(m->w2, "engine_create w2");
      need(m->b2, "engine_create b2");
      spec.w1.assign(m->w1, m->w1 + n1);
      spec.b1.assign(m->b1, m->b1 + nb1);
      spec.w2.assign(m->w2, m->w2 + n2);
      spec.b2.assign(m->b2, m->b2 + nb2);
    }
    auto h = std::make_unique<mgg_engine>();
    h->e = std::make_unique<Engine>(g->g, num_parts,
                                    std::vector<int32_t>(part_device, part_device + num_parts),
                                    KernelConfig{ps, dist, wpb}, std::move(spec));
    *out = h.release();
  });
}

int mgg_engine_destroy(mgg_engine* e) {
  delete e;
  return MGG_OK;
}

int mgg_engine_ipc_export(const mgg_engine* e, uint32_t part, void* blob, size_t* len) {
  return guard([&] {
    const auto b = e->e->export_ipc(part);
    if (blob) {
      if (*len < b.size()) throw InputError("engine_ipc_export: buffer too small");
      std::memcpy(blob, b.data(), b.size());
    }
    *len = b.size();
  });
}

int mgg_engine_ipc_import(mgg_engine* e, uint32_t part, const void* blob, size_t len) {
  return guard([&] {
    const auto* p = static_cast<const std::uint8_t*>(blob);
    e->e->import_ipc(part, std::vector<std::uint8_t>(p, p + len));
  });
}

int mgg_engine_vmm_ipc(const mgg_engine* e, int* on) {
  return guard([&] { *on = e->e->vmm_ipc() ? 1 : 0; });
}

int mgg_engine_vmm_export(const mgg_engine* e, uint32_t part, int* fds, size_t* count) {
  return guard([&] {
    const auto v = e->e->export_vmm(part);
    if (fds) {
      if (*count < v.size()) throw InputError("engine_vmm_export: buffer too small");
      std::memcpy(fds, v.data(), v.size() * sizeof(int));
    }
    *count = v.size();
  });
}

int mgg_engine_vmm_import(mgg_engine* e, uint32_t part, const int* fds, size_t count) {
  return guard([&] { e->e->import_vmm(part, std::vector<int>(fds, fds + count)); });
}

int mgg_engine_set_config(mgg_engine* e, uint32_t ps, uint32_t dist, uint32_t wpb) {
  return guard([&] { e->e->set_config(KernelConfig{ps, dist, wpb}); });
}
int mgg_engine_set_remote_fetch(mgg_engine* e, int mode) {
  return guard([&] {
    e->e->set_remote_fetch(mode == 1   ? Engine::RemoteFetch::fine
                           : mode == 2 ? Engine::RemoteFetch::halo
                                       : Engine::RemoteFetch::automatic);
  });
}

int mgg_engine_set_mapping(mgg_engine* e, int mapping, int granularity) {
  return guard([&] {
    e->e->set_mapping(mapping == 0 ? MappingMode::interleaved : MappingMode::segregated,
                      granularity == 0 ? Granularity::partitioned : Granularity::whole_list);
  });
}

uint64_t mgg_remote_partition_bytes(uint64_t part_size, uint64_t dim, int paged,
                                    uint64_t page_bytes) {
  return remote_partition_bytes(part_size, dim, paged ? Transport::paged : Transport::fine_grained,
                                page_bytes);
}

int mgg_engine_set_input(mgg_engine* e, const float* x) {
  return guard([&] { e->e->set_input(x); });
}
int mgg_engine_forward(mgg_engine* e) {
  return guard([&] { e->e->forward(); });
}
int mgg_engine_get_output(mgg_engine* e, float* z) {
  return guard([&] { e->e->get_output(z); });
}
int mgg_engine_forward_host(mgg_engine* e, const float* x, float* z) {
  return guard([&] { e->e->forward_host(x, z); });
}
int mgg_engine_set_k1_form(mgg_engine* e, uint32_t form) {
  return guard([&] { e->e->set_k1_form(form); });
}
int mgg_engine_set_graphs(mgg_engine* e, int on) {
  return guard([&] { e->e->set_graphs(on != 0); });
}
int mgg_engine_submit_host(mgg_engine* e, const float* x, float* z, uint64_t* ticket) {
  return guard([&] {
    if (!ticket) throw mgg::InputError("submit_host: null ticket");
    *ticket = e->e->submit_host(x, z);
  });
}
int mgg_engine_wait(mgg_engine* e, uint64_t ticket) {
  return guard([&] { e->e->wait(ticket); });
}
int mgg_engine_get_hidden(mgg_engine* e, uint32_t which, float* rows, uint32_t* width) {
  return guard([&] {
    const std::uint32_t w = e->e->get_hidden(which, rows);
    if (width) *width = w;
  });
}
int mgg_engine_aggregate_host(mgg_engine* e, const float* x, uint32_t dim, float self_scale,
                              int relu_in, float* out) {
  return guard([&] { e->e->aggregate_host(x, dim, self_scale, relu_in != 0, out); });
}
int mgg_engine_aggregate_phase_host(mgg_engine* e, const float* x, uint32_t dim,
                                    float self_scale, int relu_in, int phase, float* out) {
  return guard([&] { e->e->aggregate_host(x, dim, self_scale, relu_in != 0, out, phase); });
}
int mgg_engine_time_aggregate(mgg_engine* e, uint32_t dim, uint32_t reps, int phase,
                              uint64_t* ns) {
  return guard([&] { *ns = e->e->time_aggregate(dim, reps, phase); });
}
int mgg_engine_time_aggregate_each(mgg_engine* e, uint32_t dim, uint32_t reps, int phase,
                                   uint64_t* ns) {
  return guard([&] {
    if (!ns) throw mgg::InputError("time_aggregate_each: null output");
    const auto v = e->e->time_aggregate_each(dim, reps, phase);
    std::memcpy(ns, v.data(), v.size() * sizeof(uint64_t));
  });
}
int mgg_engine_measure_multi_gpu(mgg_engine* e, uint32_t dim, uint32_t reps,
                                 uint64_t* summary, uint64_t* per_part, double* per_part_f) {
  return guard([&] {
    if (!summary || !per_part || !per_part_f)
      throw mgg::InputError("measure_multi_gpu: null output");
    const auto r = e->e->measure_multi_gpu(dim, reps);
    summary[0] = r.max_gpu_ns;
    summary[1] = r.barrier_ns;
    summary[2] = r.total_ns;
    summary[3] = r.remote_bytes;
    summary[4] = r.max_alone_ns;
    summary[5] = r.devices;
    const uint32_t n = e->e->num_parts();
    std::memset(per_part, 0, sizeof(uint64_t) * 9 * n);
    std::memset(per_part_f, 0, sizeof(double) * 2 * n);
    for (const auto& p : r.per_gpu) {
      uint64_t* q = per_part + 9 * p.part;
      q[0] = 1;
      q[1] = p.total_ns;
      q[2] = p.alone_ns;
      q[3] = p.remote_bytes;
      q[4] = p.local_bytes;
      q[5] = p.num_warps;
      q[6] = p.num_blocks;
      q[7] = p.active_sms;
      q[8] = p.part;
      per_part_f[2 * p.part] = p.achieved_occupancy;
      per_part_f[2 * p.part + 1] = p.sm_utilization;
    }
  });
}
int mgg_engine_get_logits(mgg_engine* e, float* rows) {
  return guard([&] {
    if (!rows) throw mgg::InputError("get_logits: null output");
    e->e->get_logits(rows);
  });
}
int mgg_engine_set_shard_memory(mgg_engine* e, uint32_t part, int kind) {
  return guard([&] { e->e->set_shard_memory(part, kind); });
}
int mgg_engine_trace_csv(mgg_engine* e, uint32_t dim, uint64_t capacity, uint32_t warp_limit,
                         char** csv) {
  return guard([&] {
    if (!csv) throw mgg::InputError("trace_csv: null output");
    *csv = dup(e->e->trace_csv(dim, capacity, warp_limit));
  });
}
int mgg_engine_stats(const mgg_engine* e, uint64_t* s) {
  return guard([&] {
    const auto st = e->e->stats();
    const uint64_t v[10] = {st.local_parts, st.remote_parts, st.local_edges, st.remote_edges,
                            st.warps,       st.blocks,       st.launches,    st.plan_build_ns,
                            st.halo_rows,   st.halo_parts};
    std::memcpy(s, v, sizeof(v));
  });
}
mgg_ctx* mgg_engine_ctx(mgg_engine* e) { return e ? e->e->ctx() : nullptr; }

int mgg_engine_k1_kernels(const mgg_engine* e, uint32_t part, char* buf, size_t cap) {
  return guard([&] {
    if (!e || !buf || cap == 0) throw InputError("engine_k1_kernels: null argument");
    const std::string s = e->e->k1_kernels(part);
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  });
}

int mgg_engine_set_profiling(mgg_engine* e, int on) {
  return guard([&] { e->e->set_profiling(on != 0); });
}

int mgg_engine_profile(mgg_engine* e, double* op_ms, uint32_t* op_kind, uint32_t* op_width,
                       size_t cap, size_t* n_ops, uint64_t* forwards) {
  return guard([&] {
    const auto prof = e->e->profile(forwards);
    *n_ops = prof.size();
    for (std::size_t i = 0; i < prof.size() && i < cap; ++i) {
      op_ms[i] = prof[i].ms;
      op_kind[i] = prof[i].kind;
      op_width[i] = prof[i].width;
    }
  });
}

}  // extern "C"
