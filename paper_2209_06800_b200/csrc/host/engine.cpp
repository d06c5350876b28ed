// GCN/GIN multi-GPU forward driver (see include/mgg/engine.hpp). Talks to the
// GPU exclusively through the C-ABI of include/mgg.h.
#include "mgg/engine.hpp"

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstring>

#include "mgg.h"
#include "mgg/errors.hpp"

namespace mgg {

namespace {

// C-ABI status -> the host API's exception taxonomy.
void ok(int st) {
  if (st == MGG_OK) return;
  const std::string msg = mgg_last_error();
  switch (st) {
    case MGG_E_PARSE: throw ParseError(msg, 0);
    case MGG_E_CONFIG: throw ConfigError(msg);
    case MGG_E_INTEGRITY: throw IntegrityError(msg);
    case MGG_E_CUDA: throw CudaError(msg);
    default: throw InputError(msg);
  }
}

}  // namespace

Engine::Engine(const CsrGraph& g, std::uint32_t num_parts,
               std::vector<std::int32_t> part_device, KernelConfig cfg, ModelSpec spec)
    : g_(g), num_parts_(num_parts), dev_(std::move(part_device)), cfg_(cfg),
      spec_(std::move(spec)) {
  if (dev_.size() != num_parts_) throw InputError("engine: part_device size != num_parts");
  if (spec_.in_dim == 0 || spec_.hidden == 0 || spec_.out_dim == 0)
    throw InputError("engine: model widths must be >= 1");
  if (spec_.kind == ModelSpec::Kind::gcn && spec_.layers != 2)
    throw ConfigError("engine: GCN is the 2-layer model of R:PAPER.md:504-508");
  if (spec_.layers < 1) throw ConfigError("engine: layers must be >= 1");
  split_ = split_by_edges(g_, num_parts_);
  ne_ = plan_ne_placement(g_, num_parts_, PlacementMode::follow_split, spec_.in_dim, &split_);
  try {
    ok(mgg_ctx_create(num_parts_, dev_.data(), &ctx_));
    std::vector<std::uint64_t> flag_lb(num_parts_ + 1);
    for (std::uint32_t p = 0; p <= num_parts_; ++p) flag_lb[p] = p;
    // K3 flags: one row per part, slot q = part q's arrival, slot num_parts =
    // the part's own epoch counter
    ok(mgg_store_create(ctx_, flag_lb.data(), kMaxOwners + 1, &flags_));
    build_row_scales();
    build_program();
    fuse_chains();
    find_io_points();
    build_plans();
  } catch (...) {
    free_plans();
    for (auto& v : rs_)
      for (auto* b : v) mgg_dbuf_destroy(b);
    mgg_store_destroy(in_bufs_[1]);
    for (auto* s : stores_) mgg_store_destroy(s);
    for (auto& slot : weights_)
      for (auto* b : slot) mgg_dbuf_destroy(b);
    mgg_store_destroy(flags_);
    mgg_ctx_destroy(ctx_);
    throw;
  }
}

Engine::~Engine() {
  if (ctx_) mgg_ctx_synchronize(ctx_);
  mgg_exec_destroy(exec_);
  exec_ = nullptr;
  free_plans();
  for (auto* s : in_bufs_)  // the one not currently installed as the input
    if (s && s != stores_[input_]) mgg_store_destroy(s);
  for (auto* s : stores_) mgg_store_destroy(s);
  for (auto* s : scratch_) mgg_store_destroy(s);
  for (auto& slot : weights_)
    for (auto* b : slot) mgg_dbuf_destroy(b);
  for (auto& v : rs_)
    for (auto* b : v) mgg_dbuf_destroy(b);
  mgg_store_destroy(flags_);
  mgg_ctx_destroy(ctx_);
}

int Engine::add_store(std::uint32_t dim) {
  std::vector<std::uint64_t> lb(num_parts_ + 1);
  for (std::uint32_t p = 0; p < num_parts_; ++p) lb[p] = ne_.ranges[p].lb;
  lb[num_parts_] = g_.num_nodes;
  mgg_store* s = nullptr;
  ok(mgg_store_create(ctx_, lb.data(), dim, &s));
  stores_.push_back(s);
  return static_cast<int>(stores_.size()) - 1;
}

int Engine::add_weight(const float* src, std::size_t n) {
  std::vector<mgg_dbuf*> per(num_parts_, nullptr);
  weights_.push_back(per);
  for (std::uint32_t p = 0; p < num_parts_; ++p)
    if (dev_[p] >= 0) ok(mgg_dbuf_create(ctx_, p, src, n * sizeof(float), &weights_.back()[p]));
  return static_cast<int>(weights_.size()) - 1;
}

// Self term A = scale * f(H). With a pending ReLU f and a gather table that
// fits the L2 (L1TEX-bound K1), the init also writes G = ReLU(H) once per row
// and the aggregation gathers G (no per-edge ReLU, H itself stays readable
// through get_hidden). An HBM-resident table is instead gathered from H with
// the ReLU applied on load (`relu_load`): K1 is DRAM-bound there, the ReLU
// is free, and the G copy (one write of the table) is not. Returns the store
// to gather.
int Engine::activated(int h, std::uint32_t width, int relu, int a, float scale, int rs,
                      int& relu_load) {
  const std::uint64_t table = g_.num_nodes * ((std::uint64_t(width) + 3) / 4 * 4) * 4;
  relu_load = relu && !rs && table > kL2GatherBytes ? 1 : 0;
  // a row-scaled (normalised GCN) gather table is always a separate copy
  const int g = ((relu && !relu_load) || rs) ? add_store(width) : h;
  Op op{OpKind::init, h, a, g != h ? g : -1, -1, -1, -1, 0, 0, scale, relu};
  op.rs = rs;
  program_.push_back(op);
  return g;
}

void Engine::build_program() {
  const auto& s = spec_;
  input_ = add_store(s.in_dim);
  int cur = input_;          // store holding the layer input
  std::uint32_t cur_w = s.in_dim;
  int fin = 0;               // pending ReLU on `cur`
  const bool gcn = s.kind == ModelSpec::Kind::gcn;
  std::size_t o1 = 0, ob1 = 0, o2 = 0, ob2 = 0;
  auto need = [](const std::vector<float>& v, std::size_t n, const char* what) {
    if (v.size() < n) throw InputError(std::string("engine: weight array too short: ") + what);
  };

  // normalised GCN: Â = D^-1/2 (A+I) D^-1/2 as row scalings around the plain
  // sum — a gather table holds D^-1/2 · (true rows) (its seed too), the sum
  // is then D^1/2 · (true result), i.e. its consumer owes one more D^-1/2.
  // `pend` is that owed power on `cur`.
  const bool norm = gcn && s.norm;
  int pend = 0;
  for (std::uint32_t l = 0; l < s.layers; ++l) {
    const bool last = l + 1 == s.layers;
    if (gcn) {
      // GCN layer l: width a -> b, W_l packed in w1 (R:PAPER.md:504-508)
      const std::uint32_t a = cur_w, b = last ? s.out_dim : s.hidden;
      need(s.w1, o1 + std::size_t(a) * b, "gcn W");
      const int W = add_weight(s.w1.data() + o1, std::size_t(a) * b);
      o1 += std::size_t(a) * b;
      if (b < a) {  // update first: T = f(H)·W, A = T + Σ T_u
        const int T = add_store(b), A = add_store(b);
        Op d{OpKind::dense, cur, T, A, W, -1, -1, std::uint32_t(fin), 0, 1.f, 0};
        d.rs = norm ? pend + 1 : 0;
        program_.push_back(d);
        program_.push_back({OpKind::barrier});
        program_.push_back({OpKind::aggregate, T, A});
        hidden_.push_back(A);
        if (last) {
          const int Z = add_store(b);
          Op sm{OpKind::softmax, A, Z};
          sm.rs = norm ? 1 : 0;
          program_.push_back(sm);
          output_ = Z;
        }
        cur = A;
        pend = norm ? 1 : 0;
      } else {  // aggregate first: A = f(H) + Σ f(H_u), then A·W
        const int A = add_store(a), Y = add_store(b);
        int rl = 0;
        const int G = activated(cur, a, fin, A, 1.f, norm ? pend + 1 : 0, rl);
        program_.push_back({OpKind::barrier});
        Op ag{OpKind::aggregate, G, A};
        ag.relu = rl;
        program_.push_back(ag);
        hidden_.push_back(A);
        Op d{OpKind::dense, A, Y, -1, W, -1, -1, 0, last ? 2u : 0u, 1.f, 0};
        d.rs = norm ? 1 : 0;
        program_.push_back(d);
        if (last) output_ = Y;
        cur = Y;
        pend = 0;
      }
      cur_w = b;
      fin = 1;
    } else {
      // GIN layer l: MLP((1+eps) h_v + Σ h_u), MLP = Lin(a,h)-ReLU-Lin(h,b)
      const std::uint32_t a = cur_w, h = s.hidden;
      const std::uint32_t b = last ? s.out_dim : s.hidden;
      need(s.w1, o1 + std::size_t(a) * h, "gin W1");
      need(s.b1, ob1 + h, "gin b1");
      need(s.w2, o2 + std::size_t(h) * b, "gin W2");
      need(s.b2, ob2 + b, "gin b2");
      const int W1 = add_weight(s.w1.data() + o1, std::size_t(a) * h);
      const int B1 = add_weight(s.b1.data() + ob1, h);
      const int W2 = add_weight(s.w2.data() + o2, std::size_t(h) * b);
      const int B2 = add_weight(s.b2.data() + ob2, b);
      o1 += std::size_t(a) * h;
      ob1 += h;
      o2 += std::size_t(h) * b;
      ob2 += b;
      const float self = 1.f + s.eps;
      const int O = add_store(b);
      // h <= a: T = f(H)·W1; A = (1+eps)T + Σ T_u; O = ReLU(A+b1)·W2 + b2.
      // At h == a the aggregation width is the same either way, but this
      // order needs no separate self-term pass (the GEMM epilogue seeds A)
      // and one GEMM after the aggregation instead of two.
      if (h <= a) {
        const int T = add_store(h), A = add_store(h);
        program_.push_back({OpKind::dense, cur, T, A, W1, -1, -1, std::uint32_t(fin), 0, self, 0});
        program_.push_back({OpKind::barrier});
        program_.push_back({OpKind::aggregate, T, A});
        hidden_.push_back(A);
        program_.push_back({OpKind::dense, A, O, -1, W2, B2, B1, 2, last ? 2u : 0u, 1.f, 0});
      } else {  // A = (1+eps) f(H) + Σ f(H_u); M = ReLU(A·W1+b1); O = M·W2+b2
        const int A = add_store(a), M = add_store(h);
        int rl = 0;
        const int G = activated(cur, a, fin, A, self, 0, rl);
        program_.push_back({OpKind::barrier});
        Op ag{OpKind::aggregate, G, A};
        ag.relu = rl;
        program_.push_back(ag);
        hidden_.push_back(A);
        program_.push_back({OpKind::dense, A, M, -1, W1, B1, -1, 0, 1, 1.f, 0});
        program_.push_back({OpKind::dense, M, O, -1, W2, B2, -1, 0, last ? 2u : 0u, 1.f, 0});
      }
      if (last) output_ = O;
      cur = O;
      cur_w = b;
      fin = 1;
    }
    // the next layer's aggregation reads this layer's output from peers
  }
}

void Engine::free_plans() {
  eager_warm_ = false;  // new plans: halo buffers are re-created by an eager pass
  if (exec_) {  // the captured forward references these plans
    mgg_ctx_synchronize(ctx_);
    mgg_exec_destroy(exec_);
    exec_ = nullptr;
    exec_input_ = nullptr;
  }
  for (auto*& p : plans_) {
    mgg_dplan_destroy(p);
    p = nullptr;
  }
  for (auto& per : halo_bufs_)
    for (auto& [dim, buf] : per) mgg_dbuf_destroy(buf);
  halo_bufs_.assign(num_parts_, {});
}

const float* Engine::halo_for(std::uint32_t p, std::uint32_t dim) {
  if (!halo_on_[p]) return nullptr;
  for (auto& [w, buf] : halo_bufs_[p])
    if (w == dim) return static_cast<const float*>(mgg_dbuf_ptr(buf));
  std::uint64_t rows = 0;
  ok(mgg_dplan_halo_len(plans_[p], &rows));
  mgg_dbuf* buf = nullptr;
  ok(mgg_dbuf_create(ctx_, p, nullptr, std::max<std::uint64_t>(rows, 1) * ((dim + 3) / 4 * 4) * 4,
                     &buf));
  halo_bufs_[p].push_back({dim, buf});
  return static_cast<const float*>(mgg_dbuf_ptr(buf));
}

void Engine::set_remote_fetch(RemoteFetch mode) {
  ok(mgg_ctx_synchronize(ctx_));
  fetch_ = mode;
  build_plans();
}

void Engine::build_plans() {
  free_plans();
  plans_.assign(num_parts_, nullptr);
  halo_on_.assign(num_parts_, 0);
  stats_ = {};
  const auto t0 = std::chrono::steady_clock::now();
  for (std::uint32_t p = 0; p < num_parts_; ++p) {
    if (dev_[p] < 0) continue;
    const FlatPlan fp =
        build_flat_plan(g_, split_, ne_, p, cfg_, spec_.in_dim, mapping_, granularity_);
    HaloPlan halo;
    if (fetch_ != RemoteFetch::fine && !fp.remote.cols.empty()) {
      halo = build_halo_plan(fp);
      halo_on_[p] = fetch_ == RemoteFetch::halo || halo.dedup_ratio() >= 2.0;
    }
    mgg_plan_desc d{};
    if (halo_on_[p]) {
      d.halo_rows = halo.rows.data();
      d.halo_len = halo.rows.size();
      d.remote_halo_cols = halo.cols.data();
      stats_.halo_rows += halo.rows.size();
      stats_.halo_parts += 1;
    }
    d.part = p;
    d.ps = cfg_.ps;
    d.dist = cfg_.dist;
    d.wpb = cfg_.wpb;
    d.mapping = mapping_ == MappingMode::interleaved ? 0 : 1;
    d.granularity = granularity_ == Granularity::partitioned ? 0 : 1;
    d.rows = fp.rows;
    d.n_local = fp.local.num_parts();
    d.n_remote = fp.remote.num_parts();
    d.local_meta = fp.local.meta.data();
    d.local_cols = fp.local.cols.data();
    d.local_cols_len = fp.local.cols.size();
    d.remote_meta = fp.remote.meta.data();
    d.remote_cols = fp.remote.cols.data();
    d.remote_cols_len = fp.remote.cols.size();
    ok(mgg_dplan_upload(ctx_, &d, &plans_[p]));
    ok(mgg_dplan_set_k1_form(plans_[p], k1_form_));
    stats_.local_parts += d.n_local;
    stats_.remote_parts += d.n_remote;
    stats_.local_edges += d.local_cols_len;
    stats_.remote_edges += d.remote_cols_len;
    stats_.warps += fp.num_warps();
    stats_.blocks += fp.num_blocks();
  }
  stats_.plan_build_ns = static_cast<std::uint64_t>(
      std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count());
}

void Engine::set_config(const KernelConfig& cfg) {
  const auto v = validate(cfg, builtin_profile("b200"), spec_.in_dim);
  if (!v.empty()) throw ConfigError("engine: config violates " + v.front().constraint);
  ok(mgg_ctx_synchronize(ctx_));
  cfg_ = cfg;
  build_plans();
}

void Engine::set_mapping(MappingMode mapping, Granularity granularity) {
  ok(mgg_ctx_synchronize(ctx_));
  mapping_ = mapping;
  granularity_ = granularity;
  build_plans();
}

std::vector<std::uint8_t> Engine::export_ipc(std::uint32_t part) const {
  std::vector<std::uint8_t> blob;
  auto put = [&](const mgg_store* s) {
    std::uint8_t h[64];
    ok(mgg_store_ipc_export(s, part, h));
    blob.insert(blob.end(), h, h + 64);
  };
  put(flags_);
  for (auto* s : stores_) put(s);
  return blob;
}

void Engine::import_ipc(std::uint32_t part, const std::vector<std::uint8_t>& blob) {
  if (blob.size() != 64 * (stores_.size() + 1))
    throw InputError("engine: IPC blob does not match this engine's stores");
  ok(mgg_store_ipc_import(flags_, part, blob.data()));
  for (std::size_t i = 0; i < stores_.size(); ++i)
    ok(mgg_store_ipc_import(stores_[i], part, blob.data() + 64 * (i + 1)));
}

bool Engine::vmm_ipc() const {
  int sym = 0;
  ok(mgg_store_layout(flags_, &sym, nullptr));
  return sym == 2;
}

std::vector<int> Engine::export_vmm(std::uint32_t part) const {
  std::vector<int> fds;
  auto put = [&](const mgg_store* s) {
    int fd = -1;
    ok(mgg_store_vmm_export(s, part, &fd));
    fds.push_back(fd);
  };
  put(flags_);
  for (auto* s : stores_) put(s);
  return fds;
}

void Engine::import_vmm(std::uint32_t part, const std::vector<int>& fds) {
  if (fds.size() != stores_.size() + 1)
    throw InputError("engine: VMM fd list does not match this engine's stores");
  ok(mgg_store_vmm_import(flags_, part, fds[0]));
  for (std::size_t i = 0; i < stores_.size(); ++i)
    ok(mgg_store_vmm_import(stores_[i], part, fds[i + 1]));
}

void Engine::run(const Op& op) {
  if (op.kind == OpKind::barrier) {
    ok(mgg_barrier(ctx_, flags_));
    return;
  }
  for (std::uint32_t p = 0; p < num_parts_; ++p) {
    if (dev_[p] < 0) continue;
    switch (op.kind) {
      case OpKind::dense: {
        mgg_dense_desc d{};
        d.w = weights_[op.w][p];
        d.bias = op.bias >= 0 ? weights_[op.bias][p] : nullptr;
        d.pre_bias = op.pre_bias >= 0 ? weights_[op.pre_bias][p] : nullptr;
        d.pre = op.pre;
        d.act = op.act;
        d.out2_scale = op.scale;
        d.row_scale = op.rs ? rs_[op.rs][p] : nullptr;
        ok(mgg_dense(ctx_, p, stores_[op.in], &d, stores_[op.out],
                     op.out2 >= 0 ? stores_[op.out2] : nullptr));
        break;
      }
      case OpKind::dense_chain: {
        mgg_dense_desc d1{}, d2{};
        d1.w = weights_[op.w][p];
        d1.bias = op.bias >= 0 ? weights_[op.bias][p] : nullptr;
        d1.pre_bias = op.pre_bias >= 0 ? weights_[op.pre_bias][p] : nullptr;
        d1.pre = op.pre;
        d2.w = weights_[op.w2][p];
        d2.pre = 1;
        d2.out2_scale = op.scale;
        std::uint32_t m1 = 0;
        ok(mgg_store_info(stores_[op.mid], &m1, nullptr));
        ok(mgg_dense_chain(ctx_, p, stores_[op.in], &d1, m1, &d2, stores_[op.out],
                           op.out2 >= 0 ? stores_[op.out2] : nullptr));
        break;
      }
      case OpKind::init:
        ok(mgg_rows_init_rs(ctx_, p, stores_[op.in], stores_[op.out], op.scale, op.relu,
                            op.out2 >= 0 ? stores_[op.out2] : nullptr,
                            op.rs ? rs_[op.rs][p] : nullptr));
        break;
      case OpKind::aggregate: {
        std::uint32_t w = 0;
        ok(mgg_store_info(stores_[op.in], &w, nullptr));
        mgg_agg_opts o{op.relu, 0, halo_for(p, w), 1};
        ok(mgg_aggregate(ctx_, plans_[p], stores_[op.in], stores_[op.out], &o));
        break;
      }
      case OpKind::softmax:
        ok(mgg_rows_softmax_rs(ctx_, p, stores_[op.in], stores_[op.out],
                               op.rs ? rs_[op.rs][p] : nullptr));
        break;
      case OpKind::barrier:
        break;
    }
  }
}

void Engine::set_input(const float* x) {
  ok(mgg_store_upload(stores_[input_], x, 0, g_.num_nodes, spec_.in_dim));
}

void Engine::forward() {
  // the forward replays as one CUDA graph of this process's parts: between
  // parts of this process the barriers are event joins across their streams,
  // towards parts in other processes K3 flag kernels (device-held epoch, so
  // every replay advances it; each process replays its own graph)
  const bool graphable = graphs_ && !profiling_;
  if (!graphable) {
    forward_ops(false);
    return;
  }
  if (exec_ && exec_input_ != stores_[input_]) drop_exec();  // streamed double buffer swapped
  if (!eager_warm_) {
    // first forward runs eagerly: one-time work (tcgen05 weight splits,
    // halo buffers) must not become nodes of the captured graph
    forward_ops(false);
    eager_warm_ = true;
    return;
  }
  if (!exec_) {
    ok(mgg_capture_begin(ctx_));
    try {
      forward_ops(false);
    } catch (...) {
      mgg_exec* junk = nullptr;
      mgg_capture_end(ctx_, &junk);
      mgg_exec_destroy(junk);
      throw;
    }
    ok(mgg_capture_end(ctx_, &exec_));
    exec_input_ = stores_[input_];
  }
  ok(mgg_exec_launch(ctx_, exec_));
}

// D^-1/2 and D^-1 over each local part's rows (d_v = |N(v)| + 1, the
// oracle's inv_sqrt_deg), for the normalised GCN's row scalings.
void Engine::build_row_scales() {
  for (auto& v : rs_) v.assign(num_parts_, nullptr);
  if (!(spec_.kind == ModelSpec::Kind::gcn && spec_.norm)) return;
  for (std::uint32_t p = 0; p < num_parts_; ++p) {
    if (dev_[p] < 0) continue;
    const std::uint64_t lb = ne_.ranges[p].lb, n = ne_.ranges[p].size();
    std::vector<float> s1(std::max<std::uint64_t>(n, 1)), s2(s1.size());
    for (std::uint64_t r = 0; r < n; ++r) {
      const double d = double(g_.row_ptr[lb + r + 1] - g_.row_ptr[lb + r]) + 1.0;
      s1[r] = static_cast<float>(1.0 / std::sqrt(d));
      s2[r] = static_cast<float>(1.0 / d);
    }
    ok(mgg_dbuf_create(ctx_, p, s1.data(), s1.size() * sizeof(float), &rs_[1][p]));
    ok(mgg_dbuf_create(ctx_, p, s2.data(), s2.size() * sizeof(float), &rs_[2][p]));
  }
}

void Engine::set_graphs(bool on) {
  graphs_ = on;
  if (!on) drop_exec();
}

void Engine::set_k1_form(std::uint32_t form) {
  if (form > 3) throw InputError("engine: k1 form must be 0..3");
  ok(mgg_ctx_synchronize(ctx_));
  drop_exec();  // the captured graph holds the previous kernels
  k1_form_ = form;
  for (auto* p : plans_)
    if (p) ok(mgg_dplan_set_k1_form(p, form));
}

void Engine::drop_exec() {
  if (!exec_) return;
  ok(mgg_ctx_synchronize(ctx_));
  mgg_exec_destroy(exec_);
  exec_ = nullptr;
  exec_input_ = nullptr;
}

// `streamed`: the forward of submit_host — its input arrives on the H2D lane
// and its output leaves on the D2H lane, fenced so that the next forward's
// H2D starts as soon as this one has consumed the input store.
void Engine::forward_ops(bool streamed) {
  auto fence_all = [&](int from, int to) {
    for (std::uint32_t p = 0; p < num_parts_; ++p)
      if (dev_[p] >= 0) ok(mgg_lane_fence(ctx_, p, from, to));
  };
  // inputs of every part must be resident before the first peer gather
  ok(mgg_barrier(ctx_, flags_));
  if (profiling_) {
    prof_starts_.push_back(next_slot_);
    ok(mgg_event_record(ctx_, prof_part_, next_slot_++));
  }
  for (std::size_t i = 0; i < program_.size(); ++i) {
    if (streamed && static_cast<int>(i) == out_first_write_)
      fence_all(MGG_LANE_D2H, MGG_LANE_COMPUTE);  // previous z has left the device
    run(program_[i]);
    if (i + 1 == program_.size()) ok(mgg_ctx_join(ctx_));  // concurrent parts: end together
    if (profiling_) ok(mgg_event_record(ctx_, prof_part_, next_slot_++));
    if (streamed && static_cast<int>(i) == in_last_use_) {
      if (in_bufs_[1]) {  // this buffer is free for the submission after next
        const int b = stores_[input_] == in_bufs_[0] ? 0 : 1;
        for (std::uint32_t p = 0; p < num_parts_; ++p)
          if (dev_[p] >= 0)
            ok(mgg_lane_mark(ctx_, p, MGG_LANE_COMPUTE, static_cast<std::uint32_t>(kMarkSlots + b)));
        in_marked_[b] = true;
      } else {
        fence_all(MGG_LANE_COMPUTE, MGG_LANE_H2D);  // next x may overwrite the input
      }
    }
  }
}

// GIN layer boundaries: dense(A -> O; W2, b2, pre b1+ReLU) followed by
// dense(O -> T', A'; W1', ReLU in, seed) become one chained tcgen05 kernel
// whose intermediate O stays in TMEM (mgg_dense_chain): 1.25 GB less HBM
// traffic per boundary on the products-shaped graph.
void Engine::fuse_chains() {
  const char* e = std::getenv("MGG_CHAIN");
  if (e && std::string(e) == "0") return;
  std::vector<Op> out;
  for (std::size_t i = 0; i < program_.size(); ++i) {
    const Op& a = program_[i];
    if (i + 1 < program_.size() && a.kind == OpKind::dense && a.act == 0 && a.out2 < 0 &&
        a.out != output_) {
      const Op& b = program_[i + 1];
      int uses = 0;  // O must feed only b
      for (const Op& o : program_) uses += (o.in == a.out) + (o.out2 == a.out);
      std::uint32_t k = 0, m1 = 0, m = 0;
      ok(mgg_store_info(stores_[a.in], &k, nullptr));
      ok(mgg_store_info(stores_[a.out], &m1, nullptr));
      if (b.kind == OpKind::dense && b.in == a.out && b.pre == 1 && b.bias < 0 && b.act == 0 &&
          uses == 1) {
        ok(mgg_store_info(stores_[b.out], &m, nullptr));
        if (mgg_dense_chain_supported(k, m1, m)) {
          Op c = b;
          c.kind = OpKind::dense_chain;
          c.in = a.in;
          c.mid = a.out;
          c.w = a.w;
          c.bias = a.bias;
          c.pre_bias = a.pre_bias;
          c.pre = a.pre;
          c.w2 = b.w;
          out.push_back(c);
          ++i;
          continue;
        }
      }
    }
    out.push_back(a);
  }
  program_ = std::move(out);
}

// Last op after which no kernel (of any part) reads the input store, and the
// first op writing the output store.
void Engine::find_io_points() {
  in_last_use_ = -1;
  out_first_write_ = -1;
  bool peer_read = false;
  for (std::size_t i = 0; i < program_.size(); ++i) {
    const Op& op = program_[i];
    if (op.in == input_) {
      in_last_use_ = static_cast<int>(i);
      peer_read = op.kind == OpKind::aggregate && num_parts_ > 1;
    }
    if (out_first_write_ < 0 && (op.out == output_ || op.out2 == output_))
      out_first_write_ = static_cast<int>(i);
  }
  bool any_gather = false;
  for (const Op& op : program_) any_gather |= op.kind == OpKind::aggregate && op.in == input_;
  if (peer_read) {
    // peers gather the input too: it is free once every part has passed the
    // next K3 barrier (each part reaches it only after its own gathers)
    int j = in_last_use_ + 1;
    while (j < static_cast<int>(program_.size()) && program_[j].kind != OpKind::barrier) ++j;
    in_last_use_ = std::min(j, static_cast<int>(program_.size()) - 1);
  }
  if (!any_gather) {
    // the input is read only by this part's own GEMM: a second buffer lets
    // the next H2D run while the current forward still reads the first
    in_bufs_[0] = stores_[input_];
    std::vector<std::uint64_t> lb(num_parts_ + 1);
    for (std::uint32_t p = 0; p < num_parts_; ++p) lb[p] = ne_.ranges[p].lb;
    lb[num_parts_] = g_.num_nodes;
    ok(mgg_store_create(ctx_, lb.data(), spec_.in_dim, &in_bufs_[1]));
  }
}

std::uint64_t Engine::submit_host(const float* x, float* z) {
  if (submitted_ - completed_ >= kMaxInFlight) wait(submitted_ - kMaxInFlight + 1);
  const std::uint64_t ticket = ++submitted_;
  if (in_bufs_[1]) {
    const int b = static_cast<int>(ticket & 1);
    stores_[input_] = in_bufs_[b];
    if (in_marked_[b])  // the forward that last read this buffer is done with it
      for (std::uint32_t p = 0; p < num_parts_; ++p)
        if (dev_[p] >= 0)
          ok(mgg_lane_wait_mark(ctx_, p, MGG_LANE_H2D, static_cast<std::uint32_t>(kMarkSlots + b)));
  }
  ok(mgg_store_upload_on(stores_[input_], x, 0, g_.num_nodes, spec_.in_dim, MGG_LANE_H2D));
  for (std::uint32_t p = 0; p < num_parts_; ++p)
    if (dev_[p] >= 0) ok(mgg_lane_fence(ctx_, p, MGG_LANE_H2D, MGG_LANE_COMPUTE));
  forward_ops(true);
  for (std::uint32_t p = 0; p < num_parts_; ++p)
    if (dev_[p] >= 0) ok(mgg_lane_fence(ctx_, p, MGG_LANE_COMPUTE, MGG_LANE_D2H));
  ok(mgg_store_download_on(stores_[output_], z, 0, g_.num_nodes, spec_.out_dim, MGG_LANE_D2H));
  for (std::uint32_t p = 0; p < num_parts_; ++p)
    if (dev_[p] >= 0)
      ok(mgg_lane_mark(ctx_, p, MGG_LANE_D2H, static_cast<std::uint32_t>(ticket % kMarkSlots)));
  return ticket;
}

void Engine::wait(std::uint64_t ticket) {
  if (ticket == 0 || ticket > submitted_) throw InputError("engine: unknown ticket");
  if (ticket <= completed_) return;
  // marks are recorded in ticket order on one lane: waiting for `ticket`
  // also completes every earlier one (a slot re-marked by a newer ticket
  // only waits longer)
  for (std::uint32_t p = 0; p < num_parts_; ++p)
    if (dev_[p] >= 0)
      ok(mgg_lane_wait_host(ctx_, p, static_cast<std::uint32_t>(ticket % kMarkSlots)));
  completed_ = ticket;
}

void Engine::set_profiling(bool on) {
  profiling_ = on;
  next_slot_ = 0;
  prof_starts_.clear();
  for (std::uint32_t p = 0; p < num_parts_; ++p)
    if (dev_[p] >= 0) {
      prof_part_ = p;
      break;
    }
}

std::vector<Engine::OpProfile> Engine::profile(std::uint64_t* forwards) {
  std::vector<OpProfile> out(program_.size());
  for (std::size_t i = 0; i < program_.size(); ++i) {
    out[i].kind = static_cast<std::uint32_t>(program_[i].kind);
    if (program_[i].out >= 0) ok(mgg_store_info(stores_[program_[i].out], &out[i].width, nullptr));
  }
  for (std::uint32_t s0 : prof_starts_)
    for (std::size_t i = 0; i < program_.size(); ++i) {
      float ms = 0;
      ok(mgg_event_elapsed(ctx_, prof_part_, s0 + static_cast<std::uint32_t>(i),
                           s0 + static_cast<std::uint32_t>(i) + 1, &ms));
      out[i].ms += ms;
    }
  if (forwards) *forwards = prof_starts_.size();
  return out;
}

void Engine::synchronize() { ok(mgg_ctx_synchronize(ctx_)); }

void Engine::get_output(float* z) {
  ok(mgg_store_download(stores_[output_], z, 0, g_.num_nodes, spec_.out_dim));
  synchronize();
}

void Engine::forward_host(const float* x, float* z) { wait(submit_host(x, z)); }

std::uint32_t Engine::get_hidden(std::uint32_t which, float* rows) {
  if (which >= hidden_.size()) throw InputError("engine: no such hidden layer");
  std::uint32_t dim = 0;
  ok(mgg_store_info(stores_[hidden_[which]], &dim, nullptr));
  if (rows) {
    ok(mgg_store_download(stores_[hidden_[which]], rows, 0, g_.num_nodes, dim));
    synchronize();
  }
  return dim;
}

std::uint32_t Engine::get_logits(float* rows) {
  // the op that produced the output: a dense with the softmax epilogue, or a
  // softmax pass over an aggregated store
  int head = -1;
  for (std::size_t i = 0; i < program_.size(); ++i)
    if (program_[i].out == output_) head = static_cast<int>(i);
  if (head < 0) throw InputError("engine: no output op");
  Op op = program_[head];
  std::uint32_t width = 0;
  ok(mgg_store_info(stores_[output_], &width, nullptr));
  if (!rows) return width;
  for (auto d : dev_)
    if (d < 0) throw InputError("engine: get_logits needs every part in this process");
  mgg_store* lg = scratch(width, 1);
  for (std::uint32_t p = 0; p < num_parts_; ++p) {
    if (op.kind == OpKind::softmax) {  // logits = (row scale ·) the aggregated rows
      ok(mgg_rows_init_rs(ctx_, p, stores_[op.in], lg, 1.f, 0, nullptr,
                          op.rs ? rs_[op.rs][p] : nullptr));
    } else if (op.kind == OpKind::dense) {  // the same K2 head, no softmax epilogue
      mgg_dense_desc d{};
      d.w = weights_[op.w][p];
      d.bias = op.bias >= 0 ? weights_[op.bias][p] : nullptr;
      d.pre_bias = op.pre_bias >= 0 ? weights_[op.pre_bias][p] : nullptr;
      d.pre = op.pre;
      d.act = op.act == 2 ? 0 : op.act;
      d.out2_scale = 1.f;
      d.row_scale = op.rs ? rs_[op.rs][p] : nullptr;
      ok(mgg_dense(ctx_, p, stores_[op.in], &d, lg, nullptr));
    } else {
      throw InputError("engine: output op is not a dense or softmax");
    }
  }
  ok(mgg_store_download(lg, rows, 0, g_.num_nodes, width));
  synchronize();
  return width;
}

mgg_store* Engine::scratch(std::uint32_t dim, int slot) {
  std::uint32_t have = 0;
  if (scratch_[slot]) ok(mgg_store_info(scratch_[slot], &have, nullptr));
  if (!scratch_[slot] || have != dim) {
    mgg_store_destroy(scratch_[slot]);
    scratch_[slot] = nullptr;
    std::vector<std::uint64_t> lb(num_parts_ + 1);
    for (std::uint32_t p = 0; p < num_parts_; ++p) lb[p] = ne_.ranges[p].lb;
    lb[num_parts_] = g_.num_nodes;
    ok(mgg_store_create(ctx_, lb.data(), dim, &scratch_[slot]));
  }
  return scratch_[slot];
}

void Engine::aggregate_host(const float* x, std::uint32_t dim, float self_scale,
                            bool relu_in, float* out, int phase) {
  if (phase < 0 || phase > 3) throw InputError("engine: aggregate phase must be 0..3");
  for (auto d : dev_)
    if (d < 0) throw InputError("engine: aggregate_host needs every part in this process");
  mgg_store* in = scratch(dim, 0);
  mgg_store* acc = scratch(dim, 1);
  ok(mgg_store_upload(in, x, 0, g_.num_nodes, dim));
  for (std::uint32_t p = 0; p < num_parts_; ++p)
    ok(mgg_rows_init(ctx_, p, in, acc, self_scale, relu_in ? 1 : 0));
  ok(mgg_barrier(ctx_, flags_));
  for (std::uint32_t p = 0; p < num_parts_; ++p) {
    mgg_agg_opts o{relu_in ? 1 : 0, phase, halo_for(p, dim), 1};
    ok(mgg_aggregate(ctx_, plans_[p], in, acc, &o));
  }
  ok(mgg_store_download(acc, out, 0, g_.num_nodes, dim));
  synchronize();
}

// A model store pair of width `dim` (valid across processes: peers imported
// them), else the scratch pair (single-process only).
std::pair<mgg_store*, mgg_store*> Engine::agg_stores(std::uint32_t dim) {
  for (const Op& op : program_)
    if (op.kind == OpKind::aggregate) {
      std::uint32_t w = 0;
      ok(mgg_store_info(stores_[op.in], &w, nullptr));
      if (w == dim) return {stores_[op.in], stores_[op.out]};
    }
  return {scratch(dim, 0), scratch(dim, 1)};
}

std::uint64_t Engine::time_aggregate(std::uint32_t dim, std::uint32_t reps, int phase) {
  const auto each = time_aggregate_each(dim, reps, phase);
  return each.empty() ? 0 : *std::max_element(each.begin(), each.end());
}

std::vector<std::uint64_t> Engine::time_aggregate_each(std::uint32_t dim, std::uint32_t reps,
                                                       int phase) {
  auto [in, out] = agg_stores(dim);
  std::vector<std::uint64_t> ns(num_parts_, 0);
  for (std::uint32_t p = 0; p < num_parts_; ++p) {
    if (dev_[p] < 0) continue;
    // halo mode: each timed rep includes the deduplicated pull
    mgg_agg_opts o{0, phase, halo_for(p, dim), 1};
    ok(mgg_time_aggregate(ctx_, plans_[p], in, out, &o, reps, &ns[p]));
  }
  return ns;
}

Engine::MultiGpuReport Engine::measure_multi_gpu(std::uint32_t dim, std::uint32_t reps) {
  reps = std::max(reps, 1u);
  auto [in, out] = agg_stores(dim);
  const auto alone = time_aggregate_each(dim, reps, 0);
  std::vector<std::uint32_t> local;
  for (std::uint32_t p = 0; p < num_parts_; ++p)
    if (dev_[p] >= 0) local.push_back(p);
  if (local.empty()) throw InputError("engine: no local part");
  const std::uint32_t p0 = local.front();
  bool one_device = true;
  for (auto p : local) one_device &= dev_[p] == dev_[p0];
  // slots: per part [base + 3r] start, [+1] K1 end, [+2] after the barrier
  constexpr std::uint32_t base = 200000;
  std::vector<std::vector<float>> k1(num_parts_), upto(num_parts_);
  for (std::uint32_t r = 0; r <= reps; ++r) {  // rep 0 warms up
    ok(mgg_barrier(ctx_, flags_));  // start-aligned: every part past its tail
    for (auto p : local) ok(mgg_event_record(ctx_, p, base + 3 * r));
    for (auto p : local) {
      mgg_agg_opts o{0, 0, halo_for(p, dim), 1};
      ok(mgg_aggregate(ctx_, plans_[p], in, out, &o));
      ok(mgg_event_record(ctx_, p, base + 3 * r + 1));
    }
    ok(mgg_barrier(ctx_, flags_));
    for (auto p : local) ok(mgg_event_record(ctx_, p, base + 3 * r + 2));
  }
  for (std::uint32_t r = 1; r <= reps; ++r)
    for (auto p : local) {
      float a = 0, b = 0;
      ok(mgg_event_elapsed(ctx_, p, base + 3 * r, base + 3 * r + 1, &a));
      if (one_device)  // parts of one device: from the common start
        ok(mgg_event_elapsed_between(ctx_, p0, base + 3 * r, p, base + 3 * r + 2, &b));
      else
        ok(mgg_event_elapsed(ctx_, p, base + 3 * r, base + 3 * r + 2, &b));
      k1[p].push_back(a);
      upto[p].push_back(b);
    }
  auto median = [](std::vector<float> v) {
    std::sort(v.begin(), v.end());
    return static_cast<std::uint64_t>(double(v[v.size() / 2]) * 1e6);
  };
  MultiGpuReport rep;
  std::uint64_t until = 0;
  for (auto p : local) {
    PartReport pr;
    pr.part = p;
    pr.total_ns = median(k1[p]);
    pr.alone_ns = alone[p];
    std::uint32_t info[4] = {0, 0, 0, 0};
    ok(mgg_dplan_k1_launch_info(plans_[p], info));
    const double slots_per_sm = 2048.0;  // 64 resident warps per sm_100 SM
    pr.active_sms = std::min(info[0], info[3]);
    const double per_sm = info[3] ? double(info[0]) / info[3] : 0.0;  // CTAs per SM
    pr.achieved_occupancy = std::min(per_sm, double(info[2])) * info[1] / slots_per_sm;
    pr.sm_utilization = info[3] ? double(pr.active_sms) / info[3] : 0.0;
    pr.kernels = k1_kernels(p);
    std::uint32_t pitch = 0;
    ok(mgg_store_info(in, nullptr, &pitch));
    const FlatPlan fp =
        build_flat_plan(g_, split_, ne_, p, cfg_, spec_.in_dim, mapping_, granularity_);
    std::uint64_t halo_rows = 0;
    ok(mgg_dplan_halo_len(plans_[p], &halo_rows));
    pr.local_bytes = std::uint64_t(fp.local.cols.size()) * pitch * 4;
    pr.remote_bytes =
        (halo_for(p, dim) ? halo_rows : std::uint64_t(fp.remote.cols.size())) * pitch * 4;
    pr.num_warps = static_cast<std::uint32_t>(fp.num_warps());
    pr.num_blocks = static_cast<std::uint32_t>(fp.num_blocks());
    rep.max_gpu_ns = std::max(rep.max_gpu_ns, pr.total_ns);
    rep.max_alone_ns = std::max(rep.max_alone_ns, pr.alone_ns);
    until = std::max(until, median(upto[p]));
    rep.remote_bytes += pr.remote_bytes;
    rep.mean_occupancy += pr.achieved_occupancy / local.size();
    rep.mean_utilization += pr.sm_utilization / local.size();
    rep.per_gpu.push_back(std::move(pr));
  }
  rep.total_ns = std::max(until, rep.max_gpu_ns);
  rep.barrier_ns = rep.total_ns - rep.max_gpu_ns;
  std::vector<std::int32_t> devs;
  for (auto p : local)
    if (std::find(devs.begin(), devs.end(), dev_[p]) == devs.end()) devs.push_back(dev_[p]);
  rep.devices = static_cast<std::uint32_t>(devs.size());
  return rep;
}

void Engine::set_shard_memory(std::uint32_t part, int kind) {
  if (part >= num_parts_ || dev_[part] < 0) throw InputError("engine: part is not local");
  for (auto d : dev_)
    if (d < 0) throw InputError("engine: shard memory kinds need every part in this process");
  synchronize();
  drop_exec();
  ok(mgg_ctx_set_shard_memory(ctx_, part, kind));
  std::vector<std::uint64_t> lb(num_parts_ + 1);
  for (std::uint32_t p = 0; p < num_parts_; ++p) lb[p] = ne_.ranges[p].lb;
  lb[num_parts_] = g_.num_nodes;
  const bool dbl = in_bufs_[1] != nullptr;
  for (auto* s : in_bufs_)
    if (s && s != stores_[input_]) mgg_store_destroy(s);
  in_bufs_[0] = in_bufs_[1] = nullptr;
  in_marked_[0] = in_marked_[1] = false;
  for (auto& s : stores_) {
    std::uint32_t dim = 0;
    ok(mgg_store_info(s, &dim, nullptr));
    mgg_store_destroy(s);
    s = nullptr;
    ok(mgg_store_create(ctx_, lb.data(), dim, &s));
  }
  if (dbl) {
    in_bufs_[0] = stores_[input_];
    ok(mgg_store_create(ctx_, lb.data(), spec_.in_dim, &in_bufs_[1]));
  }
  for (auto*& s : scratch_) {
    mgg_store_destroy(s);
    s = nullptr;
  }
  eager_warm_ = false;
}

std::string Engine::trace_csv(std::uint32_t dim, std::uint64_t capacity,
                              std::uint32_t warp_limit) {
  static constexpr const char* kStage[] = {"LR", "LL", "AC"};
  auto [in, out] = agg_stores(dim);
  std::string csv = "# mgg device trace: K1 width " + std::to_string(dim) + ", ps=" +
                    std::to_string(cfg_.ps) + " dist=" + std::to_string(cfg_.dist) +
                    " wpb=" + std::to_string(cfg_.wpb) +
                    "; cycle = SM clocks since the part's first event\n";
  csv += "gpu,cycle,sm,warp,stage,event\n";
  for (std::uint32_t p = 0; p < num_parts_; ++p) {
    if (dev_[p] < 0) continue;
    mgg_trace* tr = nullptr;
    ok(mgg_trace_create(ctx_, p, capacity, warp_limit, &tr));
    std::vector<std::uint64_t> ev;
    std::uint64_t n = 0, emitted = 0;
    try {
      mgg_agg_opts o{0, 0, nullptr, 0};
      ok(mgg_aggregate_traced(ctx_, plans_[p], in, out, &o, tr));
      ok(mgg_trace_read(tr, nullptr, 0, &n, &emitted));
      ev.resize(4 * n);
      ok(mgg_trace_read(tr, ev.data(), n, &n, &emitted));
    } catch (...) {
      mgg_trace_destroy(tr);
      throw;
    }
    mgg_trace_destroy(tr);
    std::vector<std::uint64_t> order(n);
    for (std::uint64_t i = 0; i < n; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](std::uint64_t a, std::uint64_t b) { return ev[4 * a] < ev[4 * b]; });
    for (std::uint64_t i : order) {
      const std::uint64_t code = ev[4 * i + 3];
      csv += std::to_string(p) + ',' + std::to_string(ev[4 * i]) + ',' +
             std::to_string(ev[4 * i + 1]) + ',' + std::to_string(ev[4 * i + 2]) + ',' +
             kStage[std::min<std::uint64_t>(code >> 1, 2)] + ',' +
             ((code & 1) ? "begin" : "end") + '\n';
    }
  }
  return csv;
}

Engine::Stats Engine::stats() const {
  Stats s = stats_;
  s.launches = mgg_ctx_launch_count(ctx_);
  return s;
}

std::string Engine::k1_kernels(std::uint32_t part) const {
  if (part >= num_parts_ || !plans_[part]) throw InputError("k1_kernels: part is not local");
  char buf[512];
  ok(mgg_dplan_k1_kernels(plans_[part], buf, sizeof buf));
  return buf;
}

}  // namespace mgg
