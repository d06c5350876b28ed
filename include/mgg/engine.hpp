// Multi-GPU GCN/GIN forward driver — the B200 counterpart of the reference's
// orchestration `multi_gpu_run` (R:proj/src/sim.cpp:597-624: split ->
// place -> per-GPU local/remote split -> plan -> execute -> max + barrier),
// now executing the layer arithmetic the reference leaves to the paper
// (GCN R:PAPER.md:504-508, GIN R:PAPER.md:511-517) on the sm_100a kernels
// through the C-ABI of include/mgg.h (layer A). Host-side C++ only.
//
// Layer programs. Every layer aggregates at the narrower of its two widths:
// Â·H·W = Â·(H·W), and for GIN the first MLP Linear commutes with the sum,
// ((1+eps)h_v + Σh_u)·W1 = (1+eps)(h_v·W1) + Σ(h_u·W1). A layer is then a
// short op list over symmetric stores — Dense (K2, may seed the aggregation
// accumulator with the self term), Init (self term), Barrier (K3: the next
// gather reads peer shards), Aggregate (K1), Softmax — and activations of a
// hidden layer are applied lazily by the consumer (ReLU-on-load), so no
// extra pass ever touches HBM for them.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "mgg/costmodel.hpp"
#include "mgg/graph.hpp"
#include "mgg/placement.hpp"
#include "mgg/workload.hpp"

struct mgg_ctx;
struct mgg_store;
struct mgg_dplan;
struct mgg_dbuf;
struct mgg_exec;

namespace mgg {

struct ModelSpec {
  enum class Kind { gcn, gin } kind = Kind::gcn;
  std::uint32_t layers = 2;
  std::uint32_t in_dim = 0, hidden = 0, out_dim = 0;
  float eps = 0.f;
  bool norm = false;  // GCN: D^-1/2 (A+I) D^-1/2, d_v = |N(v)| + 1
  // packed weights, layout of mgg_model_desc (include/mgg.h)
  std::vector<float> w1, b1, w2, b2;
};

class Engine {
 public:
  /// part_device[p] >= 0: this process drives part p on that device;
  /// -1: another process does (import its shards with import_ipc).
  /// `g` must outlive the engine (re-planning reads it).
  Engine(const CsrGraph& g, std::uint32_t num_parts,
         std::vector<std::int32_t> part_device, KernelConfig cfg, ModelSpec spec);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const WorkloadSplit& split() const { return split_; }
  const NePlacement& placement() const { return ne_; }
  const KernelConfig& config() const { return cfg_; }
  mgg_ctx* ctx() const { return ctx_; }
  std::uint32_t num_parts() const { return num_parts_; }

  std::vector<std::uint8_t> export_ipc(std::uint32_t part) const;
  void import_ipc(std::uint32_t part, const std::vector<std::uint8_t>& blob);
  /// Cross-process symmetric VMM stores (MGG_VMM_IPC=1): true when this
  /// engine's stores are fd-exportable VMM ranges; export returns one POSIX
  /// fd per store (the K3 flags first, caller-owned), import maps a peer's.
  bool vmm_ipc() const;
  std::vector<int> export_vmm(std::uint32_t part) const;
  void import_vmm(std::uint32_t part, const std::vector<int>& fds);

  void set_config(const KernelConfig& cfg);
  /// Ablation knobs of the reference's baselines (R:proj/src/sim.cpp:571-595):
  /// segregated = no_interleave, whole_list = no_np.
  void set_mapping(MappingMode mapping, Granularity granularity);
  /// Remote rows: per-edge peer reads inside K1 (fine, the paper's design),
  /// one deduplicated halo pull per layer then local reads (halo, a B200
  /// addition), or auto = halo when it moves >= 2x fewer NVLink bytes.
  enum class RemoteFetch { automatic, fine, halo };
  void set_remote_fetch(RemoteFetch mode);
  void set_input(const float* x);            // N x in_dim host rows
  void forward();                            // async, device resident
  /// Replay forward() from a captured CUDA graph when the context allows it
  /// (one device, all parts local, not profiling); on by default there.
  void set_graphs(bool on);
  /// Local-only K1 form for every plan (0 by shape, 1 warp-window, 2 group with
  /// 8 rows in flight, 3 group with 4); kept across re-plans.
  void set_k1_form(std::uint32_t form);
  std::uint32_t k1_form() const { return k1_form_; }
  void synchronize();
  void get_output(float* z);                 // N x out_dim host rows
  void forward_host(const float* x, float* z);  // submit_host + wait
  /// Streamed end to end (see mgg_engine_submit_host): the H2D of x and the
  /// D2H of z run on copy lanes fenced against the compute stream, so
  /// consecutive submissions overlap PCIe with kernels. x must stay valid and
  /// z untouched until wait(ticket).
  std::uint64_t submit_host(const float* x, float* z);
  void wait(std::uint64_t ticket);
  /// Post-aggregation accumulator of layer `which` (N x width host rows).
  std::uint32_t get_hidden(std::uint32_t which, float* rows);
  /// Pre-softmax logits of the last forward (N x out_dim host rows): the
  /// head K2 re-run on the device without its softmax epilogue (or the
  /// aggregated rows a softmax pass reads). Returns the width; rows may be null.
  std::uint32_t get_logits(float* rows);

  /// Standalone K1 through the engine's plans (single-process only);
  /// phase 1 = local partitions only, 2 = remote only (0 = both).
  void aggregate_host(const float* x, std::uint32_t dim, float self_scale,
                      bool relu_in, float* out, int phase = 0);
  /// Median K1 ns at width `dim`, max over local parts (each part alone).
  std::uint64_t time_aggregate(std::uint32_t dim, std::uint32_t reps, int phase);
  /// The same per local part (0 for parts of other processes).
  std::vector<std::uint64_t> time_aggregate_each(std::uint32_t dim, std::uint32_t reps,
                                                 int phase);

  /// Measured counterpart of the reference's SimReport / MultiGpuReport
  /// (R:proj/include/pipeshard/sim.hpp:62-78, 115-123; multi_gpu_run
  /// R:proj/src/sim.cpp:597-624): one K1 at width `dim` on every local part
  /// *concurrently* (start-aligned, then the K3/event barrier), median of
  /// `reps`. Per part: its K1 ns inside the concurrent run and alone, the
  /// remote bytes it moved, launch occupancy and SM coverage. total = max
  /// over parts + barrier. Several processes: each reports its own parts;
  /// the caller takes the max over ranks.
  struct PartReport {
    std::uint32_t part = 0;
    std::uint64_t total_ns = 0;    // K1 of this part while the others run too
    std::uint64_t alone_ns = 0;    // the same K1 with the device to itself
    double achieved_occupancy = 0; // resident warps / warp slots of the SMs it ran on
                                   // (occupancy calculator x grid; not an ncu counter)
    double sm_utilization = 0;     // SMs given CTAs / SMs of the device
    std::uint64_t remote_bytes = 0, local_bytes = 0;  // gathered-row bytes
    std::uint32_t num_warps = 0, num_blocks = 0, active_sms = 0;
    std::string kernels;
  };
  struct MultiGpuReport {
    std::vector<PartReport> per_gpu;
    std::uint64_t max_gpu_ns = 0, barrier_ns = 0, total_ns = 0, remote_bytes = 0;
    double mean_occupancy = 0, mean_utilization = 0;
    /// max over parts of alone_ns: the per-GPU time when logical parts share
    /// one device (their concurrent run measures contention a multi-GPU
    /// system does not have); equals ~max_gpu_ns with one part per device
    std::uint64_t max_alone_ns = 0;
    std::uint32_t devices = 0;  // distinct devices of the local parts
  };
  MultiGpuReport measure_multi_gpu(std::uint32_t dim, std::uint32_t reps);

  /// Placement of local part `part`'s shards (MGG_MEM_* of include/mgg.h):
  /// device (default), host-mapped (slow-peer emulation) or managed (the
  /// paged_remote baseline). Re-creates every store (contents are lost:
  /// set_input again); single-process engines only.
  void set_shard_memory(std::uint32_t part, int kind);
  /// Device event trace of one K1 at width `dim` on every local part, in the
  /// reference's multi-GPU trace CSV schema (R:proj/tools/cli.cpp:144-155).
  std::string trace_csv(std::uint32_t dim, std::uint64_t capacity, std::uint32_t warp_limit);

  /// Per-op device timing (CUDA events on the first local part's stream).
  void set_profiling(bool on);
  struct OpProfile {
    double ms = 0;           // accumulated over profiled forwards
    std::uint32_t kind = 0;  // 0 dense 1 init 2 aggregate 3 barrier 4 softmax 5 dense_chain
    std::uint32_t width = 0; // output columns
  };
  std::vector<OpProfile> profile(std::uint64_t* forwards);

  struct Stats {
    std::uint64_t local_parts = 0, remote_parts = 0, local_edges = 0,
                  remote_edges = 0, warps = 0, blocks = 0, launches = 0,
                  plan_build_ns = 0, halo_rows = 0, halo_parts = 0;
  };
  Stats stats() const;
  /// Kernels the latest K1 of local part `part` launched (mgg_dplan_k1_kernels).
  std::string k1_kernels(std::uint32_t part) const;

 private:
  enum class OpKind { dense, init, aggregate, barrier, softmax, dense_chain };
  struct Op {
    OpKind kind;
    int in = -1, out = -1, out2 = -1;  // store indices
    int w = -1, bias = -1, pre_bias = -1;  // weight slots
    std::uint32_t pre = 0, act = 0;
    float scale = 1.f;
    int relu = 0;
    int w2 = -1;  // dense_chain: second weight (O·W2), O = `mid` store's width
    int mid = -1;
    int rs = 0;   // normalised GCN: multiply the op's rows by D^-rs/2
  };

  int add_store(std::uint32_t dim);
  int add_weight(const float* src, std::size_t n);
  void build_program();
  int activated(int h, std::uint32_t width, int relu, int a, float scale, int rs,
                int& relu_load);
  // gather tables above this size are HBM-resident for K1 (half the 126 MB L2)
  static constexpr std::uint64_t kL2GatherBytes = 63ull << 20;
  void build_plans();
  void free_plans();
  void run(const Op& op);
  void forward_ops(bool streamed);
  void find_io_points();
  void fuse_chains();
  void build_row_scales();
  std::vector<mgg_dbuf*> rs_[3];  // [power][part]: D^-power/2 over the part's rows
  static constexpr std::uint64_t kMaxInFlight = 32, kMarkSlots = 64;
  int in_last_use_ = -1, out_first_write_ = -1;
  std::uint64_t submitted_ = 0, completed_ = 0;
  // Streamed input double buffer (only when no peer gathers the input):
  // submission t uploads into in_bufs_[t % 2] while t-1 computes on the other
  mgg_store* in_bufs_[2] = {nullptr, nullptr};
  bool in_marked_[2] = {false, false};
  mgg_store* scratch(std::uint32_t dim, int slot);
  std::pair<mgg_store*, mgg_store*> agg_stores(std::uint32_t dim);
  /// Halo buffer of part p for gather width `dim` (null when p reads fine).
  const float* halo_for(std::uint32_t p, std::uint32_t dim);
  RemoteFetch fetch_ = RemoteFetch::automatic;
  std::vector<std::uint8_t> halo_on_;                        // per part
  std::vector<std::vector<std::pair<std::uint32_t, mgg_dbuf*>>> halo_bufs_;  // per part

  const CsrGraph& g_;
  std::uint32_t num_parts_;
  std::vector<std::int32_t> dev_;
  KernelConfig cfg_;
  MappingMode mapping_ = MappingMode::interleaved;
  Granularity granularity_ = Granularity::partitioned;
  ModelSpec spec_;
  WorkloadSplit split_;
  NePlacement ne_;
  mgg_ctx* ctx_ = nullptr;
  std::vector<mgg_dplan*> plans_;     // per part (null if remote)
  std::vector<mgg_store*> stores_;    // model stores (IPC-exported)
  mgg_store* flags_ = nullptr;        // K3 flags
  std::vector<std::vector<mgg_dbuf*>> weights_;  // [slot][part]
  std::vector<Op> program_;
  int input_ = -1, output_ = -1;
  std::vector<int> hidden_;           // post-aggregation stores per layer
  mgg_store* scratch_[2] = {nullptr, nullptr};
  bool profiling_ = false;
  bool graphs_ = true;
  std::uint32_t k1_form_ = 0;
  bool eager_warm_ = false;           // one eager forward before the first capture
  mgg_exec* exec_ = nullptr;          // captured forward()
  mgg_store* exec_input_ = nullptr;   // input store the capture read
  void drop_exec();
  std::uint32_t prof_part_ = 0, next_slot_ = 0;
  std::vector<std::uint32_t> prof_starts_;  // first slot of each profiled forward
  Stats stats_;
};

}  // namespace mgg
