// Internal declarations of the device runtime (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "mgg.h"

namespace mgg::dev {

constexpr uint32_t kMaxParts = 16;

/// Thrown inside the runtime, turned into MGG_E_* at the ABI edge.
struct Status {
  int code;
  std::string msg;
};

void check(cudaError_t e, const char* what);
/// Thread-local message behind mgg_last_error() (shared with the host facade).
std::string& last_error();
#define MGG_CUDA(x) ::mgg::dev::check((x), #x)

}  // namespace mgg::dev

struct mgg_ctx {
  uint32_t num_parts = 0;
  std::vector<int32_t> device;         // -1: remote process
  std::vector<cudaStream_t> stream;    // per part (null for remote)
  std::vector<cudaEvent_t> ev0, ev1;   // timing events per part
  std::vector<cudaStream_t> aux;       // per part: halo pulls overlap local K1
  std::vector<cudaEvent_t> fork, join; // per part: main->aux, aux->main
  std::vector<std::vector<cudaEvent_t>> evpool;  // mgg_event_record slots
  // copy lanes (MGG_LANE_H2D / MGG_LANE_D2H): per device, shared by its parts
  std::vector<cudaStream_t> h2d, d2h;
  std::vector<cudaStream_t> rp;                   // per device: staging re-pitch kernels
  std::vector<std::vector<cudaEvent_t>> lane_ev;  // per part: [from*3+to] fences
  std::vector<std::vector<cudaEvent_t>> marks;    // per part: host-waitable slots
  uint64_t launches = 0;
  uint64_t capture_base = 0;           // launch count at mgg_capture_begin
  bool capturing = false;
  bool all_local = true;
  bool single_device = true;
  // parts sharing a device get their own compute/aux streams (concurrent
  // logical partitions); the K3 barrier becomes a cross-stream event join
  bool part_streams = false;
  std::vector<cudaEvent_t> bar_ev;     // per part: barrier join events
  std::vector<int> shard_mem;          // per part: MGG_MEM_* of new stores
};

struct mgg_store {
  mgg_ctx* ctx = nullptr;
  uint32_t dim = 0, pitch = 0;
  std::vector<uint64_t> lb;            // num_parts + 1
  std::vector<float*> shard;           // as seen by this process
  std::vector<uint8_t> owned, imported;
  std::vector<uint8_t> mem;            // per part: MGG_MEM_* of the shard
  std::vector<size_t> bytes;           // per local part: shard allocation
  // per local part: device copy of the shard table for that part's device
  std::vector<const float**> dtable;
  // per local part: two dense H2D/D2H slabs (2p, 2p+1) and their events
  // (5p + {full0, full1, free0, free1, tail}) — copies and re-pitch kernels
  // alternate slabs so the DMA engine never waits for a re-pitch
  std::vector<float*> stage;
  std::vector<cudaEvent_t> stage_ev;
  // symmetric VMM layout (single-process stores of device memory): one
  // virtual range, part p's shard at vmm_base + p * vmm_stride, physically
  // on part p's device and mapped for every local device (vmm_size per part)
  char* vmm_base = nullptr;
  uint64_t vmm_stride = 0;
  std::vector<size_t> vmm_size;
  // cross-process symmetric stores (MGG_VMM_IPC=1): the local shard's VMM
  // allocation handle (exported as a POSIX fd) and which slots are mapped
  bool vmm_ipc = false;
  std::vector<unsigned long long> vmm_handle;
  std::vector<uint8_t> vmm_mapped;
  uint64_t rows(uint32_t p) const { return lb[p + 1] - lb[p]; }
};

struct mgg_dbuf {
  mgg_ctx* ctx = nullptr;
  uint32_t part = 0;
  void* ptr = nullptr;
  size_t bytes = 0;
  void* tc_cache = nullptr;  // W^T hi/lo split for the tcgen05 GEMM
  uint32_t tc_k = 0, tc_m = 0;
};

struct mgg_exec {
  cudaGraphExec_t exec = nullptr;
  uint64_t kernels = 0;  // library launches captured (replays count them)
  int device = 0;
};

struct mgg_trace {
  mgg_ctx* ctx = nullptr;
  uint32_t part = 0;
  uint64_t capacity = 0;
  uint32_t warp_limit = 0;
  void* events = nullptr;  // capacity x 16 B
  unsigned long long* count = nullptr;
};

#ifndef MGG_KSHARDS
#define MGG_KSHARDS 16  // pair-kernel ticket counters (aggregate.cu for_each_ticket)
#endif
constexpr size_t kSchedBytes = (MGG_KSHARDS + 1) * 128;

struct mgg_dplan {
  mgg_ctx* ctx = nullptr;
  uint32_t part = 0;
  uint32_t ps = 1, dist = 1, wpb = 1, mapping = 0, granularity = 0;
  uint64_t rows = 0, n_local = 0, n_remote = 0;
  uint64_t local_edges = 0, remote_edges = 0;  // column ids per kind
  // local-only K1 form: 0 by the plan's shape, 1 warp-window, 2 group (8 rows
  // in flight per group), 3 group (4 rows in flight) — mgg_dplan_set_k1_form
  uint32_t k1_form = 0;
  int2* lmeta = nullptr;
  uint32_t* lcols = nullptr;
  int2* rmeta = nullptr;
  uint32_t* rcols = nullptr;
  uint64_t num_warps = 0, num_local_warps = 0;
  uint32_t* halo_rows = nullptr;   // distinct packed remote rows
  uint64_t halo_len = 0;
  uint32_t* rcols_halo = nullptr;  // remote columns -> halo rows
  // dynamic work queue of the pair kernel (aggregate.cu for_each_ticket):
  // 16 shard counters + a retire counter, 128 B apart, kSchedBytes; zero
  // between launches (the last warp to retire resets them)
  uint32_t* sched = nullptr;
  // kernels launched by the plan's latest K1 (';'-separated, demangled;
  // mgg_dplan_k1_kernels) — the bench labels its roofline with them
  mutable std::string k1_names;
  // geometry of the plan's latest K1 launch (mgg_dplan_k1_launch_info)
  mutable uint32_t last_grid = 0, last_threads = 0, last_resident = 0, last_sms = 0;
};

namespace mgg::dev {

/// Switch to the part's device; returns its stream.
cudaStream_t enter(mgg_ctx* ctx, uint32_t part);
void count_launch(mgg_ctx* ctx, uint64_t n = 1);

// launchers (aggregate.cu / dense.cu)
// Device event trace of a K1 launch (mgg_trace): 16-B records + counter.
struct TraceSink {
  void* events;
  void* count;
  uint32_t capacity, warp_limit;
};
// pull_dst (halo mode, the local pass): also copy the plan's distinct remote
// rows into pull_dst — fused into the local pass when its kernel is a group
// form, else by the pull kernel on `st` first.
void launch_aggregate(mgg_ctx* ctx, const mgg_dplan* p, const mgg_store* in,
                      mgg_store* out, int relu_in, int phase, const float* halo,
                      cudaStream_t st, const TraceSink* trace = nullptr,
                      float* pull_dst = nullptr);
int halo_fuse_mode();
void launch_strip_owner(uint32_t* cols, uint64_t n, cudaStream_t st);
void launch_halo_pull(const mgg_dplan* p, const mgg_store* in, float* halo, cudaStream_t st);
void run_aggregate(mgg_ctx* ctx, const mgg_dplan* plan, const mgg_store* in, mgg_store* out,
                   const mgg_agg_opts* o, cudaStream_t st);
// row_scale (optional): per-row multiplier of the part's rows (normalised GCN)
void launch_rows_init(const float* in, float* out, uint64_t rows, uint32_t pitch,
                      float scale, int relu_in, float* copy, cudaStream_t st,
                      const float* row_scale = nullptr);
void launch_dense(const float* in, uint32_t in_pitch, uint32_t k, uint64_t rows,
                  const float* w, const float* bias, const float* pre_bias,
                  uint32_t m, uint32_t pre, uint32_t act, float* out,
                  uint32_t out_pitch, float* out2, float out2_scale,
                  cudaStream_t st, const float* row_scale = nullptr);
void launch_softmax(const float* in, float* out, uint64_t rows, uint32_t pitch,
                    uint32_t m, cudaStream_t st, const float* row_scale = nullptr);
bool gemm_tc_supported(uint32_t k, uint32_t m);
bool gemm_tc_chain_supported(uint32_t k, uint32_t m1, uint32_t m);
void launch_dense_tc_chain(const float* in, uint32_t in_pitch, uint32_t k, uint64_t rows,
                           const float* wt1, const float* bias1, uint32_t m1,
                           const float* pre_bias, uint32_t pre, const float* wt2,
                           uint32_t m, float* out, uint32_t out_pitch, float* out2,
                           float out2_scale, cudaStream_t st);
const float* gemm_tc_prepare(mgg_dbuf* w, uint32_t k, uint32_t m, cudaStream_t st);
void launch_dense_tc(const float* in, uint32_t in_pitch, uint32_t k, uint64_t rows,
                     const float* wt, const float* bias, const float* pre_bias, uint32_t m,
                     uint32_t pre, uint32_t act, float* out, uint32_t out_pitch, float* out2,
                     float out2_scale, cudaStream_t st, const float* row_scale = nullptr);
/// Managed shards of `s` back to their home (see mgg_store_rehome).
void rehome(mgg_store* s, cudaStream_t st);
void launch_barrier(unsigned* const* flag_shards_dev, unsigned* own, uint32_t me,
                    uint32_t num_parts, cudaStream_t st);

}  // namespace mgg::dev
