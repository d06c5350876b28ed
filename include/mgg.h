/*
 * mgg.h — C-ABI of the B200-native MGG hot path (libmgg.so).
 *
 * Plain C types only: pointers, sizes, status codes. No exceptions, no torch
 * types. Every call returns an int status (0 OK, 1 INPUT, 2 PARSE, 3 CONFIG,
 * 4 INTEGRITY, 5 CUDA — the reference's exception taxonomy,
 * R:proj/include/pipeshard/errors.hpp:26-59, plus CUDA) and mgg_last_error()
 * returns the thread-local message of the last failure.
 *
 * Two layers:
 *
 *  A. The thin CUDA layer ("device runtime"): contexts, symmetric
 *     peer-mapped embedding stores, device plans, and the kernels — K1
 *     pipelined aggregation, K2 Update GEMM, K3 cross-GPU barrier. The C++
 *     host engine (include/mgg/engine.hpp) drives the GPU only through these.
 *     Together they replace the reference's execution model
 *     `simulate(plan, hw, dim, mode)` (R:proj/include/pipeshard/sim.hpp:91-93)
 *     and the per-GPU loop of `multi_gpu_run` (R:proj/src/sim.cpp:597-624).
 *
 *  B. Host facade for non-C++ callers (Python/ctypes, cgo, JNI): graph
 *     ingestion, the Alg. 1 split, the neighbor-partition builder, the cost
 *     model, the tuner, and the GCN/GIN engine. Each entry cites the
 *     reference interface it stands in for.
 *
 * Ownership: handles are library-owned (free with the matching *_destroy);
 * host arrays are caller-owned and only read/written during the call.
 * Threading: a context and everything created from it must be driven by one
 * host thread at a time; distinct contexts are independent.
 */
#ifndef MGG_H_
#define MGG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MGG_OK = 0,
  MGG_E_INPUT = 1,
  MGG_E_PARSE = 2,
  MGG_E_CONFIG = 3,
  MGG_E_INTEGRITY = 4,
  MGG_E_CUDA = 5
};

const char* mgg_last_error(void);
const char* mgg_version(void);
/* 1 if a CUDA device is visible, 0 otherwise (never fails). */
int mgg_cuda_available(void);
/* Number of visible CUDA devices (0 when none; never fails). */
int mgg_device_count(void);
/* Frees memory the library returned (JSON strings, CSV). */
void mgg_free(void* p);

/* ======================================================================= */
/* A. device runtime                                                        */
/* ======================================================================= */

typedef struct mgg_ctx mgg_ctx;
typedef struct mgg_store mgg_store;
typedef struct mgg_dplan mgg_dplan;
typedef struct mgg_dbuf mgg_dbuf;

/* A context spans `num_parts` logical partitions (the reference's "GPUs",
 * R:proj/src/sim.cpp:609). part_device[p] >= 0: this process drives part p on
 * that CUDA device (several parts may share one device — the "logical
 * partitions" configuration); -1: part p is driven by another process and its
 * memory is imported with mgg_store_ipc_import. At most 16 parts. */
int mgg_ctx_create(uint32_t num_parts, const int32_t* part_device, mgg_ctx** out);
int mgg_ctx_destroy(mgg_ctx* ctx);
/* Waits for all work this process queued on every local part. */
int mgg_ctx_synchronize(mgg_ctx* ctx);
/* Parts sharing a device each have their own stream (logical partitions run
 * concurrently; MGG_PART_STREAMS=0 reverts to one stream per device). This
 * orders every part's stream after every other's current tail; a no-op when
 * the parts of a device share a stream. */
int mgg_ctx_join(mgg_ctx* ctx);

/* Symmetric embedding store — the paper's NVSHMEM "shared" NE space
 * (R:PAPER.md:333-345) as per-part shards: part p holds global rows
 * [part_lb[p], part_lb[p+1]) (follow_split ranges,
 * R:proj/src/placement.cpp:96-103), `dim` fp32 columns at a pitch rounded up
 * to 4 floats (16-B rows for 128-bit loads). Padding is zero and stays zero.
 * Local shards are allocated here; remote shards are imported. */
int mgg_store_create(mgg_ctx* ctx, const uint64_t* part_lb, uint32_t dim,
                     mgg_store** out);
int mgg_store_destroy(mgg_store* s);
int mgg_store_info(const mgg_store* s, uint32_t* dim, uint32_t* pitch);
/* Layout of a store's shards: *symmetric = 1 when every part's shard lives
 * in ONE virtual range reserved with the CUDA VMM API (cuMemAddressReserve +
 * one cuMemCreate per part on its device, mapped for every local device):
 * part p at base + p * stride, so kernels address a peer's rows
 * arithmetically. Used for single-process contexts whose shards are device
 * memory (MGG_VMM=0 disables it); stores of multi-process contexts are one
 * allocation per shard plus CUDA IPC imports (*symmetric = 0). */
int mgg_store_layout(const mgg_store* s, int* symmetric, uint64_t* stride);
/* Cross-process symmetric stores (opt-in, MGG_VMM_IPC=1; *symmetric = 2 from
 * mgg_store_layout): every process reserves the same range layout, allocates
 * its local shard with a POSIX-fd-exportable VMM handle, and maps each peer's
 * shard at base + q * stride from the fd the peer exported (passed between
 * processes by the caller, e.g. SCM_RIGHTS over a Unix socket). The fd
 * returned by export is owned by the caller; import does not keep the fd. */
int mgg_store_vmm_export(const mgg_store* s, uint32_t part, int* fd);
int mgg_store_vmm_import(mgg_store* s, uint32_t part, int fd);
/* Where a local part's shards live (stores created after the call):
 *  MGG_MEM_DEVICE (0)       cudaMalloc on the part's device (default);
 *  MGG_MEM_HOST_MAPPED (1)  pinned host memory mapped into the device: a slow
 *      "peer" — every row read crosses PCIe with microsecond latency; measures
 *      remote-latency hiding (R:PAPER.md:405-419) on a one-GPU box;
 *  MGG_MEM_MANAGED (2)      cudaMallocManaged, home = the part's device: a
 *      reader on another device faults the pages it touches over — the
 *      reference's paged_remote baseline (R:proj/src/sim.cpp:503-518,
 *      571-595) on real multi-GPU hardware;
 *  MGG_MEM_MANAGED_HOST (3) cudaMallocManaged, home = host memory: the same
 *      page-fault-driven remote fetch on one GPU (pages migrate over PCIe).
 * Non-device shards cannot be IPC-exported. */
enum { MGG_MEM_DEVICE = 0, MGG_MEM_HOST_MAPPED = 1, MGG_MEM_MANAGED = 2,
       MGG_MEM_MANAGED_HOST = 3 };
int mgg_ctx_set_shard_memory(mgg_ctx* ctx, uint32_t part, int kind);
/* Prefetches the store's managed shards back to their home (every paged
 * measurement starts cold; mgg_time_aggregate does this before each timed
 * rep, outside the timed window). No-op for device / host-mapped shards. */
int mgg_store_rehome(mgg_store* s);
/* CUDA IPC handle (64 bytes) of a local shard / import a peer's shard. */
int mgg_store_ipc_export(const mgg_store* s, uint32_t part, void* handle64);
int mgg_store_ipc_import(mgg_store* s, uint32_t part, const void* handle64);
/* Copies global rows [row_begin, row_begin+row_count) between host (ld floats
 * per host row, ld >= dim) and whichever local shards hold them; rows of
 * remote parts are skipped. Asynchronous on the parts' streams when the host
 * memory is pinned; synchronize before reusing the host buffer. */
int mgg_store_upload(mgg_store* s, const float* host, uint64_t row_begin,
                     uint64_t row_count, uint32_t ld);
int mgg_store_download(const mgg_store* s, float* host, uint64_t row_begin,
                       uint64_t row_count, uint32_t ld);
/* Copy lanes. Every local part has a compute stream (lane 0, where all
 * kernels run) and two copy streams shared by the parts of a device, so host
 * transfers of one forward overlap the kernels of another:
 * MGG_LANE_H2D (1) and MGG_LANE_D2H (2). The _on variants enqueue the copy
 * (and its re-pitch kernel, when host rows are dense) on `lane`. */
enum { MGG_LANE_COMPUTE = 0, MGG_LANE_H2D = 1, MGG_LANE_D2H = 2 };
int mgg_store_upload_on(mgg_store* s, const float* host, uint64_t row_begin,
                        uint64_t row_count, uint32_t ld, int lane);
int mgg_store_download_on(const mgg_store* s, float* host, uint64_t row_begin,
                          uint64_t row_count, uint32_t ld, int lane);
/* Orders lane `to` after everything enqueued on lane `from` so far (device
 * side; the host does not block). */
int mgg_lane_fence(mgg_ctx* ctx, uint32_t part, int from, int to);
/* Host-waitable marks: record `slot` at the current tail of `lane`; wait
 * (blocking the calling thread) until the device reaches it. */
int mgg_lane_mark(mgg_ctx* ctx, uint32_t part, int lane, uint32_t slot);
int mgg_lane_wait_host(mgg_ctx* ctx, uint32_t part, uint32_t slot);
/* Device-side: lane `lane` waits until the device reaches mark `slot`. */
int mgg_lane_wait_mark(mgg_ctx* ctx, uint32_t part, int lane, uint32_t slot);
/* Device pointer of a shard as seen by this process (local or imported). */
int mgg_store_shard(const mgg_store* s, uint32_t part, void** dptr);

/* Small device buffers (weights, biases) on one local part's device. */
int mgg_dbuf_create(mgg_ctx* ctx, uint32_t part, const void* host, size_t bytes,
                    mgg_dbuf** out);
int mgg_dbuf_destroy(mgg_dbuf* b);
/* Device address of a buffer (for the probes below). */
void* mgg_dbuf_ptr(const mgg_dbuf* b);

/* Pinned host memory for zero-staging H2D/D2H. */
int mgg_host_alloc(size_t bytes, void** out);
int mgg_host_free(void* p);

/* Device form of one part's launch plan (FlatPlan, include/mgg/workload.hpp):
 * per kind, (target_row, begin) int32 pairs with a sentinel and one packed
 * column per neighbor ((owner << 28) | offset). Warps are implicit: warp w
 * owns partitions [w*dist, (w+1)*dist) of each kind (interleaved) or the
 * local groups then the remote groups (segregated); a CTA is wpb warps
 * (R:proj/src/workload.cpp:103-172). */
typedef struct {
  uint32_t part;
  uint32_t ps, dist, wpb;
  uint32_t mapping;     /* 0 interleaved, 1 segregated */
  uint32_t granularity; /* 0 partitioned, 1 whole_list */
  uint64_t rows;        /* chunk rows (target rows of this part) */
  uint64_t n_local, n_remote;            /* partitions per kind */
  const int32_t* local_meta;  /* 2*(n_local+1) */
  const uint32_t* local_cols; uint64_t local_cols_len;
  const int32_t* remote_meta; /* 2*(n_remote+1) */
  const uint32_t* remote_cols; uint64_t remote_cols_len;
  /* optional deduplicated remote fetch (HaloPlan, include/mgg/workload.hpp):
   * halo_len distinct packed remote rows, and remote_cols re-pointed at them
   * (remote_cols_len entries); NULL/0 when unused */
  const uint32_t* halo_rows; uint64_t halo_len;
  const uint32_t* remote_halo_cols;
} mgg_plan_desc;

int mgg_dplan_upload(mgg_ctx* ctx, const mgg_plan_desc* desc, mgg_dplan** out);
int mgg_dplan_destroy(mgg_dplan* p);

/* K1 — pipelined aggregation over one part's plan:
 *   out[t] += Σ_{u in partitions of t} f(in[u])        f = ReLU if relu_in
 * Local rows come from the part's own shard with coalesced 128-bit loads;
 * remote rows from peer shards (NVLink/NVSwitch peer-mapped pointers) are
 * issued before the paired local partition is reduced and consumed after it
 * — the async discipline of R:proj/src/sim.cpp:102-125 / R:PAPER.md:406-419.
 * Partials of one target combine in registers while consecutive partitions
 * of a warp share it, then with fp32 vector reductions into `out` (the
 * paper's "shuffling and atomics", R:PAPER.md:309). `out` must hold the self
 * term already (mgg_rows_init). */
typedef struct {
  int relu_in;
  int phase; /* 0 all, 1 local partitions only, 2 remote only (phase-split
                measurement, R:proj/src/sim.cpp:127-142); 3 = local only
                through the fine-fetch pair kernel itself (its own local
                leg: T_pipe vs T_local + T_remote of one kernel) */
  const float* halo; /* non-NULL: remote partitions read this part's halo
                        buffer instead of peers (local pass, then remote pass) */
  int halo_pull;     /* with halo: refill it first (mgg_halo_pull) on the
                        part's aux stream, overlapped with the local pass */
} mgg_agg_opts;
int mgg_aggregate(mgg_ctx* ctx, const mgg_dplan* plan, const mgg_store* in,
                  mgg_store* out, const mgg_agg_opts* opts);

/* Device event trace of K1 — the reference's per-warp trace
 * (TraceEvent, R:proj/include/pipeshard/sim.hpp:71; CSV
 * R:proj/src/sim.cpp:626-635) recorded by the real kernel: per logical warp
 * and pair, LR (remote get: issue -> staged rows landed), LL (local
 * partition load + reduce) and AC (accumulate of the remote partition)
 * begin/end stamps from %globaltimer, plus the SM id. Only logical warps
 * < warp_limit record; at most `capacity` events are kept. */
typedef struct mgg_trace mgg_trace;
int mgg_trace_create(mgg_ctx* ctx, uint32_t part, uint64_t capacity, uint32_t warp_limit,
                     mgg_trace** out);
int mgg_trace_destroy(mgg_trace* t);
/* One traced K1 launch (always the fine-grained pipelined kernel; no
 * ReLU-on-load; rows <= 128 floats). Same result as mgg_aggregate. */
int mgg_aggregate_traced(mgg_ctx* ctx, const mgg_dplan* plan, const mgg_store* in,
                         mgg_store* out, const mgg_agg_opts* opts, mgg_trace* trace);
/* Waits for the part's stream, then copies up to `cap` events as 4 x u64
 * {cycle, sm, warp, stage*2 + begin} (stage 0 LR, 1 LL, 2 AC; cycle = SM
 * clocks since the earliest recorded event). *n = events returned,
 * *emitted = events the kernel tried to record (> capacity: truncated). */
int mgg_trace_read(mgg_trace* t, uint64_t* events, uint64_t cap, uint64_t* n,
                   uint64_t* emitted);

/* Deduplicated remote fetch: copy the plan's distinct remote rows of `in`
 * from the peer shards (NVLink) into `halo` (halo_len x pitch floats, device
 * memory of the plan's part), one coalesced pass; the next mgg_aggregate
 * with opts.halo reads them locally. */
int mgg_halo_pull(mgg_ctx* ctx, const mgg_dplan* plan, const mgg_store* in, float* halo);
int mgg_dplan_halo_len(const mgg_dplan* plan, uint64_t* halo_len);
/* Geometry of the plan's latest K1 launch: info[4] = {grid CTAs, threads per
 * CTA, resident CTAs per SM (cudaOccupancyMaxActiveBlocksPerMultiprocessor),
 * SMs of the device}. */
int mgg_dplan_k1_launch_info(const mgg_dplan* plan, uint32_t* info);
/* Names of the kernels the plan's latest K1 (mgg_aggregate / _traced /
 * mgg_time_aggregate) launched, demangled, ';'-separated (halo mode: the
 * local pass then the remote pass), NUL-terminated into buf[cap]. */
int mgg_dplan_k1_kernels(const mgg_dplan* plan, char* buf, size_t cap);
/* Local-only K1 form for this plan's launches (single-part and halo passes):
 * 0 = by the plan's shape (default), 1 = warp-window, 2 = group-per-partition
 * with 8 rows in flight per group, 3 = the same with 4. Same partitions and
 * sums in every form; the tuner's post-pass picks among them. */
int mgg_dplan_set_k1_form(mgg_dplan* plan, uint32_t form);

/* out[r] = scale * f(in[r]) for the part's own rows (self term / copies).
 * f: 0 identity, 1 ReLU. */
int mgg_rows_init(mgg_ctx* ctx, uint32_t part, const mgg_store* in,
                  mgg_store* out, float scale, int relu_in);
/* mgg_rows_init that also writes copy[r] = f(in[r]) (same width; null = no
 * copy): the activated layer input, which the next mgg_aggregate then
 * gathers with relu_in = 0 instead of applying f once per edge. */
/* rows_init_copy with an optional per-row multiplier (the part's rows). */
int mgg_rows_init_rs(mgg_ctx* ctx, uint32_t part, const mgg_store* in, mgg_store* out,
                     float scale, int relu_in, mgg_store* copy, const mgg_dbuf* row_scale);
/* rows_softmax of row_scale[r] * in[r]. */
int mgg_rows_softmax_rs(mgg_ctx* ctx, uint32_t part, const mgg_store* in, mgg_store* out,
                        const mgg_dbuf* row_scale);
int mgg_rows_init_copy(mgg_ctx* ctx, uint32_t part, const mgg_store* in,
                       mgg_store* out, float scale, int relu_in, mgg_store* copy);

/* Row softmax over the `dim` columns of the part's rows (in place allowed). */
int mgg_rows_softmax(mgg_ctx* ctx, uint32_t part, const mgg_store* in,
                     mgg_store* out);

/* K2 — Update GEMM on one part's rows:
 *   x   = pre(in[r])          pre: 0 none, 1 ReLU, 2 ReLU(x + pre_bias)
 *   y   = x · W (+ bias)      W: k x m row-major fp32, k = in dim, m = out dim
 *   out = act(y)              act: 0 none, 1 ReLU, 2 row softmax
 *   out2 (optional) = out2_scale * y   (accumulator seeding)
 * fp32 accumulate. */
typedef struct {
  const mgg_dbuf* w;
  const mgg_dbuf* bias;     /* m floats or NULL */
  const mgg_dbuf* pre_bias; /* k floats, for pre == 2 */
  uint32_t pre;
  uint32_t act;
  float out2_scale;
  const mgg_dbuf* row_scale; /* optional: per-row multiplier of the product
                                (the part's rows; normalised GCN) */
} mgg_dense_desc;
int mgg_dense(mgg_ctx* ctx, uint32_t part, const mgg_store* in,
              const mgg_dense_desc* d, mgg_store* out, mgg_store* out2);
/* Chained Update (the GIN layer boundary, Linear2 -> ReLU -> next Linear1):
 *   O    = ReLU(pre(in)·W1 + b1)            (m1 columns, kept in TMEM)
 *   out  = O·W2,  out2 = out2_scale·O·W2    (d2: W2, no bias, pre = 1)
 * one tcgen05 kernel; O never touches HBM. d1->act must be 0. */
int mgg_dense_chain(mgg_ctx* ctx, uint32_t part, const mgg_store* in,
                    const mgg_dense_desc* d1, uint32_t m1, const mgg_dense_desc* d2,
                    mgg_store* out, mgg_store* out2);
/* 1 when mgg_dense_chain handles in-width k -> m1 -> m. */
int mgg_dense_chain_supported(uint32_t k, uint32_t m1, uint32_t m);

/* K3 — cross-GPU layer barrier (R:PAPER.md:258 "result synchronization at
 * the end"; barrier_cycles, R:proj/src/sim.cpp:620), never a host round trip:
 *  - every part in this process (one device or several): each part's stream
 *    waits for every other part's tail through events (cudaStreamWaitEvent
 *    orders streams across devices; capturable into one CUDA graph);
 *  - parts in other processes: the K3 kernel — release/acquire flags at
 *    system scope in the peer-mapped `flags` store (one row per part, at
 *    least num_parts + 1 columns: arrivals + the part's device-side epoch
 *    counter, so captured barriers advance on every replay).
 * MGG_BARRIER=k3 forces the kernel for same-process parts too (validation). */
int mgg_barrier(mgg_ctx* ctx, mgg_store* flags);

/* Timing with CUDA events on the part's stream around `reps` launches of
 * K1; returns the median ns (backs the tuner's SimulateFn,
 * R:proj/include/pipeshard/tuner.hpp:28-30). */
int mgg_time_aggregate(mgg_ctx* ctx, const mgg_dplan* plan, const mgg_store* in,
                       mgg_store* out, const mgg_agg_opts* opts, uint32_t reps,
                       uint64_t* median_ns);

/* K5 — hardware probes (re-fit the b200 cost-model profile, roofline
 * denominators): sustained gather GB/s of rows table[idx[i]] (device
 * pointers; pitch floats per row) and dependent-load latency (ns) of a
 * random cycle `next` (device pointer) — local HBM, L2 or a peer GPU. */
int mgg_probe_gather(mgg_ctx* ctx, uint32_t part, const float* table, uint32_t pitch,
                     const uint32_t* idx, uint64_t n, uint32_t reps, double* gbps);
int mgg_probe_chase(mgg_ctx* ctx, uint32_t part, const uint32_t* next, uint32_t steps,
                    double* ns_per_load);

/* CUDA graphs: capture the calls made between begin and end on the streams
 * of the context's local parts (one or several devices) — the aux streams
 * join back through events — into an executable graph, then replay it with
 * one launch. Parts driven by other processes are not captured; K3 barriers
 * towards them are captured flag kernels whose epoch lives on the device, so
 * every process replays its own graph and the barriers still pair up.
 * Replays count their kernels in mgg_ctx_launch_count. */
typedef struct mgg_exec mgg_exec;
int mgg_capture_begin(mgg_ctx* ctx);
int mgg_capture_end(mgg_ctx* ctx, mgg_exec** out);
int mgg_exec_launch(mgg_ctx* ctx, const mgg_exec* g);
int mgg_exec_destroy(mgg_exec* g);

/* Number of kernels this library launched since the context was created. */
uint64_t mgg_ctx_launch_count(const mgg_ctx* ctx);

/* CUDA events on a part's stream, addressed by slot (created on first use):
 * the only clock the benchmark and tuner trust (device time, never host). */
int mgg_event_record(mgg_ctx* ctx, uint32_t part, uint32_t slot);
/* Waits for slot b, then *ms = elapsed(a -> b). */
int mgg_event_elapsed(mgg_ctx* ctx, uint32_t part, uint32_t a, uint32_t b, float* ms);
/* ms between slot a of part_a and slot b of part_b (both parts on the same
 * device: their streams share the device clock). */
int mgg_event_elapsed_between(mgg_ctx* ctx, uint32_t part_a, uint32_t a, uint32_t part_b,
                              uint32_t b, float* ms);

/* ======================================================================= */
/* B. host facade                                                           */
/* ======================================================================= */

typedef struct mgg_graph mgg_graph;
typedef struct mgg_flat_plan mgg_flat_plan;
typedef struct mgg_engine mgg_engine;

/* Graph ingestion — R:proj/include/pipeshard/graph.hpp:59-85. */
int mgg_graph_from_csr(uint64_t num_nodes, uint64_t num_edges,
                       const uint64_t* row_ptr, const uint64_t* col_idx,
                       mgg_graph** out); /* validate_csr */
int mgg_graph_from_edges(uint64_t num_nodes, uint64_t num_edges,
                         const uint64_t* src, const uint64_t* dst,
                         mgg_graph** out); /* from_edges */
/* kind 0 uniform, 1 powerlaw (gen_synthetic, bit-identical to the
 * reference); 2 rmat (a=0.57,b=0.19,c=0.19; `avg_degree` = edge count). */
int mgg_graph_generate(int kind, uint64_t num_nodes, double avg_degree,
                       uint64_t seed, mgg_graph** out);
int mgg_graph_load_edge_list(const char* path, mgg_graph** out);
int mgg_graph_load_csr(const char* path, mgg_graph** out);
int mgg_graph_save_csr(const mgg_graph* g, const char* path);
int mgg_graph_dims(const mgg_graph* g, uint64_t* num_nodes, uint64_t* num_edges);
const uint64_t* mgg_graph_row_ptr(const mgg_graph* g);
const uint64_t* mgg_graph_col_idx(const mgg_graph* g);
int mgg_graph_destroy(mgg_graph* g);

/* Alg. 1 — split_by_edges (R:proj/src/placement.cpp:44): num_gpus-1 points. */
int mgg_split_by_edges(const mgg_graph* g, uint32_t num_gpus, uint64_t* split_points);
/* plan_ne_placement (R:proj/src/placement.cpp:73); mode 0 equal_nodes,
 * 1 follow_split; ranges = 2*num_gpus (lb, ub). */
int mgg_plan_ne_placement(const mgg_graph* g, uint32_t num_gpus, int mode,
                          uint64_t dim, uint64_t* ranges);
/* translate (R:proj/src/placement.cpp:108) for `count` ids. */
int mgg_translate(const mgg_graph* g, uint32_t num_gpus, int mode, uint64_t count,
                  const uint64_t* ids, uint32_t* gpu, uint64_t* offset);
/* memory_footprint (R:proj/src/placement.cpp:121): per_gpu = 2*num_gpus
 * (ne_bytes, gp_bytes). */
int mgg_memory_footprint(const mgg_graph* g, uint32_t num_gpus, int mode,
                         uint64_t dim, uint64_t device_mem_bytes,
                         uint64_t* per_gpu, int* fits);

/* Neighbor-partition builder: split_local_remote + build_launch_plan
 * (R:proj/src/workload.cpp:26-211) for one gpu, in device form.
 * mapping 0 interleaved 1 segregated; granularity 0 partitioned 1 whole_list. */
int mgg_flat_plan_build(const mgg_graph* g, uint32_t num_gpus, int placement_mode,
                        uint32_t gpu, uint32_t ps, uint32_t dist, uint32_t wpb,
                        uint64_t dim, int mapping, int granularity,
                        mgg_flat_plan** out);
/* info[10] = {n_local, n_remote, local_cols, remote_cols, num_warps,
 *             num_blocks, first_target, rows, smem_bytes_per_block,
 *             launch_smem_bytes} */
int mgg_flat_plan_info(const mgg_flat_plan* p, uint64_t* info);
const int32_t* mgg_flat_plan_meta(const mgg_flat_plan* p, int kind);
const uint32_t* mgg_flat_plan_cols(const mgg_flat_plan* p, int kind);
/* Canonical reference JSON of the expanded plan (to_json(KernelLaunchPlan),
 * R:proj/src/workload.cpp:276-305). Free with mgg_free. */
int mgg_flat_plan_json(const mgg_flat_plan* p, char** json);
/* Expanded warp/task view: warp_off[num_warps+1], task_kind[], task_idx[]. */
int mgg_flat_plan_tasks(const mgg_flat_plan* p, uint64_t* warp_off,
                        uint8_t* task_kind, uint32_t* task_idx);
int mgg_flat_plan_destroy(mgg_flat_plan* p);

/* Cost model — R:proj/src/costmodel.cpp:27-77. */
uint64_t mgg_wpw(uint32_t ps, uint32_t dist, uint32_t wpb, uint64_t dim);
uint64_t mgg_smem(uint32_t ps, uint32_t dist, uint32_t wpb, uint64_t dim);
int mgg_launch_geometry(uint64_t n_local, uint64_t n_remote, uint32_t ps,
                        uint32_t dist, uint32_t wpb, const char* profile,
                        uint64_t* num_warps_blocks, double* blocks_per_sm);
/* Violations joined as "name;name;" into buf; returns their count (>= 0) or
 * a negative status. */
int mgg_validate(uint32_t ps, uint32_t dist, uint32_t wpb, uint64_t dim,
                 uint32_t num_sms, uint32_t max_warps, uint64_t smem_per_sm,
                 char* buf, size_t buflen);
/* resolve_profile (R:proj/src/costmodel.cpp:118): JSON text, mgg_free it. */
int mgg_profile_json(const char* name_or_path, char** json);

/* Tuner — R:proj/src/tuner.cpp:129-243. The callback returns the latency of
 * one configuration; a non-zero *err from it aborts the search with that
 * configuration named in the error. trace: 4 u64 per entry (ps, dist, wpb,
 * cycles), capacity `cap` entries, count in *n; best[4]. */
typedef uint64_t (*mgg_measure_fn)(uint32_t ps, uint32_t dist, uint32_t wpb,
                                   void* user, int* err);
int mgg_optimize(mgg_measure_fn fn, void* user, uint32_t num_sms,
                 uint32_t max_warps, uint64_t smem_per_sm, uint64_t dim,
                 int retreat_value_rank, uint64_t max_evaluations,
                 uint64_t* trace, size_t cap, size_t* n, uint64_t* best);
int mgg_exhaustive(mgg_measure_fn fn, void* user, uint32_t num_sms,
                   uint32_t max_warps, uint64_t smem_per_sm, uint64_t dim,
                   uint64_t* table, size_t cap, size_t* n);

/* GCN / GIN engine — the multi-GPU forward driver (the shape of
 * multi_gpu_run, R:proj/src/sim.cpp:597-624, with the layer arithmetic of
 * R:PAPER.md:504-517 that the reference leaves out). */
typedef struct {
  uint32_t kind;       /* 0 GCN (R:PAPER.md:504-508), 1 GIN (511-517) */
  uint32_t layers;     /* GCN: 2; GIN: any >= 1 */
  uint32_t in_dim;
  uint32_t hidden;     /* GCN hidden width; GIN MLP hidden width */
  uint32_t out_dim;    /* classes */
  float eps;           /* GIN epsilon */
  /* Weights, fp32 row-major, packed layer after layer:
   *  GCN: w1 = [W^1 (in x hidden), W^2 (hidden x out)]; b1/w2/b2 unused.
   *  GIN layer l (d_l -> d_{l+1}, d_0 = in, d_L = out, inner = hidden):
   *    w1 += d_l x hidden, b1 += hidden, w2 += hidden x d_{l+1},
   *    b2 += d_{l+1}. */
  const float* w1;
  const float* b1;
  const float* w2;
  const float* b2;
  uint32_t norm;       /* GCN: 1 = symmetric normalisation D^-1/2 (A+I) D^-1/2
                          with d_v = |N(v)| + 1 (oracle norm=1); 0 = the
                          paper's plain sum over N(v) ∪ {v} */
} mgg_model_desc;

/* Builds split (Alg. 1), follow_split placement, per-part plans, stores and
 * weights for the parts this process drives (part_device as in
 * mgg_ctx_create). */
int mgg_engine_create(const mgg_graph* g, uint32_t num_parts,
                      const int32_t* part_device, uint32_t ps, uint32_t dist,
                      uint32_t wpb, const mgg_model_desc* model,
                      mgg_engine** out);
int mgg_engine_destroy(mgg_engine* e);
/* IPC blob of every shard of local part `part` (stores + barrier flags). */
int mgg_engine_ipc_export(const mgg_engine* e, uint32_t part, void* blob,
                          size_t* len);
int mgg_engine_ipc_import(mgg_engine* e, uint32_t part, const void* blob,
                          size_t len);
/* Cross-process symmetric VMM stores (MGG_VMM_IPC=1, see mgg_store_vmm_export):
 * *on = 1 when this engine's stores are fd-exportable VMM ranges; export
 * writes one POSIX fd per store of local part `part` (caller-owned, count in
 * *count; fds may be NULL to query), import maps a peer's from its fds. */
int mgg_engine_vmm_ipc(const mgg_engine* e, int* on);
int mgg_engine_vmm_export(const mgg_engine* e, uint32_t part, int* fds, size_t* count);
int mgg_engine_vmm_import(mgg_engine* e, uint32_t part, const int* fds, size_t count);
/* Remote fetch: 0 auto (halo when it moves >= 2x fewer bytes), 1 fine
 * (per-edge peer reads in K1, the paper's design), 2 halo (deduplicated
 * pull, then local reads). Re-plans. */
int mgg_engine_set_remote_fetch(mgg_engine* e, int mode);
/* Ablation mappings (R:proj/src/sim.cpp:571-595): mapping 1 = segregated
 * (no_interleave), granularity 1 = whole_list (no_np). Re-plans. */
int mgg_engine_set_mapping(mgg_engine* e, int mapping, int granularity);
/* remote_partition_bytes (R:proj/src/sim.cpp:503-518): fine-grained or paged. */
uint64_t mgg_remote_partition_bytes(uint64_t part_size, uint64_t dim, int paged,
                                    uint64_t page_bytes);
/* Re-plan with a new (ps, dist, wpb) (tuner hook). */
int mgg_engine_set_config(mgg_engine* e, uint32_t ps, uint32_t dist, uint32_t wpb);
/* x: num_nodes x in_dim host rows (only this process's rows are read). */
int mgg_engine_set_input(mgg_engine* e, const float* x);
/* Device-resident forward (async). The layer program of this process's parts
 * is captured once into a CUDA graph and replayed (re-captured after
 * re-planning); mgg_engine_set_graphs(e, 0) disables it. With parts in other
 * processes every process must call it the same number of times. */
int mgg_engine_forward(mgg_engine* e);
int mgg_engine_set_graphs(mgg_engine* e, int on);
/* Local-only K1 form of every plan of the engine (mgg_dplan_set_k1_form). */
int mgg_engine_set_k1_form(mgg_engine* e, uint32_t form);
/* z: num_nodes x out_dim; only this process's rows are written. */
int mgg_engine_get_output(mgg_engine* e, float* z);
/* End to end: H2D x, forward, D2H z (synchronous). */
int mgg_engine_forward_host(mgg_engine* e, const float* x, float* z);
/* Streamed end to end: enqueue one forward whose H2D of x runs on the copy
 * lane as soon as the previous forward has consumed its input, and whose
 * D2H of z runs on the other copy lane, so consecutive forwards overlap
 * their PCIe transfers with each other's kernels. Returns immediately with a
 * ticket; x must stay valid and z untouched until mgg_engine_wait(ticket).
 * At most 32 forwards may be outstanding (the call then waits for the
 * oldest). forward_host == submit + wait. */
int mgg_engine_submit_host(mgg_engine* e, const float* x, float* z, uint64_t* ticket);
int mgg_engine_wait(mgg_engine* e, uint64_t ticket);
/* Layer-k intermediate (post-aggregation accumulator) rows, for parity. */
int mgg_engine_get_hidden(mgg_engine* e, uint32_t which, float* rows, uint32_t* width);
/* Pre-softmax logits of the last forward (N x out_dim): the engine's head
 * GEMM re-run on the device without the softmax epilogue. */
int mgg_engine_get_logits(mgg_engine* e, float* rows);
/* Standalone aggregation through the engine's plans (K1 over every local
 * part): out = self_scale*f(x) + Σ f(x_u); x/out num_nodes x dim host rows. */
int mgg_engine_aggregate_host(mgg_engine* e, const float* x, uint32_t dim,
                              float self_scale, int relu_in, float* out);
/* The same restricted to one kind of partition: phase 1 = local only, 2 =
 * remote only (the phase-separated ablation's halves; their sums add up to
 * the full aggregation). */
int mgg_engine_aggregate_phase_host(mgg_engine* e, const float* x, uint32_t dim,
                                    float self_scale, int relu_in, int phase, float* out);
/* Median-of-reps K1 latency (ns) at aggregation width `dim` for the current
 * config, max over local parts — the tuner's SimulateFn. */
int mgg_engine_time_aggregate(mgg_engine* e, uint32_t dim, uint32_t reps,
                              int phase, uint64_t* median_ns);
/* The same per part: ns[num_parts] (0 for parts of other processes). */
int mgg_engine_time_aggregate_each(mgg_engine* e, uint32_t dim, uint32_t reps, int phase,
                                   uint64_t* ns);
/* Measured MultiGpuReport (R:proj/include/pipeshard/sim.hpp:115-123,
 * multi_gpu_run R:proj/src/sim.cpp:597-624): every local part's K1 at width
 * `dim` run concurrently, median of `reps`. summary[6] = {max_gpu_ns,
 * barrier_ns, total_ns (max + barrier), remote_bytes, max_alone_ns (max over
 * parts of each part's K1 with the device to itself: the per-GPU time when
 * logical parts share a device), devices}; per_part[num_parts x 9]
 * = {local (1/0), total_ns (concurrent), alone_ns, remote_bytes, local_bytes,
 * num_warps, num_blocks, active_sms, part}; per_part_f[num_parts x 2] =
 * {achieved_occupancy (occupancy calculator x grid), sm_utilization (SMs
 * given CTAs / SMs)}. */
int mgg_engine_measure_multi_gpu(mgg_engine* e, uint32_t dim, uint32_t reps,
                                 uint64_t* summary, uint64_t* per_part, double* per_part_f);
/* Shard placement of local part `part` (MGG_MEM_*); re-creates the engine's
 * stores (set the input again). Single-process engines only. */
int mgg_engine_set_shard_memory(mgg_engine* e, uint32_t part, int kind);
/* Device event trace of one K1 launch at width `dim` on every local part
 * (mgg_aggregate_traced), as the reference's multi-GPU trace CSV
 * (R:proj/tools/cli.cpp:144-155): "gpu,cycle,sm,warp,stage,event" rows,
 * stage LR/LL/AC, event begin/end, per part sorted by cycle. Free with
 * mgg_free. */
int mgg_engine_trace_csv(mgg_engine* e, uint32_t dim, uint64_t capacity, uint32_t warp_limit,
                         char** csv);
/* stats[10] = {local_parts_total, remote_parts_total, local_edges,
 * remote_edges, num_warps, num_blocks, kernel_launches, plan_build_ns,
 * halo_rows, halo_parts} */
int mgg_engine_stats(const mgg_engine* e, uint64_t* stats);
mgg_ctx* mgg_engine_ctx(mgg_engine* e);
/* mgg_dplan_k1_kernels of local part `part`'s plan (the K1 forms the
 * engine's latest aggregation of that part ran). */
int mgg_engine_k1_kernels(const mgg_engine* e, uint32_t part, char* buf, size_t cap);
/* Per-op device timing of subsequent forwards (events around every op of the
 * layer program on the first local part's stream; no host sync added). */
int mgg_engine_set_profiling(mgg_engine* e, int on);
/* Program size / per-op accumulated ms, op kind (0 dense, 1 init,
 * 2 aggregate, 3 barrier, 4 softmax, 5 dense_chain), op width (output columns) and the
 * number of profiled forwards. Arrays hold `cap` entries. */
int mgg_engine_profile(mgg_engine* e, double* op_ms, uint32_t* op_kind,
                       uint32_t* op_width, size_t cap, size_t* n_ops,
                       uint64_t* forwards);

#ifdef __cplusplus
}
#endif
#endif /* MGG_H_ */
