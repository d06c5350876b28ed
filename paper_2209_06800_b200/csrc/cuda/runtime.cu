// Device runtime: contexts, symmetric stores, device plans, K3 barrier and
// the C-ABI of layer A (include/mgg.h).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace mgg::dev {

thread_local std::string g_last_error;
std::string& last_error() { return g_last_error; }

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Status{MGG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

cudaStream_t enter(mgg_ctx* ctx, uint32_t part) {
  if (!ctx || part >= ctx->num_parts) throw Status{MGG_E_INPUT, "part out of range"};
  if (ctx->device[part] < 0)
    throw Status{MGG_E_INPUT, "part " + std::to_string(part) + " is not local"};
  MGG_CUDA(cudaSetDevice(ctx->device[part]));
  return ctx->stream[part];
}

void count_launch(mgg_ctx* ctx, uint64_t n) { ctx->launches += n; }

namespace {

// K3: announce this barrier's epoch to every part, then wait until every part
// announced it. The epoch lives on the device (own[n], this part's counter,
// advanced by each barrier launch of the part — they are stream-ordered), so
// a barrier captured into a CUDA graph still advances on every replay.
__global__ void barrier_kernel(unsigned* const* shards, unsigned* own, uint32_t me,
                               uint32_t n) {
  const uint32_t q = threadIdx.x;
  __threadfence_system();  // this GPU's prior kernels' writes before the flag
  const unsigned epoch = *reinterpret_cast<volatile unsigned*>(own + n) + 1;
  if (q < n) {
    unsigned* slot = shards[q] + me;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(slot), "r"(epoch) : "memory");
    unsigned seen;
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(seen) : "l"(own + q) : "memory");
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      // a peer that never arrives (crashed rank) fails the launch instead of
      // hanging the GPU: 60 s watchdog
      if (t - t0 > 60ull * 1000000000ull) __trap();
    } while (static_cast<int>(seen - epoch) < 0);
  }
  __syncwarp();
  if (q == 0) own[n] = epoch;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return MGG_OK;
  } catch (const Status& s) {
    g_last_error = s.msg;
    return s.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host out of memory";
    return MGG_E_INPUT;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MGG_E_INPUT;
  }
}

void refresh_tables(mgg_store* s) {
  mgg_ctx* ctx = s->ctx;
  for (uint32_t p = 0; p < ctx->num_parts; ++p) {
    if (ctx->device[p] < 0) continue;
    MGG_CUDA(cudaSetDevice(ctx->device[p]));
    std::vector<const float*> host(kMaxParts, nullptr);
    for (uint32_t q = 0; q < ctx->num_parts; ++q) host[q] = s->shard[q];
    if (!s->dtable[p]) {
      void* d = nullptr;
      MGG_CUDA(cudaMalloc(&d, kMaxParts * sizeof(float*)));
      s->dtable[p] = static_cast<const float**>(d);
    }
    // the table is read by kernels on the part's non-blocking streams, which
    // do not order behind a legacy-stream cudaMemcpy (a pageable H2D copy may
    // return before its DMA lands): copy on the part's stream and wait
    MGG_CUDA(cudaMemcpyAsync(s->dtable[p], host.data(), kMaxParts * sizeof(float*),
                             cudaMemcpyHostToDevice, ctx->stream[p]));
    MGG_CUDA(cudaStreamSynchronize(ctx->stream[p]));
  }
}

// Setup uploads are ordered on `st` (the consumer's stream); the caller
// synchronises `st` before the buffers are handed out.
template <class T>
T* upload_array(const T* host, size_t n, cudaStream_t st) {
  void* d = nullptr;
  const size_t bytes = std::max<size_t>(n * sizeof(T), 16);
  MGG_CUDA(cudaMalloc(&d, bytes));
  if (n) MGG_CUDA(cudaMemcpyAsync(d, host, n * sizeof(T), cudaMemcpyHostToDevice, st));
  return static_cast<T*>(d);
}

}  // namespace

// Managed shards back to their home (owner device or host), ordered on `st`
// (each part's own stream when null), and waited for when st is null.
void rehome(mgg_store* s, cudaStream_t st) {
  mgg_ctx* ctx = s->ctx;
  for (uint32_t p = 0; p < ctx->num_parts; ++p) {
    if (!s->owned[p] || (s->mem[p] != MGG_MEM_MANAGED && s->mem[p] != MGG_MEM_MANAGED_HOST))
      continue;
    MGG_CUDA(cudaSetDevice(ctx->device[p]));
    const int home = s->mem[p] == MGG_MEM_MANAGED ? ctx->device[p] : cudaCpuDeviceId;
    cudaStream_t q = st ? st : ctx->stream[p];
    MGG_CUDA(cudaMemPrefetchAsync(s->shard[p], s->bytes[p], home, q));
    if (!st) MGG_CUDA(cudaStreamSynchronize(q));
  }
}

void launch_barrier(unsigned* const* shards, unsigned* own, uint32_t me, uint32_t n,
                    cudaStream_t st) {
  barrier_kernel<<<1, 32, 0, st>>>(shards, own, me, n);
  MGG_CUDA(cudaGetLastError());
}

// K1 entry: fine-grained (one launch, remote rows read from peers in the
// pair loop), or halo mode — the deduplicated pull runs on the part's aux
// stream while the local partitions are reduced on the main stream, then the
// remote partitions are reduced from the local halo.
void run_aggregate(mgg_ctx* ctx, const mgg_dplan* plan, const mgg_store* in, mgg_store* out,
                   const mgg_agg_opts* o, cudaStream_t st) {
  const int relu = o ? o->relu_in : 0, phase = o ? o->phase : 0;
  const float* halo = o ? o->halo : nullptr;
  plan->k1_names.clear();
  if (!halo) {
    launch_aggregate(ctx, plan, in, out, relu, phase, nullptr, st);
    return;
  }
  if (!plan->rcols_halo) throw Status{MGG_E_INPUT, "aggregate: plan has no halo"};
  const uint32_t p = plan->part;
  const bool pull = o->halo_pull && phase != 1 && phase != 3;
  bool fuse = halo_fuse_mode() == 1;
  if (halo_fuse_mode() < 0)  // auto: the halo comes over a link slower than own HBM
    for (uint32_t q = 0; q < ctx->num_parts; ++q)
      if (q != p)
        fuse |= in->imported[q] || in->mem[q] != MGG_MEM_DEVICE ||
                (ctx->device[q] >= 0 && ctx->device[q] != ctx->device[p]);
  if (pull && phase == 0 && fuse) {
    // the pull rides along the local pass (HaloPull), then the remote pass
    launch_aggregate(ctx, plan, in, out, relu, 1, halo, st, nullptr, const_cast<float*>(halo));
    launch_aggregate(ctx, plan, in, out, relu, 2, halo, st);
    return;
  }
  if (pull) {
    MGG_CUDA(cudaEventRecord(ctx->fork[p], st));
    MGG_CUDA(cudaStreamWaitEvent(ctx->aux[p], ctx->fork[p], 0));
    launch_halo_pull(plan, in, const_cast<float*>(halo), ctx->aux[p]);
    MGG_CUDA(cudaEventRecord(ctx->join[p], ctx->aux[p]));
    count_launch(ctx);
  }
  if (phase != 2) launch_aggregate(ctx, plan, in, out, relu, 1, halo, st);
  if (phase != 1 && phase != 3) {
    if (pull) MGG_CUDA(cudaStreamWaitEvent(st, ctx->join[p], 0));
    launch_aggregate(ctx, plan, in, out, relu, 2, halo, st);
  }
}

}  // namespace mgg::dev

using namespace mgg::dev;

extern "C" {

const char* mgg_last_error(void) { return g_last_error.c_str(); }

int mgg_cuda_available(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n > 0 ? 1 : 0;
}

int mgg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int mgg_ctx_create(uint32_t num_parts, const int32_t* part_device, mgg_ctx** out) {
  return guard([&] {
    if (!out || !part_device) throw Status{MGG_E_INPUT, "ctx_create: null argument"};
    if (num_parts < 1 || num_parts > kMaxParts)
      throw Status{MGG_E_CONFIG, "ctx_create: num_parts must be in [1,16]"};
    int ndev = 0;
    MGG_CUDA(cudaGetDeviceCount(&ndev));
    auto* c = new mgg_ctx();
    try {
      c->num_parts = num_parts;
      c->device.assign(part_device, part_device + num_parts);
      c->stream.assign(num_parts, nullptr);
      c->ev0.assign(num_parts, nullptr);
      c->ev1.assign(num_parts, nullptr);
      c->aux.assign(num_parts, nullptr);
      c->fork.assign(num_parts, nullptr);
      c->join.assign(num_parts, nullptr);
      c->evpool.assign(num_parts, {});
      c->bar_ev.assign(num_parts, nullptr);
      {
        const char* e = std::getenv("MGG_PART_STREAMS");
        c->part_streams = !(e && std::string(e) == "0");
      }
      c->h2d.assign(num_parts, nullptr);
      c->d2h.assign(num_parts, nullptr);
      c->rp.assign(num_parts, nullptr);
      c->lane_ev.assign(num_parts, std::vector<cudaEvent_t>(9, nullptr));
      c->marks.assign(num_parts, {});
      c->shard_mem.assign(num_parts, MGG_MEM_DEVICE);
      int first = -1;
      for (uint32_t p = 0; p < num_parts; ++p) {
        const int d = c->device[p];
        if (d < 0) {
          c->all_local = false;
          continue;
        }
        if (d >= ndev) throw Status{MGG_E_INPUT, "ctx_create: no CUDA device " + std::to_string(d)};
        if (first < 0) first = d;
        if (d != first) c->single_device = false;
        MGG_CUDA(cudaSetDevice(d));
        // one compute/aux stream per part, also for logical partitions sharing
        // a device: they run concurrently and join at barriers with events
        // (MGG_PART_STREAMS=0: one stream per device, stream order instead)
        for (uint32_t q = 0; q < p && !c->part_streams; ++q)
          if (c->device[q] == d) c->stream[p] = c->stream[q];
        if (!c->stream[p]) MGG_CUDA(cudaStreamCreateWithFlags(&c->stream[p], cudaStreamNonBlocking));
        MGG_CUDA(cudaEventCreate(&c->ev0[p]));
        MGG_CUDA(cudaEventCreate(&c->ev1[p]));
        for (uint32_t q = 0; q < p && !c->part_streams; ++q)
          if (c->device[q] == d) c->aux[p] = c->aux[q];
        MGG_CUDA(cudaEventCreateWithFlags(&c->bar_ev[p], cudaEventDisableTiming));
        if (!c->aux[p]) MGG_CUDA(cudaStreamCreateWithFlags(&c->aux[p], cudaStreamNonBlocking));
        for (uint32_t q = 0; q < p; ++q)
          if (c->device[q] == d) {
            c->h2d[p] = c->h2d[q];
            c->d2h[p] = c->d2h[q];
            c->rp[p] = c->rp[q];
          }
        if (!c->h2d[p]) MGG_CUDA(cudaStreamCreateWithFlags(&c->h2d[p], cudaStreamNonBlocking));
        if (!c->d2h[p]) MGG_CUDA(cudaStreamCreateWithFlags(&c->d2h[p], cudaStreamNonBlocking));
        if (!c->rp[p]) MGG_CUDA(cudaStreamCreateWithFlags(&c->rp[p], cudaStreamNonBlocking));
        for (auto& e : c->lane_ev[p])
          MGG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        MGG_CUDA(cudaEventCreateWithFlags(&c->fork[p], cudaEventDisableTiming));
        MGG_CUDA(cudaEventCreateWithFlags(&c->join[p], cudaEventDisableTiming));
      }
      // peer access between every pair of local devices (single-process
      // multi-GPU); imported IPC shards enable it lazily
      for (uint32_t p = 0; p < num_parts; ++p)
        for (uint32_t q = 0; q < num_parts; ++q) {
          const int a = c->device[p], b = c->device[q];
          if (a < 0 || b < 0 || a == b) continue;
          int ok = 0;
          MGG_CUDA(cudaDeviceCanAccessPeer(&ok, a, b));
          if (!ok) throw Status{MGG_E_CUDA, "ctx_create: no peer access between devices"};
          MGG_CUDA(cudaSetDevice(a));
          const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled)
            cudaGetLastError();
          else
            MGG_CUDA(e);
        }
    } catch (...) {
      mgg_ctx_destroy(c);
      throw;
    }
    *out = c;
  });
}

int mgg_ctx_destroy(mgg_ctx* c) {
  if (!c) return MGG_OK;
  for (uint32_t p = 0; p < c->num_parts; ++p) {
    if (c->device[p] < 0) continue;
    cudaSetDevice(c->device[p]);
    bool shared = false;
    for (uint32_t q = 0; q < p; ++q) shared |= c->stream[q] == c->stream[p];
    if (c->stream[p] && !shared) cudaStreamDestroy(c->stream[p]);
    if (c->ev0[p]) cudaEventDestroy(c->ev0[p]);
    if (c->ev1[p]) cudaEventDestroy(c->ev1[p]);
    bool shared_aux = false;
    for (uint32_t q = 0; q < p; ++q) shared_aux |= c->aux[q] == c->aux[p];
    if (c->aux[p] && !shared_aux) cudaStreamDestroy(c->aux[p]);
    if (c->fork[p]) cudaEventDestroy(c->fork[p]);
    if (c->join[p]) cudaEventDestroy(c->join[p]);
    for (cudaEvent_t e : c->evpool[p])
      if (e) cudaEventDestroy(e);
    bool shared_cp = false;
    for (uint32_t q = 0; q < p; ++q) shared_cp |= c->h2d[q] == c->h2d[p];
    if (!shared_cp) {
      if (c->h2d[p]) cudaStreamDestroy(c->h2d[p]);
      if (c->d2h[p]) cudaStreamDestroy(c->d2h[p]);
      if (c->rp[p]) cudaStreamDestroy(c->rp[p]);
    }
    for (cudaEvent_t e : c->lane_ev[p])
      if (e) cudaEventDestroy(e);
    if (c->bar_ev[p]) cudaEventDestroy(c->bar_ev[p]);
    for (cudaEvent_t e : c->marks[p])
      if (e) cudaEventDestroy(e);
  }
  delete c;
  return MGG_OK;
}

int mgg_ctx_synchronize(mgg_ctx* c) {
  return guard([&] {
    for (uint32_t p = 0; p < c->num_parts; ++p) {
      if (c->device[p] < 0) continue;
      MGG_CUDA(cudaSetDevice(c->device[p]));
      MGG_CUDA(cudaStreamSynchronize(c->h2d[p]));
      MGG_CUDA(cudaStreamSynchronize(c->stream[p]));
      MGG_CUDA(cudaStreamSynchronize(c->d2h[p]));
    }
  });
}

static cudaStream_t lane_stream(mgg_ctx* ctx, uint32_t part, int lane) {
  cudaStream_t st = enter(ctx, part);
  switch (lane) {
    case MGG_LANE_COMPUTE: return st;
    case MGG_LANE_H2D: return ctx->h2d[part];
    case MGG_LANE_D2H: return ctx->d2h[part];
    default: throw Status{MGG_E_INPUT, "lane must be 0 (compute), 1 (h2d) or 2 (d2h)"};
  }
}

int mgg_lane_fence(mgg_ctx* ctx, uint32_t part, int from, int to) {
  return guard([&] {
    cudaStream_t a = lane_stream(ctx, part, from), b = lane_stream(ctx, part, to);
    if (a == b) return;
    cudaEvent_t e = ctx->lane_ev[part][from * 3 + to];
    MGG_CUDA(cudaEventRecord(e, a));
    MGG_CUDA(cudaStreamWaitEvent(b, e, 0));
  });
}

int mgg_lane_mark(mgg_ctx* ctx, uint32_t part, int lane, uint32_t slot) {
  return guard([&] {
    cudaStream_t st = lane_stream(ctx, part, lane);
    auto& m = ctx->marks[part];
    if (slot >= m.size()) m.resize(slot + 1, nullptr);
    if (!m[slot]) MGG_CUDA(cudaEventCreateWithFlags(&m[slot], cudaEventDisableTiming));
    MGG_CUDA(cudaEventRecord(m[slot], st));
  });
}

int mgg_lane_wait_mark(mgg_ctx* ctx, uint32_t part, int lane, uint32_t slot) {
  return guard([&] {
    cudaStream_t st = lane_stream(ctx, part, lane);
    const auto& m = ctx->marks[part];
    if (slot >= m.size() || !m[slot]) throw Status{MGG_E_INPUT, "lane_wait_mark: slot never marked"};
    MGG_CUDA(cudaStreamWaitEvent(st, m[slot], 0));
  });
}

int mgg_lane_wait_host(mgg_ctx* ctx, uint32_t part, uint32_t slot) {
  return guard([&] {
    enter(ctx, part);
    const auto& m = ctx->marks[part];
    if (slot >= m.size() || !m[slot]) throw Status{MGG_E_INPUT, "lane_wait_host: slot never marked"};
    MGG_CUDA(cudaEventSynchronize(m[slot]));
  });
}

uint64_t mgg_ctx_launch_count(const mgg_ctx* c) { return c ? c->launches : 0; }

static uint32_t first_local(mgg_ctx* ctx) {
  for (uint32_t p = 0; p < ctx->num_parts; ++p)
    if (ctx->device[p] >= 0) return p;
  throw Status{MGG_E_INPUT, "context has no local part"};
}

int mgg_ctx_join(mgg_ctx* ctx) {
  return guard([&] {
    if (!ctx || !ctx->part_streams) return;
    for (uint32_t p = 0; p < ctx->num_parts; ++p)
      if (ctx->device[p] >= 0) {
        enter(ctx, p);
        MGG_CUDA(cudaEventRecord(ctx->bar_ev[p], ctx->stream[p]));
      }
    for (uint32_t p = 0; p < ctx->num_parts; ++p)
      for (uint32_t q = 0; q < ctx->num_parts; ++q)
        if (q != p && ctx->device[p] >= 0 && ctx->device[q] == ctx->device[p]) {
          enter(ctx, p);
          MGG_CUDA(cudaStreamWaitEvent(ctx->stream[p], ctx->bar_ev[q], 0));
        }
  });
}

int mgg_capture_begin(mgg_ctx* ctx) {
  return guard([&] {
    if (!ctx) throw Status{MGG_E_INPUT, "capture_begin: null context"};
    // parts driven by other processes are not captured: their side of every
    // K3 barrier is their own replay (the barrier's epoch lives on the device)
    if (ctx->capturing) throw Status{MGG_E_INPUT, "capture_begin: already capturing"};
    const uint32_t p0 = first_local(ctx);
    cudaStream_t st = enter(ctx, p0);
    MGG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    ctx->capturing = true;
    ctx->capture_base = ctx->launches;
    // pull the other parts' streams (other devices' too) into the capture
    MGG_CUDA(cudaEventRecord(ctx->bar_ev[p0], st));
    for (uint32_t p = 0; p < ctx->num_parts; ++p)
      if (p != p0 && ctx->device[p] >= 0 && ctx->stream[p] != st) {
        enter(ctx, p);
        MGG_CUDA(cudaStreamWaitEvent(ctx->stream[p], ctx->bar_ev[p0], 0));
      }
    enter(ctx, p0);
  });
}

int mgg_capture_end(mgg_ctx* ctx, mgg_exec** out) {
  return guard([&] {
    if (!ctx || !out) throw Status{MGG_E_INPUT, "capture_end: null argument"};
    if (!ctx->capturing) throw Status{MGG_E_INPUT, "capture_end: not capturing"};
    const uint32_t p = first_local(ctx);
    cudaStream_t st = enter(ctx, p);
    ctx->capturing = false;
    for (uint32_t q = 0; q < ctx->num_parts; ++q)  // join the other parts' streams back
      if (q != p && ctx->device[q] >= 0 && ctx->stream[q] != st) {
        enter(ctx, q);
        MGG_CUDA(cudaEventRecord(ctx->bar_ev[q], ctx->stream[q]));
        enter(ctx, p);
        MGG_CUDA(cudaStreamWaitEvent(st, ctx->bar_ev[q], 0));
      }
    enter(ctx, p);
    cudaGraph_t g = nullptr;
    MGG_CUDA(cudaStreamEndCapture(st, &g));
    auto* e = new mgg_exec();
    e->device = ctx->device[p];
    e->kernels = ctx->launches - ctx->capture_base;
    ctx->launches = ctx->capture_base;  // captured, not launched
    const cudaError_t r = cudaGraphInstantiate(&e->exec, g, 0);
    cudaGraphDestroy(g);
    if (r != cudaSuccess) {
      delete e;
      check(r, "cudaGraphInstantiate");
    }
    *out = e;
  });
}

int mgg_exec_launch(mgg_ctx* ctx, const mgg_exec* g) {
  return guard([&] {
    if (!ctx || !g) throw Status{MGG_E_INPUT, "exec_launch: null argument"};
    cudaStream_t st = enter(ctx, first_local(ctx));
    MGG_CUDA(cudaGraphLaunch(g->exec, st));
    ctx->launches += g->kernels;
  });
}

int mgg_exec_destroy(mgg_exec* g) {
  if (!g) return MGG_OK;
  // at process teardown the runtime may already be gone: leak, don't crash
  if (cudaSetDevice(g->device) == cudaSuccess) cudaGraphExecDestroy(g->exec);
  delete g;
  return MGG_OK;
}

int mgg_event_record(mgg_ctx* ctx, uint32_t part, uint32_t slot) {
  return guard([&] {
    cudaStream_t st = enter(ctx, part);
    auto& pool = ctx->evpool[part];
    if (slot >= pool.size()) pool.resize(slot + 1, nullptr);
    if (!pool[slot]) MGG_CUDA(cudaEventCreate(&pool[slot]));
    MGG_CUDA(cudaEventRecord(pool[slot], st));
  });
}

int mgg_event_elapsed(mgg_ctx* ctx, uint32_t part, uint32_t a, uint32_t b, float* ms) {
  return guard([&] {
    enter(ctx, part);
    const auto& pool = ctx->evpool[part];
    if (a >= pool.size() || b >= pool.size() || !pool[a] || !pool[b])
      throw Status{MGG_E_INPUT, "event_elapsed: slot never recorded"};
    MGG_CUDA(cudaEventSynchronize(pool[b]));
    MGG_CUDA(cudaEventElapsedTime(ms, pool[a], pool[b]));
  });
}

int mgg_event_elapsed_between(mgg_ctx* ctx, uint32_t part_a, uint32_t a, uint32_t part_b,
                              uint32_t b, float* ms) {
  return guard([&] {
    enter(ctx, part_a);
    enter(ctx, part_b);
    if (ctx->device[part_a] != ctx->device[part_b])
      throw Status{MGG_E_INPUT, "event_elapsed_between: parts on different devices"};
    const auto& pa = ctx->evpool[part_a];
    const auto& pb = ctx->evpool[part_b];
    if (a >= pa.size() || b >= pb.size() || !pa[a] || !pb[b])
      throw Status{MGG_E_INPUT, "event_elapsed_between: slot never recorded"};
    MGG_CUDA(cudaEventSynchronize(pb[b]));
    MGG_CUDA(cudaEventSynchronize(pa[a]));
    MGG_CUDA(cudaEventElapsedTime(ms, pa[a], pb[b]));
  });
}

// ---- symmetric VMM stores -------------------------------------------------
// Driver entry points are fetched through the runtime (no link-time libcuda
// dependency: the library still loads where no driver exists).
struct Vmm {
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemSetAccess) access = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemAddressFree) vfree = nullptr;
  decltype(&cuMemExportToShareableHandle) export_fd = nullptr;
  decltype(&cuMemImportFromShareableHandle) import_fd = nullptr;
  bool ok = false, fd_ok = false;
};
const Vmm& vmm() {
  static const Vmm v = [] {
    Vmm r;
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q{};
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
    r.ok = get("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&r.granularity)) &&
           get("cuMemCreate", reinterpret_cast<void**>(&r.create)) &&
           get("cuMemAddressReserve", reinterpret_cast<void**>(&r.reserve)) &&
           get("cuMemMap", reinterpret_cast<void**>(&r.map)) &&
           get("cuMemSetAccess", reinterpret_cast<void**>(&r.access)) &&
           get("cuMemRelease", reinterpret_cast<void**>(&r.release)) &&
           get("cuMemUnmap", reinterpret_cast<void**>(&r.unmap)) &&
           get("cuMemAddressFree", reinterpret_cast<void**>(&r.vfree));
    r.fd_ok = r.ok && get("cuMemExportToShareableHandle", reinterpret_cast<void**>(&r.export_fd)) &&
              get("cuMemImportFromShareableHandle", reinterpret_cast<void**>(&r.import_fd));
    cudaGetLastError();
    return r;
  }();
  return v;
}
// MGG_VMM=0 keeps one cudaMalloc per shard (the pointer-table layout).
bool vmm_wanted() {
  static const bool m = [] {
    const char* e = std::getenv("MGG_VMM");
    return !e || std::atoi(e) != 0;
  }();
  return m;
}
// MGG_VMM_IPC=1: one-process-per-GPU stores are symmetric VMM ranges too,
// each rank's shard exported as a POSIX fd and mapped by its peers at the same
// offset (mgg_store_vmm_export / _import); default: CUDA IPC handles.
bool vmm_ipc_wanted() {
  static const bool m = [] {
    const char* e = std::getenv("MGG_VMM_IPC");
    return e && std::atoi(e) != 0;
  }();
  return m;
}
void drv(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw Status{MGG_E_CUDA, std::string("VMM ") + what + " failed"};
}

// Allocates every local part's shard in one symmetric virtual range (all
// parts local and in device memory); false when VMM is off or unavailable.
bool vmm_store_alloc(mgg_store* s) {
  mgg_ctx* ctx = s->ctx;
  const bool cross = !ctx->all_local;  // parts in other processes: fd-exported shards
  if (!vmm_wanted() || !vmm().ok) return false;
  if (cross && !(vmm_ipc_wanted() && vmm().fd_ok)) return false;
  for (uint32_t p = 0; p < ctx->num_parts; ++p)
    if (ctx->device[p] >= 0 && ctx->shard_mem[p] != MGG_MEM_DEVICE) return false;
  const Vmm& v = vmm();
  size_t gran = 0;
  std::vector<int> devs;
  for (uint32_t p = 0; p < ctx->num_parts; ++p)
    if (ctx->device[p] >= 0 &&
        std::find(devs.begin(), devs.end(), ctx->device[p]) == devs.end())
      devs.push_back(ctx->device[p]);
  for (int d : devs) {
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = d;
    size_t g = 0;
    drv(v.granularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "granularity");
    gran = std::max(gran, g);
  }
  auto up = [&](size_t x) { return (x + gran - 1) / gran * gran; };
  s->vmm_size.assign(ctx->num_parts, 0);
  size_t stride = gran;
  for (uint32_t p = 0; p < ctx->num_parts; ++p) {
    s->vmm_size[p] = up(std::max<size_t>(s->rows(p) * s->pitch * sizeof(float), 256));
    stride = std::max(stride, s->vmm_size[p]);
  }
  CUdeviceptr base = 0;
  drv(v.reserve(&base, stride * ctx->num_parts, gran, 0, 0), "address reserve");
  s->vmm_base = reinterpret_cast<char*>(base);
  s->vmm_stride = stride;
  std::vector<CUmemAccessDesc> acc(devs.size());
  for (size_t i = 0; i < devs.size(); ++i) {
    acc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[i].location.id = devs[i];
    acc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  s->vmm_ipc = cross;
  s->vmm_handle.assign(ctx->num_parts, 0);
  s->vmm_mapped.assign(ctx->num_parts, 0);
  for (uint32_t p = 0; p < ctx->num_parts; ++p) {
    if (ctx->device[p] < 0) continue;  // a peer's slot: mapped by mgg_store_vmm_import
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = ctx->device[p];
    if (cross) prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle h = 0;
    drv(v.create(&h, s->vmm_size[p], &prop, 0), "create");
    const CUdeviceptr at = base + p * stride;
    const CUresult mr = v.map(at, s->vmm_size[p], 0, h, 0);
    if (cross && mr == CUDA_SUCCESS)
      s->vmm_handle[p] = h;  // kept for the fd export, released at destroy
    else
      v.release(h);  // the mapping keeps the memory alive
    drv(mr, "map");
    s->vmm_mapped[p] = 1;
    s->shard[p] = reinterpret_cast<float*>(at);  // mapped: unmapped by vmm_store_free
    drv(v.access(at, s->vmm_size[p], acc.data(), acc.size()), "set access");
    s->owned[p] = 1;
    s->mem[p] = MGG_MEM_DEVICE;
    s->bytes[p] = std::max<size_t>(s->rows(p) * s->pitch * sizeof(float), 256);
    MGG_CUDA(cudaSetDevice(ctx->device[p]));
    MGG_CUDA(cudaMemsetAsync(s->shard[p], 0, s->bytes[p], ctx->stream[p]));
    MGG_CUDA(cudaStreamSynchronize(ctx->stream[p]));
  }
  return true;
}

void vmm_store_free(mgg_store* s) {
  if (!s->vmm_base) return;
  const Vmm& v = vmm();
  const CUdeviceptr base = reinterpret_cast<CUdeviceptr>(s->vmm_base);
  for (uint32_t p = 0; p < s->ctx->num_parts; ++p) {
    if (p < s->vmm_mapped.size() && s->vmm_mapped[p])
      v.unmap(base + p * s->vmm_stride, s->vmm_size[p]);
    if (p < s->vmm_handle.size() && s->vmm_handle[p]) v.release(s->vmm_handle[p]);
  }
  v.vfree(base, s->vmm_stride * s->ctx->num_parts);
  s->vmm_base = nullptr;
  s->vmm_mapped.clear();
  s->vmm_handle.clear();
}

int mgg_store_create(mgg_ctx* ctx, const uint64_t* part_lb, uint32_t dim, mgg_store** out) {
  return guard([&] {
    if (!ctx || !part_lb || !out) throw Status{MGG_E_INPUT, "store_create: null argument"};
    if (dim == 0) throw Status{MGG_E_INPUT, "store_create: dim must be >= 1"};
    auto* s = new mgg_store();
    try {
      s->ctx = ctx;
      s->dim = dim;
      s->pitch = (dim + 3) / 4 * 4;
      s->lb.assign(part_lb, part_lb + ctx->num_parts + 1);
      for (uint32_t p = 0; p < ctx->num_parts; ++p)
        if (s->lb[p + 1] < s->lb[p]) throw Status{MGG_E_INPUT, "store_create: ranges must be ascending"};
      s->shard.assign(ctx->num_parts, nullptr);
      s->owned.assign(ctx->num_parts, 0);
      s->imported.assign(ctx->num_parts, 0);
      s->mem.assign(ctx->num_parts, MGG_MEM_DEVICE);
      s->bytes.assign(ctx->num_parts, 0);
      s->dtable.assign(ctx->num_parts, nullptr);
      s->stage.assign(2 * ctx->num_parts, nullptr);
      s->stage_ev.assign(5 * ctx->num_parts, nullptr);
      bool symmetric = false;
      try {
        symmetric = vmm_store_alloc(s);
      } catch (const Status&) {  // e.g. devices without peer mappings: per-shard allocations
        vmm_store_free(s);
        std::fill(s->shard.begin(), s->shard.end(), nullptr);
        std::fill(s->owned.begin(), s->owned.end(), 0);
        s->vmm_size.clear();
        s->vmm_stride = 0;
        cudaGetLastError();
      }
      for (uint32_t p = 0; p < ctx->num_parts && !symmetric; ++p) {
        if (ctx->device[p] < 0) continue;
        MGG_CUDA(cudaSetDevice(ctx->device[p]));
        const size_t bytes = std::max<size_t>(s->rows(p) * s->pitch * sizeof(float), 256);
        const int kind = ctx->shard_mem[p];
        void* d = nullptr;
        switch (kind) {
          case MGG_MEM_HOST_MAPPED: {
            void* h = nullptr;
            MGG_CUDA(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
            std::memset(h, 0, bytes);
            s->shard[p] = static_cast<float*>(h);  // freed through the host pointer
            MGG_CUDA(cudaHostGetDevicePointer(&d, h, 0));
            if (d != h) {
              cudaFreeHost(h);
              s->shard[p] = nullptr;
              throw Status{MGG_E_CUDA, "store_create: host-mapped shard needs unified addressing"};
            }
            break;
          }
          case MGG_MEM_MANAGED:
          case MGG_MEM_MANAGED_HOST:
            MGG_CUDA(cudaMallocManaged(&d, bytes, cudaMemAttachGlobal));
            break;
          default:
            MGG_CUDA(cudaMalloc(&d, bytes));
        }
        s->shard[p] = static_cast<float*>(d);
        s->owned[p] = 1;
        s->mem[p] = static_cast<uint8_t>(kind);
        s->bytes[p] = bytes;
        if (kind != MGG_MEM_HOST_MAPPED) {
          // zero padding/rows on the part's stream, complete before any use
          // (a legacy-stream memset is not ordered before non-blocking streams)
          MGG_CUDA(cudaMemsetAsync(d, 0, bytes, ctx->stream[p]));
          MGG_CUDA(cudaStreamSynchronize(ctx->stream[p]));
        }
      }
      refresh_tables(s);
      rehome(s, nullptr);
    } catch (...) {
      mgg_store_destroy(s);
      throw;
    }
    *out = s;
  });
}

int mgg_ctx_set_shard_memory(mgg_ctx* ctx, uint32_t part, int kind) {
  return guard([&] {
    enter(ctx, part);
    if (kind < MGG_MEM_DEVICE || kind > MGG_MEM_MANAGED_HOST)
      throw Status{MGG_E_INPUT, "set_shard_memory: unknown memory kind"};
    if (kind != MGG_MEM_DEVICE) {
      int v = 0;
      MGG_CUDA(cudaDeviceGetAttribute(&v, kind == MGG_MEM_HOST_MAPPED
                                              ? cudaDevAttrCanMapHostMemory
                                              : cudaDevAttrConcurrentManagedAccess,
                                      ctx->device[part]));
      if (!v) throw Status{MGG_E_CONFIG, "set_shard_memory: device cannot use that memory kind"};
    }
    ctx->shard_mem[part] = kind;
  });
}

int mgg_store_rehome(mgg_store* s) {
  return guard([&] {
    if (!s) throw Status{MGG_E_INPUT, "store_rehome: null store"};
    rehome(s, nullptr);
  });
}

int mgg_store_destroy(mgg_store* s) {
  if (!s) return MGG_OK;
  mgg_ctx* ctx = s->ctx;
  if (s->vmm_base) {  // symmetric range: every device done with it, then unmapped
    for (uint32_t p = 0; p < ctx->num_parts; ++p)
      if (ctx->device[p] >= 0 && cudaSetDevice(ctx->device[p]) == cudaSuccess)
        cudaDeviceSynchronize();
    vmm_store_free(s);
    std::fill(s->owned.begin(), s->owned.end(), 0);
  }
  for (uint32_t p = 0; p < ctx->num_parts; ++p) {
    if (s->owned[p] && s->shard[p]) {
      cudaSetDevice(ctx->device[p]);
      if (s->mem[p] == MGG_MEM_HOST_MAPPED)
        cudaFreeHost(s->shard[p]);
      else
        cudaFree(s->shard[p]);
    }
    if (s->imported[p] && s->shard[p]) cudaIpcCloseMemHandle(s->shard[p]);
    if (s->dtable[p]) {
      cudaSetDevice(ctx->device[p]);
      cudaFree(s->dtable[p]);
    }
    for (int i = 0; i < 2; ++i)
      if (s->stage[2 * p + i]) {
        cudaSetDevice(ctx->device[p]);
        cudaFree(s->stage[2 * p + i]);
      }
    for (int i = 0; i < 5; ++i)
      if (s->stage_ev[5 * p + i]) cudaEventDestroy(s->stage_ev[5 * p + i]);
  }
  delete s;
  return MGG_OK;
}

int mgg_store_vmm_export(const mgg_store* s, uint32_t part, int* fd) {
  return guard([&] {
    if (!s || !fd || part >= s->ctx->num_parts) throw Status{MGG_E_INPUT, "vmm_export: bad argument"};
    if (!s->vmm_ipc || part >= s->vmm_handle.size() || !s->vmm_handle[part])
      throw Status{MGG_E_CONFIG, "vmm_export: not a local shard of a cross-process VMM store"};
    int out = -1;
    drv(vmm().export_fd(&out, s->vmm_handle[part], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
        "export");
    *fd = out;
  });
}

int mgg_store_vmm_import(mgg_store* s, uint32_t part, int fd) {
  return guard([&] {
    if (!s || part >= s->ctx->num_parts) throw Status{MGG_E_INPUT, "vmm_import: bad argument"};
    mgg_ctx* ctx = s->ctx;
    if (!s->vmm_ipc) throw Status{MGG_E_CONFIG, "vmm_import: not a cross-process VMM store"};
    if (ctx->device[part] >= 0) throw Status{MGG_E_INPUT, "vmm_import: part is local"};
    if (s->vmm_mapped[part]) throw Status{MGG_E_INPUT, "vmm_import: slot already mapped"};
    const Vmm& v = vmm();
    CUmemGenericAllocationHandle h = 0;
    drv(v.import_fd(&h, reinterpret_cast<void*>(static_cast<intptr_t>(fd)),
                    CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
        "import");
    const CUdeviceptr at = reinterpret_cast<CUdeviceptr>(s->vmm_base) + part * s->vmm_stride;
    const CUresult mr = v.map(at, s->vmm_size[part], 0, h, 0);
    v.release(h);
    drv(mr, "map (import)");
    s->vmm_mapped[part] = 1;
    s->shard[part] = reinterpret_cast<float*>(at);
    std::vector<CUmemAccessDesc> acc;
    for (uint32_t p = 0; p < ctx->num_parts; ++p)
      if (ctx->device[p] >= 0) {
        CUmemAccessDesc d{};
        d.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        d.location.id = ctx->device[p];
        d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        bool dup = false;
        for (auto& x : acc) dup |= x.location.id == d.location.id;
        if (!dup) acc.push_back(d);
      }
    drv(v.access(at, s->vmm_size[part], acc.data(), acc.size()), "set access (import)");
    refresh_tables(s);
  });
}

int mgg_store_layout(const mgg_store* s, int* symmetric, uint64_t* stride) {
  if (!s) return MGG_E_INPUT;
  if (symmetric) *symmetric = s->vmm_base ? (s->vmm_ipc ? 2 : 1) : 0;
  if (stride) *stride = s->vmm_stride;
  return MGG_OK;
}

int mgg_store_info(const mgg_store* s, uint32_t* dim, uint32_t* pitch) {
  if (!s) return MGG_E_INPUT;
  if (dim) *dim = s->dim;
  if (pitch) *pitch = s->pitch;
  return MGG_OK;
}

int mgg_store_ipc_export(const mgg_store* s, uint32_t part, void* handle64) {
  return guard([&] {
    if (!s || part >= s->ctx->num_parts || !s->owned[part])
      throw Status{MGG_E_INPUT, "ipc_export: part is not a local shard"};
    if (s->mem[part] != MGG_MEM_DEVICE)
      throw Status{MGG_E_CONFIG, "ipc_export: shard is not device memory"};
    if (s->vmm_base)
      throw Status{MGG_E_CONFIG, "ipc_export: symmetric (VMM) store of a single-process context"};
    MGG_CUDA(cudaSetDevice(s->ctx->device[part]));
    cudaIpcMemHandle_t h;
    MGG_CUDA(cudaIpcGetMemHandle(&h, s->shard[part]));
    std::memcpy(handle64, &h, sizeof(h));
  });
}

int mgg_store_ipc_import(mgg_store* s, uint32_t part, const void* handle64) {
  return guard([&] {
    mgg_ctx* ctx = s->ctx;
    if (part >= ctx->num_parts || ctx->device[part] >= 0)
      throw Status{MGG_E_INPUT, "ipc_import: part is local"};
    int dev = -1;
    for (uint32_t p = 0; p < ctx->num_parts; ++p)
      if (ctx->device[p] >= 0) dev = ctx->device[p];
    if (dev < 0) throw Status{MGG_E_INPUT, "ipc_import: context has no local part"};
    MGG_CUDA(cudaSetDevice(dev));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    void* d = nullptr;
    MGG_CUDA(cudaIpcOpenMemHandle(&d, h, cudaIpcMemLazyEnablePeerAccess));
    if (s->imported[part] && s->shard[part]) cudaIpcCloseMemHandle(s->shard[part]);
    s->shard[part] = static_cast<float*>(d);
    s->imported[part] = 1;
    refresh_tables(s);
  });
}

}  // extern "C"

namespace mgg::dev {

// Dense <-> pitched row copies on the device (the H2D/D2H legs stay 1D:
// PCIe DMA of 2D copies with 2.4 KB rows runs at a third of the 1D rate).
__global__ void repitch_kernel(const float* __restrict__ src, uint32_t src_ld,
                               float* __restrict__ dst, uint32_t dst_ld, uint64_t rows,
                               uint32_t cols) {
  // one warp per row, lanes stride the columns (coalesced on both sides;
  // no per-element division)
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
       r += warps) {
    const float* a = src + r * src_ld;
    float* b = dst + r * dst_ld;
    for (uint32_t c = lane; c < cols; c += 32) b[c] = __ldg(a + c);
  }
}

void repitch(const float* src, uint32_t src_ld, float* dst, uint32_t dst_ld, uint64_t rows,
             uint32_t cols, cudaStream_t st) {
  const uint64_t total = rows * cols;
  if (!total) return;
  const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((rows + 7) / 8, 148 * 16));
  repitch_kernel<<<blocks, 256, 0, st>>>(src, src_ld, dst, dst_ld, rows, cols);
  MGG_CUDA(cudaGetLastError());
}

constexpr size_t kStageBytes = 32u << 20;

}  // namespace mgg::dev

extern "C" {

static int copy_rows(const mgg_store* cs, float* host_rw, const float* host_ro,
                     uint64_t row_begin, uint64_t row_count, uint32_t ld, bool up, int lane) {
  return guard([&] {
    if (!cs) throw Status{MGG_E_INPUT, "store copy: null store"};
    if (ld < cs->dim) throw Status{MGG_E_INPUT, "store copy: ld < dim"};
    auto* s = const_cast<mgg_store*>(cs);
    mgg_ctx* ctx = s->ctx;
    const uint64_t end = row_begin + row_count;
    for (uint32_t p = 0; p < ctx->num_parts; ++p) {
      if (ctx->device[p] < 0) continue;
      const uint64_t a = std::max(row_begin, s->lb[p]), b = std::min(end, s->lb[p + 1]);
      if (a >= b) continue;
      cudaStream_t st = lane_stream(ctx, p, lane);
      float* dev = s->shard[p] + (a - s->lb[p]) * s->pitch;
      const size_t hoff = (a - row_begin) * (size_t)ld;
      const size_t row_bytes = size_t(s->dim) * 4;
      if (ld == s->pitch && s->pitch == s->dim) {  // identical, unpadded layout: one 1D copy
        if (up)
          MGG_CUDA(cudaMemcpyAsync(dev, host_ro + hoff, (b - a) * row_bytes, cudaMemcpyHostToDevice, st));
        else
          MGG_CUDA(cudaMemcpyAsync(host_rw + hoff, dev, (b - a) * row_bytes, cudaMemcpyDeviceToHost, st));
        continue;
      }
      if (ld != s->dim) {  // strided host rows: the DMA engine's 2D path
        if (up)
          MGG_CUDA(cudaMemcpy2DAsync(dev, s->pitch * 4, host_ro + hoff, ld * 4, row_bytes, b - a,
                                     cudaMemcpyHostToDevice, st));
        else
          MGG_CUDA(cudaMemcpy2DAsync(host_rw + hoff, ld * 4, dev, s->pitch * 4, row_bytes, b - a,
                                     cudaMemcpyDeviceToHost, st));
        continue;
      }
      // dense host rows, padded device rows: 1D DMA through two staging
      // slabs; the re-pitch kernels run on the device's rp stream so the
      // copy of chunk i+1 proceeds while chunk i is re-pitched
      float** slab = &s->stage[2 * p];
      cudaEvent_t* ev = &s->stage_ev[5 * p];  // full0 full1 free0 free1 tail
      if (!slab[0]) {
        for (int i = 0; i < 2; ++i) {
          MGG_CUDA(cudaMalloc(reinterpret_cast<void**>(&slab[i]), kStageBytes));
          MGG_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
          MGG_CUDA(cudaEventCreateWithFlags(&ev[2 + i], cudaEventDisableTiming));
        }
        MGG_CUDA(cudaEventCreateWithFlags(&ev[4], cudaEventDisableTiming));
      }
      cudaStream_t rs = ctx->rp[p];
      // the re-pitch stream starts after whatever the lane was ordered behind
      MGG_CUDA(cudaEventRecord(ev[4], st));
      MGG_CUDA(cudaStreamWaitEvent(rs, ev[4], 0));
      const uint64_t chunk = std::max<uint64_t>(1, kStageBytes / row_bytes);
      int i = 0;
      for (uint64_t r = a; r < b; r += chunk, i ^= 1) {
        const uint64_t n = std::min(chunk, b - r);
        float* d = s->shard[p] + (r - s->lb[p]) * s->pitch;
        const size_t h = (r - row_begin) * (size_t)ld;
        if (up) {
          MGG_CUDA(cudaStreamWaitEvent(st, ev[2 + i], 0));  // slab drained
          MGG_CUDA(cudaMemcpyAsync(slab[i], host_ro + h, n * row_bytes, cudaMemcpyHostToDevice, st));
          MGG_CUDA(cudaEventRecord(ev[i], st));
          MGG_CUDA(cudaStreamWaitEvent(rs, ev[i], 0));
          repitch(slab[i], s->dim, d, s->pitch, n, s->dim, rs);
          MGG_CUDA(cudaEventRecord(ev[2 + i], rs));
        } else {
          MGG_CUDA(cudaStreamWaitEvent(rs, ev[2 + i], 0));  // slab copied out
          repitch(d, s->pitch, slab[i], s->dim, n, s->dim, rs);
          MGG_CUDA(cudaEventRecord(ev[i], rs));
          MGG_CUDA(cudaStreamWaitEvent(st, ev[i], 0));
          MGG_CUDA(cudaMemcpyAsync(host_rw + h, slab[i], n * row_bytes, cudaMemcpyDeviceToHost, st));
          MGG_CUDA(cudaEventRecord(ev[2 + i], st));
        }
      }
      if (up) {  // the lane completes only when the last re-pitch has
        MGG_CUDA(cudaEventRecord(ev[4], rs));
        MGG_CUDA(cudaStreamWaitEvent(st, ev[4], 0));
      }
    }
  });
}

int mgg_store_upload(mgg_store* s, const float* host, uint64_t row_begin,
                     uint64_t row_count, uint32_t ld) {
  return copy_rows(s, nullptr, host, row_begin, row_count, ld, true, MGG_LANE_COMPUTE);
}

int mgg_store_download(const mgg_store* s, float* host, uint64_t row_begin,
                       uint64_t row_count, uint32_t ld) {
  return copy_rows(s, host, nullptr, row_begin, row_count, ld, false, MGG_LANE_COMPUTE);
}

int mgg_store_upload_on(mgg_store* s, const float* host, uint64_t row_begin,
                        uint64_t row_count, uint32_t ld, int lane) {
  return copy_rows(s, nullptr, host, row_begin, row_count, ld, true, lane);
}

int mgg_store_download_on(const mgg_store* s, float* host, uint64_t row_begin,
                          uint64_t row_count, uint32_t ld, int lane) {
  return copy_rows(s, host, nullptr, row_begin, row_count, ld, false, lane);
}

int mgg_store_shard(const mgg_store* s, uint32_t part, void** dptr) {
  if (!s || part >= s->ctx->num_parts || !dptr) return MGG_E_INPUT;
  *dptr = s->shard[part];
  return MGG_OK;
}

int mgg_dbuf_create(mgg_ctx* ctx, uint32_t part, const void* host, size_t bytes,
                    mgg_dbuf** out) {
  return guard([&] {
    enter(ctx, part);
    auto* b = new mgg_dbuf();
    b->ctx = ctx;
    b->part = part;
    b->bytes = bytes;
    const cudaError_t e = cudaMalloc(&b->ptr, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) {
      delete b;
      check(e, "cudaMalloc");
    }
    if (bytes && host) {
      cudaStream_t st = ctx->stream[part];
      MGG_CUDA(cudaMemcpyAsync(b->ptr, host, bytes, cudaMemcpyHostToDevice, st));
      MGG_CUDA(cudaStreamSynchronize(st));
    }
    *out = b;
  });
}

int mgg_dbuf_destroy(mgg_dbuf* b) {
  if (!b) return MGG_OK;
  cudaSetDevice(b->ctx->device[b->part]);
  cudaFree(b->ptr);
  if (b->tc_cache) cudaFree(b->tc_cache);
  delete b;
  return MGG_OK;
}

void* mgg_dbuf_ptr(const mgg_dbuf* b) { return b ? b->ptr : nullptr; }

int mgg_host_alloc(size_t bytes, void** out) {
  return guard([&] { MGG_CUDA(cudaHostAlloc(out, std::max<size_t>(bytes, 16), cudaHostAllocPortable)); });
}

int mgg_host_free(void* p) {
  return guard([&] { MGG_CUDA(cudaFreeHost(p)); });
}

int mgg_dplan_upload(mgg_ctx* ctx, const mgg_plan_desc* d, mgg_dplan** out) {
  return guard([&] {
    if (!d || !out) throw Status{MGG_E_INPUT, "dplan_upload: null argument"};
    enter(ctx, d->part);
    if (d->ps < 1 || d->dist < 1 || d->wpb < 1 || d->wpb > 16)
      throw Status{MGG_E_CONFIG, "dplan_upload: bad ps/dist/wpb"};
    if (d->n_local > 0x7fffffffull || d->n_remote > 0x7fffffffull)
      throw Status{MGG_E_CONFIG, "dplan_upload: too many partitions"};
    auto* p = new mgg_dplan();
    try {
      p->ctx = ctx;
      p->part = d->part;
      p->ps = d->ps;
      p->dist = d->dist;
      p->wpb = d->wpb;
      p->mapping = d->mapping;
      p->granularity = d->granularity;
      p->rows = d->rows;
      p->n_local = d->n_local;
      p->n_remote = d->n_remote;
      p->local_edges = d->local_cols_len;
      p->remote_edges = d->remote_cols_len;
      // every upload and the owner strip are ordered on the part's stream and
      // complete before the plan is returned: the plan is later read from
      // the part's aux stream and from captured graphs too
      cudaStream_t st = ctx->stream[d->part];
      p->lmeta = reinterpret_cast<int2*>(upload_array(d->local_meta, 2 * (d->n_local + 1), st));
      p->rmeta = reinterpret_cast<int2*>(upload_array(d->remote_meta, 2 * (d->n_remote + 1), st));
      p->lcols = upload_array(d->local_cols, d->local_cols_len, st);
      launch_strip_owner(p->lcols, d->local_cols_len, st);
      p->rcols = upload_array(d->remote_cols, d->remote_cols_len, st);
      if (d->halo_rows && d->halo_len && d->remote_halo_cols) {
        p->halo_rows = upload_array(d->halo_rows, d->halo_len, st);
        p->halo_len = d->halo_len;
        p->rcols_halo = upload_array(d->remote_halo_cols, d->remote_cols_len, st);
      }
      MGG_CUDA(cudaMalloc(&p->sched, kSchedBytes));
      MGG_CUDA(cudaMemsetAsync(p->sched, 0, kSchedBytes, st));
      MGG_CUDA(cudaStreamSynchronize(st));
      p->num_local_warps = (d->n_local + d->dist - 1) / d->dist;
      const uint64_t nr_w = (d->n_remote + d->dist - 1) / d->dist;
      p->num_warps = d->mapping == 0 ? std::max(p->num_local_warps, nr_w)
                                     : p->num_local_warps + nr_w;
    } catch (...) {
      mgg_dplan_destroy(p);
      throw;
    }
    *out = p;
  });
}

int mgg_dplan_destroy(mgg_dplan* p) {
  if (!p) return MGG_OK;
  cudaSetDevice(p->ctx->device[p->part]);
  cudaFree(p->lmeta);
  cudaFree(p->rmeta);
  cudaFree(p->lcols);
  cudaFree(p->rcols);
  cudaFree(p->halo_rows);
  cudaFree(p->rcols_halo);
  cudaFree(p->sched);
  delete p;
  return MGG_OK;
}

int mgg_aggregate(mgg_ctx* ctx, const mgg_dplan* plan, const mgg_store* in,
                  mgg_store* out, const mgg_agg_opts* opts) {
  return guard([&] {
    if (!plan || !in || !out) throw Status{MGG_E_INPUT, "aggregate: null argument"};
    if (in->pitch != out->pitch) throw Status{MGG_E_INPUT, "aggregate: in/out width differ"};
    cudaStream_t st = enter(ctx, plan->part);
    run_aggregate(ctx, plan, in, out, opts, st);
  });
}

int mgg_trace_create(mgg_ctx* ctx, uint32_t part, uint64_t capacity, uint32_t warp_limit,
                     mgg_trace** out) {
  return guard([&] {
    if (!out) throw Status{MGG_E_INPUT, "trace_create: null argument"};
    if (capacity == 0 || capacity > 0xffffffffull)
      throw Status{MGG_E_CONFIG, "trace_create: capacity must be in [1, 2^32)"};
    enter(ctx, part);
    auto* t = new mgg_trace();
    t->ctx = ctx;
    t->part = part;
    t->capacity = capacity;
    t->warp_limit = warp_limit;
    if (cudaMalloc(&t->events, capacity * 16) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&t->count), 8) != cudaSuccess) {
      cudaFree(t->events);
      delete t;
      throw Status{MGG_E_CUDA, "trace_create: cudaMalloc failed"};
    }
    MGG_CUDA(cudaMemset(t->count, 0, 8));
    *out = t;
  });
}

int mgg_trace_destroy(mgg_trace* t) {
  if (!t) return MGG_OK;
  cudaSetDevice(t->ctx->device[t->part]);
  cudaFree(t->events);
  cudaFree(t->count);
  delete t;
  return MGG_OK;
}

int mgg_aggregate_traced(mgg_ctx* ctx, const mgg_dplan* plan, const mgg_store* in,
                         mgg_store* out, const mgg_agg_opts* opts, mgg_trace* trace) {
  return guard([&] {
    if (!plan || !in || !out || !trace) throw Status{MGG_E_INPUT, "aggregate_traced: null argument"};
    if (in->pitch != out->pitch) throw Status{MGG_E_INPUT, "aggregate: in/out width differ"};
    if (trace->part != plan->part) throw Status{MGG_E_INPUT, "aggregate_traced: trace of another part"};
    cudaStream_t st = enter(ctx, plan->part);
    MGG_CUDA(cudaMemsetAsync(trace->count, 0, 8, st));
    TraceSink sink{trace->events, trace->count, static_cast<uint32_t>(trace->capacity),
                   trace->warp_limit};
    launch_aggregate(ctx, plan, in, out, opts ? opts->relu_in : 0, opts ? opts->phase : 0,
                     nullptr, st, &sink);
  });
}

int mgg_trace_read(mgg_trace* t, uint64_t* events, uint64_t cap, uint64_t* n,
                   uint64_t* emitted) {
  return guard([&] {
    if (!t || !n) throw Status{MGG_E_INPUT, "trace_read: null argument"};
    cudaStream_t st = enter(t->ctx, t->part);
    MGG_CUDA(cudaStreamSynchronize(st));
    unsigned long long cnt = 0;
    MGG_CUDA(cudaMemcpy(&cnt, t->count, 8, cudaMemcpyDeviceToHost));
    const uint64_t have = std::min<uint64_t>(cnt, t->capacity);
    if (emitted) *emitted = cnt;
    *n = have;
    if (!events || !cap) return;
    const uint64_t m = std::min(have, cap);
    std::vector<uint32_t> raw(4 * m);
    if (m) MGG_CUDA(cudaMemcpy(raw.data(), t->events, m * 16, cudaMemcpyDeviceToHost));
    int clk_khz = 0;
    MGG_CUDA(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, t->ctx->device[t->part]));
    uint64_t t0 = ~0ull;
    for (uint64_t i = 0; i < m; ++i)
      t0 = std::min(t0, uint64_t(raw[4 * i]) | (uint64_t(raw[4 * i + 1]) << 32));
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t ns = (uint64_t(raw[4 * i]) | (uint64_t(raw[4 * i + 1]) << 32)) - t0;
      events[4 * i] = static_cast<uint64_t>(double(ns) * clk_khz * 1e-6);  // SM cycles
      events[4 * i + 1] = raw[4 * i + 2] >> 8;                             // sm
      events[4 * i + 2] = raw[4 * i + 3];                                  // logical warp
      events[4 * i + 3] = raw[4 * i + 2] & 0xff;                           // stage*2+begin
    }
    *n = m;
  });
}

int mgg_halo_pull(mgg_ctx* ctx, const mgg_dplan* plan, const mgg_store* in, float* halo) {
  return guard([&] {
    if (!plan || !in || !halo) throw Status{MGG_E_INPUT, "halo_pull: null argument"};
    cudaStream_t st = enter(ctx, plan->part);
    launch_halo_pull(plan, in, halo, st);
    count_launch(ctx);
  });
}

int mgg_dplan_set_k1_form(mgg_dplan* plan, uint32_t form) {
  if (!plan || form > 3) return MGG_E_INPUT;
  plan->k1_form = form;
  return MGG_OK;
}

int mgg_dplan_k1_kernels(const mgg_dplan* plan, char* buf, size_t cap) {
  if (!plan || !buf || cap == 0) return MGG_E_INPUT;
  const size_t n = std::min(cap - 1, plan->k1_names.size());
  std::memcpy(buf, plan->k1_names.data(), n);
  buf[n] = 0;
  return MGG_OK;
}

int mgg_dplan_k1_launch_info(const mgg_dplan* plan, uint32_t* info) {
  if (!plan || !info) return MGG_E_INPUT;
  info[0] = plan->last_grid;
  info[1] = plan->last_threads;
  info[2] = plan->last_resident;
  info[3] = plan->last_sms;
  return MGG_OK;
}

int mgg_dplan_halo_len(const mgg_dplan* plan, uint64_t* n) {
  if (!plan || !n) return MGG_E_INPUT;
  *n = plan->halo_len;
  return MGG_OK;
}

int mgg_rows_init(mgg_ctx* ctx, uint32_t part, const mgg_store* in, mgg_store* out,
                  float scale, int relu_in) {
  return mgg_rows_init_copy(ctx, part, in, out, scale, relu_in, nullptr);
}

int mgg_rows_init_copy(mgg_ctx* ctx, uint32_t part, const mgg_store* in, mgg_store* out,
                       float scale, int relu_in, mgg_store* copy) {
  return mgg_rows_init_rs(ctx, part, in, out, scale, relu_in, copy, nullptr);
}

int mgg_rows_softmax_rs(mgg_ctx* ctx, uint32_t part, const mgg_store* in, mgg_store* out,
                        const mgg_dbuf* row_scale) {
  return guard([&] {
    if (!in || !out) throw Status{MGG_E_INPUT, "rows_softmax: null store"};
    if (in->pitch != out->pitch) throw Status{MGG_E_INPUT, "rows_softmax: in/out width differ"};
    cudaStream_t st = enter(ctx, part);
    launch_softmax(in->shard[part], out->shard[part], in->rows(part), in->pitch, in->dim, st,
                   row_scale ? static_cast<const float*>(row_scale->ptr) : nullptr);
    count_launch(ctx);
  });
}

int mgg_rows_init_rs(mgg_ctx* ctx, uint32_t part, const mgg_store* in, mgg_store* out,
                     float scale, int relu_in, mgg_store* copy, const mgg_dbuf* row_scale) {
  return guard([&] {
    if (!in || !out) throw Status{MGG_E_INPUT, "rows_init: null store"};
    if (in->pitch != out->pitch || (copy && copy->pitch != in->pitch))
      throw Status{MGG_E_INPUT, "rows_init: in/out width differ"};
    cudaStream_t st = enter(ctx, part);
    launch_rows_init(in->shard[part], out->shard[part], in->rows(part), in->pitch, scale,
                     relu_in, copy ? copy->shard[part] : nullptr, st,
                     row_scale ? static_cast<const float*>(row_scale->ptr) : nullptr);
    count_launch(ctx);
  });
}

int mgg_dense(mgg_ctx* ctx, uint32_t part, const mgg_store* in, const mgg_dense_desc* d,
              mgg_store* out, mgg_store* out2) {
  return guard([&] {
    if (!in || !d || !out || !d->w) throw Status{MGG_E_INPUT, "dense: null argument"};
    if (out2 && out2->pitch != out->pitch) throw Status{MGG_E_INPUT, "dense: out2 width differs"};
    cudaStream_t st = enter(ctx, part);
    const float* bias = d->bias ? static_cast<const float*>(d->bias->ptr) : nullptr;
    const float* pre_bias = d->pre_bias ? static_cast<const float*>(d->pre_bias->ptr) : nullptr;
    const float* rs = d->row_scale ? static_cast<const float*>(d->row_scale->ptr) : nullptr;
    static const bool force_simt = [] {
      const char* e = std::getenv("MGG_GEMM");
      return e && std::string(e) == "simt";
    }();
    if (!force_simt && gemm_tc_supported(in->dim, out->dim)) {
      const float* wt = gemm_tc_prepare(const_cast<mgg_dbuf*>(d->w), in->dim, out->dim, st);
      launch_dense_tc(in->shard[part], in->pitch, in->dim, in->rows(part), wt, bias, pre_bias,
                      out->dim, d->pre, d->act, out->shard[part], out->pitch,
                      out2 ? out2->shard[part] : nullptr, d->out2_scale, st, rs);
      count_launch(ctx);
      return;
    }
    launch_dense(in->shard[part], in->pitch, in->dim, in->rows(part),
                 static_cast<const float*>(d->w->ptr), bias, pre_bias, out->dim, d->pre, d->act,
                 out->shard[part], out->pitch, out2 ? out2->shard[part] : nullptr,
                 d->out2_scale, st, rs);
    count_launch(ctx, (out->dim + 63) / 64);
  });
}

int mgg_dense_chain_supported(uint32_t k, uint32_t m1, uint32_t m) {
  return gemm_tc_chain_supported(k, m1, m) ? 1 : 0;
}

int mgg_dense_chain(mgg_ctx* ctx, uint32_t part, const mgg_store* in, const mgg_dense_desc* d1,
                    uint32_t m1, const mgg_dense_desc* d2, mgg_store* out, mgg_store* out2) {
  return guard([&] {
    if (!in || !d1 || !d2 || !out || !d1->w || !d2->w)
      throw Status{MGG_E_INPUT, "dense_chain: null argument"};
    if (out2 && out2->pitch != out->pitch) throw Status{MGG_E_INPUT, "dense_chain: out2 width differs"};
    if (!gemm_tc_chain_supported(in->dim, m1, out->dim))
      throw Status{MGG_E_CONFIG, "dense_chain: unsupported widths"};
    if (d2->bias || d2->pre != 1 || d2->act != 0 || d1->act != 0)
      throw Status{MGG_E_CONFIG, "dense_chain: second GEMM must be ReLU-in, no bias, no act"};
    cudaStream_t st = enter(ctx, part);
    const float* w1 = gemm_tc_prepare(const_cast<mgg_dbuf*>(d1->w), in->dim, m1, st);
    const float* w2 = gemm_tc_prepare(const_cast<mgg_dbuf*>(d2->w), m1, out->dim, st);
    const float* b1 = d1->bias ? static_cast<const float*>(d1->bias->ptr) : nullptr;
    const float* pb = d1->pre_bias ? static_cast<const float*>(d1->pre_bias->ptr) : nullptr;
    launch_dense_tc_chain(in->shard[part], in->pitch, in->dim, in->rows(part), w1, b1, m1, pb,
                          d1->pre, w2, out->dim, out->shard[part], out->pitch,
                          out2 ? out2->shard[part] : nullptr, d2->out2_scale, st);
    count_launch(ctx);
  });
}

int mgg_rows_softmax(mgg_ctx* ctx, uint32_t part, const mgg_store* in, mgg_store* out) {
  return guard([&] {
    if (in->pitch != out->pitch) throw Status{MGG_E_INPUT, "rows_softmax: in/out width differ"};
    cudaStream_t st = enter(ctx, part);
    launch_softmax(in->shard[part], out->shard[part], in->rows(part), in->pitch, in->dim, st);
    count_launch(ctx);
  });
}

// Barrier mode: 0 = events where possible (default), 1 = the K3 flag kernel
// for every context with a flags store, also same-process parts (validation:
// MGG_BARRIER=k3 exercises the cross-process kernel on a one-GPU box).
static int barrier_mode() {
  static const int m = [] {
    const char* e = std::getenv("MGG_BARRIER");
    return e && std::string(e) == "k3" ? 1 : 0;
  }();
  return m;
}

int mgg_barrier(mgg_ctx* ctx, mgg_store* flags) {
  return guard([&] {
    const bool k3 = !ctx->all_local || (barrier_mode() == 1 && flags && ctx->num_parts > 1);
    if (!k3) {
      // every part is driven by this process (one device or several): each
      // part's stream waits for every other part's tail through events —
      // cudaStreamWaitEvent orders streams across devices too, so there is
      // no host round trip and the join is capturable into a CUDA graph
      if (ctx->single_device && !ctx->part_streams) return;  // one stream: stream order
      for (uint32_t p = 0; p < ctx->num_parts; ++p) {
        enter(ctx, p);
        MGG_CUDA(cudaEventRecord(ctx->bar_ev[p], ctx->stream[p]));
      }
      for (uint32_t p = 0; p < ctx->num_parts; ++p) {
        enter(ctx, p);
        for (uint32_t q = 0; q < ctx->num_parts; ++q)
          if (q != p && ctx->stream[q] != ctx->stream[p])
            MGG_CUDA(cudaStreamWaitEvent(ctx->stream[p], ctx->bar_ev[q], 0));
      }
      return;
    }
    // K3: some parts live in other processes — device-side flags over the
    // peer-mapped flag store, release/acquire at system scope
    if (!flags) throw Status{MGG_E_INPUT, "barrier: flags store required"};
    if (flags->dim < ctx->num_parts + 1)
      throw Status{MGG_E_INPUT, "barrier: flags store needs num_parts + 1 columns"};
    for (uint32_t p = 0; p < ctx->num_parts; ++p)
      if (flags->lb[p + 1] - flags->lb[p] != 1)
        throw Status{MGG_E_INPUT, "barrier: flags store must hold one row per part"};
    for (uint32_t p = 0; p < ctx->num_parts; ++p) {
      if (ctx->device[p] < 0) continue;
      cudaStream_t st = enter(ctx, p);
      launch_barrier(reinterpret_cast<unsigned* const*>(const_cast<float**>(flags->dtable[p])),
                     reinterpret_cast<unsigned*>(flags->shard[p]), p, ctx->num_parts, st);
      count_launch(ctx);
    }
  });
}

int mgg_time_aggregate(mgg_ctx* ctx, const mgg_dplan* plan, const mgg_store* in,
                       mgg_store* out, const mgg_agg_opts* opts, uint32_t reps,
                       uint64_t* median_ns) {
  return guard([&] {
    cudaStream_t st = enter(ctx, plan->part);
    reps = std::max(reps, 1u);
    std::vector<float> ms(reps);
    bool paged = false;
    for (uint32_t q = 0; q < ctx->num_parts; ++q)
      paged |= in->owned[q] && (in->mem[q] == MGG_MEM_MANAGED || in->mem[q] == MGG_MEM_MANAGED_HOST);
    run_aggregate(ctx, plan, in, out, opts, st);
    for (uint32_t r = 0; r < reps; ++r) {
      if (paged) {  // every rep starts with the pages at home (outside the window)
        rehome(const_cast<mgg_store*>(in), st);
        MGG_CUDA(cudaSetDevice(ctx->device[plan->part]));
      }
      MGG_CUDA(cudaEventRecord(ctx->ev0[plan->part], st));
      run_aggregate(ctx, plan, in, out, opts, st);
      MGG_CUDA(cudaEventRecord(ctx->ev1[plan->part], st));
      MGG_CUDA(cudaEventSynchronize(ctx->ev1[plan->part]));
      MGG_CUDA(cudaEventElapsedTime(&ms[r], ctx->ev0[plan->part], ctx->ev1[plan->part]));
    }
    std::sort(ms.begin(), ms.end());
    *median_ns = static_cast<uint64_t>(ms[reps / 2] * 1e6);
  });
}

}  // extern "C"
