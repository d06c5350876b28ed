// K1 — MGG pipelined neighbor aggregation for sm_100a.
//
// Work geometry is the plan's, unchanged: logical CTA = wpb warps, logical
// warp w owns partitions [w·dist, (w+1)·dist) of the local list and of the
// remote list (interleaved mapping, R:proj/src/workload.cpp:103-124), or the
// local groups then the remote groups (segregated, 126-146); partitions hold
// <= ps neighbors. The kernel is persistent: a resident CTA of wpb warps
// walks a contiguous chunk of logical CTAs (grid = SMs x occupancy), so the
// millions of logical CTAs cost no launch/scheduling overhead and a physical
// warp can keep one target's partial sum in registers across consecutive
// logical warps.
//
// Per logical warp the pair loop follows the reference's async discipline
// (R:proj/src/sim.cpp:102-125, paper Fig. 6b):
//   pair i:  issue the remote-row loads of R_i   (peer shard over NVLink)
//            reduce local partition L_i          (own shard, HBM/L2)
//            consume R_i                          (registers)
// so R_i's NVLink latency hides under L_i's local work inside one kernel,
// with no host round trip and no NCCL call.
//
// Memory access: a warp loads the (target, begin) records of its dist
// partitions with one coalesced 64-bit load, then each partition's <= 32
// column ids with one coalesced 32-bit load, and distributes both by
// shuffles. Rows are gathered with 128-bit loads, VEC (power of two >= row
// float4s) lanes per row, RPW = 32/VEC rows per step, up to 4 steps in
// flight per lane. A target's partials fold across the RPW row groups with
// xor-shuffles and land in `out` with one 128-bit vector reduction
// (REDG.ADD.F32x4) per lane, only when the warp's target changes.
//
// Group-per-partition forms (agg_group local-only, agg_gpair paired): the
// same plan geometry, but each VEC-lane group of a warp walks its own
// partitions (pairs) with 4-8 rows in flight, so short partitions keep
// 32/VEC gather streams per warp busy. The launcher picks the form per
// launch from the plan's shape (pick_lean / pick_pair below).
#include <cuda_runtime.h>

#include <cxxabi.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

// Row-load flavour (A/B builds): 0 __ldg, 1 L1::no_allocate, 2 .cg (L2
// only), 3 L1::evict_first. Measured (profiles/r01_k1_experiments.md): .cg
// equals __ldg on L2-resident tables and is 3.6% faster on the HBM-resident
// GIN table; the L1 qualifiers are 30-40% slower.
#ifndef MGG_LD_MODE
#define MGG_LD_MODE 2
#endif
#if MGG_LD_MODE == 1
#define MGG_LD_INSN "ld.global.nc.L1::no_allocate.v4.f32"
#elif MGG_LD_MODE == 2
#define MGG_LD_INSN "ld.global.cg.v4.f32"
#elif MGG_LD_MODE == 3
#define MGG_LD_INSN "ld.global.nc.L1::evict_first.v4.f32"
#endif

#ifndef MGG_AGG_PF
#define MGG_AGG_PF 4
#endif

#ifndef MGG_AGG_UNROLL
#define MGG_AGG_UNROLL 4
#endif

namespace mgg::dev {
namespace {

struct AggArgs {
  const int2* lmeta;
  const uint32_t* lcols;
  const int2* rmeta;
  const uint32_t* rcols;
  const float* const* table;  // per-owner shard base (device array)
  const float* own;           // this part's gather shard
  float* out;                 // this part's accumulator shard
  uint32_t nL, nR;
  uint32_t pitch;             // floats per row (multiple of 4)
  uint32_t vec;               // float4 per row = pitch / 4
  uint32_t dist, wpb;
  uint32_t mapping;           // 0 interleaved, 1 segregated
  uint32_t local_warps;       // segregated: warps holding local groups
  uint32_t num_warps;         // logical warps
  uint32_t num_lblocks;       // logical CTAs = ceil(num_warps / wpb)
  uint32_t num_owners;
  int phase;                  // 0 all, 1 local only, 2 remote only
  // pair kernels: logical CTAs dealt round-robin over the resident CTAs (1)
  // instead of contiguous chunks (0)
  uint32_t strided;
  // pair kernels, dynamic schedule: resident warps take tickets of `wchunk`
  // consecutive logical warps from sched[0] (null = the static schedule)
  uint32_t* sched;
  uint32_t wchunk;
  const float* halo;          // deduplicated remote rows (halo mode) or null
  // halo pull fused into a local-only group pass (halo mode): copy the
  // plan's pull_n distinct remote rows (packed owner|offset in pull_rows)
  // from the owners' shards (`table`) into pull_dst, a proportional slice
  // per logical warp interleaved with its partitions (HaloPull below)
  const uint32_t* pull_rows;
  uint64_t pull_n;
  float* pull_dst;
  // device event trace (traced launches only): 16-B records
  // {globaltimer lo, hi, (smid << 8) | (stage << 1) | begin, logical warp}
  uint4* trace;
  unsigned long long* trace_n;
  uint32_t trace_cap, trace_warps;  // capacity; only warps < trace_warps record
};

constexpr uint32_t kShift = 28;
constexpr uint32_t kMask = (1u << kShift) - 1;
constexpr unsigned kFull = 0xffffffffu;

// Two packed FADD2 (add.rn.f32x2, sm_100+): per-element IEEE round-to-
// nearest adds, bit-identical to four FADDs at half the issue slots.
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  float4 r;
  asm("{\n\t.reg .b64 a0, a1, b0, b1, d0, d1;\n\t"
      "mov.b64 a0, {%4, %5};\n\tmov.b64 a1, {%6, %7};\n\t"
      "mov.b64 b0, {%8, %9};\n\tmov.b64 b1, {%10, %11};\n\t"
      "add.rn.f32x2 d0, a0, b0;\n\tadd.rn.f32x2 d1, a1, b1;\n\t"
      "mov.b64 {%0, %1}, d0;\n\tmov.b64 {%2, %3}, d1;\n\t}"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w));
  return r;
}
__device__ __forceinline__ float4 f4zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ float4 f4relu(float4 a) {
  return make_float4(fmaxf(a.x, 0.f), fmaxf(a.y, 0.f), fmaxf(a.z, 0.f), fmaxf(a.w, 0.f));
}
// Read-only path. (An explicit ld.global.nc.L1::no_allocate asm was 45%
// slower: the volatile asm pins the loads in program order and the compiler
// can no longer batch the 4 steps' loads ahead of their shuffles.)
__device__ __forceinline__ float4 ld_row4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void red_add4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
// Stage codes of the reference's TraceEvent (R:proj/include/pipeshard/sim.hpp:71,
// names R:proj/src/sim.cpp:627): LR remote get, LL local load, AC accumulate.
enum : uint32_t { kLR = 0, kLL = 1, kAC = 2 };

// Global-timer stamp ordered after `dep` is available (a fake operand: the
// read cannot issue before the loads feeding `dep` have landed).
__device__ __forceinline__ uint64_t stamp_after(float dep) {
  uint64_t t;
  asm volatile("{\n\t.reg .f32 d;\n\tmov.f32 d, %1;\n\tmov.u64 %0, %%globaltimer;\n\t}"
               : "=l"(t)
               : "f"(dep)
               : "memory");
  return t;
}
__device__ __forceinline__ void trace_emit(const AggArgs& a, uint32_t w, uint32_t stage,
                                           bool begin, uint64_t t) {
  if ((threadIdx.x & 31) != 0 || w >= a.trace_warps) return;
  const unsigned long long i = atomicAdd(a.trace_n, 1ull);
  if (i >= a.trace_cap) return;
  uint32_t sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  a.trace[i] = make_uint4(static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32),
                          (sm << 8) | (stage << 1) | (begin ? 1u : 0u), w);
}

// Group form (agg_gpair): the group's first lane records, id = w * groups + group.
__device__ __forceinline__ void trace_emit_g(const AggArgs& a, uint32_t w, uint32_t id,
                                             bool leader, uint32_t stage, bool begin,
                                             uint64_t t) {
  if (!leader || w >= a.trace_warps) return;
  const unsigned long long i = atomicAdd(a.trace_n, 1ull);
  if (i >= a.trace_cap) return;
  uint32_t sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  a.trace[i] = make_uint4(static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32),
                          (sm << 8) | (stage << 1) | (begin ? 1u : 0u), id);
}

__device__ __forceinline__ const float* shfl_ptr(const float* p, int src) {
  const unsigned long long v = reinterpret_cast<unsigned long long>(p);
  return reinterpret_cast<const float*>(__shfl_sync(kFull, v, src));
}

// Warp-uniform ranges [l0,l1) of local and [r0,r1) of remote partitions.
__device__ __forceinline__ void warp_groups(const AggArgs& a, uint32_t w, uint32_t& l0,
                                            uint32_t& l1, uint32_t& r0, uint32_t& r1) {
  if (a.mapping == 0) {
    l0 = r0 = w * a.dist;
    l1 = min(l0 + a.dist, a.nL);
    r1 = min(r0 + a.dist, a.nR);
  } else if (w < a.local_warps) {
    l0 = w * a.dist;
    l1 = min(l0 + a.dist, a.nL);
    r0 = r1 = 0;
  } else {
    l0 = l1 = 0;
    r0 = (w - a.local_warps) * a.dist;
    r1 = min(r0 + a.dist, a.nR);
  }
  if (l1 < l0) l1 = l0;
  if (r1 < r0) r1 = r0;
  if (a.phase == 2) l1 = l0;
  if (a.phase == 1) r1 = r0;
}

// Contiguous chunk of logical CTAs owned by this resident CTA.
__device__ __forceinline__ void cta_chunk(uint32_t total, uint32_t& b0, uint32_t& b1) {
  const uint32_t per = (total + gridDim.x - 1) / gridDim.x;
  b0 = min(blockIdx.x * per, total);
  b1 = min(b0 + per, total);
}
// Logical CTAs of this resident CTA: chunks of `chunk` consecutive logical
// CTAs dealt round-robin over the resident CTAs (a.strided = chunk size;
// 0 = one contiguous chunk per resident CTA). Round-robin is the reference's
// in-order block dispatch over the SMs: the interleaved mapping packs the
// shorter kind's partitions into the FIRST logical warps (w·dist, ...), and
// contiguous chunks would hand all of them to a few resident CTAs; chunks of
// a few logical CTAs keep the metadata streams sequential.
struct LbRange {
  uint32_t first, end, chunk, jump;
  __device__ __forceinline__ uint32_t next(uint32_t lb) const {
    ++lb;
    return lb % chunk ? lb : lb + jump;
  }
};
__device__ __forceinline__ LbRange lb_range(const AggArgs& a) {
  if (a.strided) {
    const uint32_t c = a.strided;
    return {blockIdx.x * c, a.num_lblocks, c, (gridDim.x - 1) * c};
  }
  const uint32_t per = max((a.num_lblocks + gridDim.x - 1) / gridDim.x, 1u);
  const uint32_t b0 = min(blockIdx.x * per, a.num_lblocks);
  return {b0, min(b0 + per, a.num_lblocks), per, a.num_lblocks};  // one chunk, then past the end
}

// Logical warps of this resident warp under the dynamic schedule. The
// static schedule deals every resident CTA a fixed share of logical CTAs up
// front, so a CTA whose warps stall on remote rows finishes its local share
// late; here warps take tickets as they go.
// * A ticket g is a chunk of a.wchunk consecutive logical warps, dealt in a
//   block-strided order: chunk = (g % kBlocks) * L + g / kBlocks with
//   L = ceil(chunks / kBlocks) (kBlocks = 512). Consecutive tickets sweep kBlocks evenly
//   spaced positions of the warp range, so any contiguous region — the
//   interleaved mapping puts every (local, remote) pair in the first
//   logical warps when one kind is scarce — is spread over the whole launch:
//   a bounded share of the resident warps works pairs at any time (enough to
//   keep the remote link busy) while the rest reduce local partitions.
// * One counter would serialise (~3 ns per same-address atomic at L2), so
//   tickets are dealt over kShards counters 128 B apart (ticket t of shard s
//   is g = t * kShards + s); a warp starts on shard (global warp id %
//   kShards) and moves on when it runs dry — shards only ever run dry, so one
//   pass over them finds all remaining work.
// * The next ticket is requested before the current chunk is worked (its
//   atomic round trip overlaps the chunk).
// Each resident warp retires once; the last one resets the counters for the
// next launch on the plan (stream order makes that visible).
constexpr uint32_t kShards = MGG_KSHARDS;  // common.cuh
constexpr uint32_t kShardStride = 32;  // u32 words between counters (128 B)
// 512 positions (profiles/r02/dyn_schedule.md, kBlocks sweep): slow-peer
// hidden remote 0.79-0.85 at 32 -> 0.92-0.95 at 512 (0.92-0.99 at 2048, with
// a 2-3% slower local leg), same-device launch unchanged
#ifndef MGG_KBLOCKS
#define MGG_KBLOCKS 512
#endif
constexpr uint32_t kBlocks = MGG_KBLOCKS;

// KINDS = 2 (agg_gsplit): every chunk is two items, its local and its remote
// partitions, adjacent in the dealing order; run_warp(w, kind).
template <int KINDS, class F>
__device__ __forceinline__ void for_each_ticket(const AggArgs& a, F&& run_warp) {
  const int lane = threadIdx.x & 31;
  const uint32_t wc = a.wchunk;
  const uint32_t chunks = (a.num_warps + wc - 1) / wc * KINDS;  // items
  const uint32_t L = (chunks + kBlocks - 1) / kBlocks;
  const uint32_t tickets = L * kBlocks;
  auto shard_len = [&](uint32_t s) { return tickets > s ? (tickets - s + kShards - 1) / kShards : 0u; };
  auto ctr = [&](uint32_t s) { return a.sched + s * kShardStride; };
  uint32_t s = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % kShards;
  auto grab = [&]() -> uint32_t {  // lane 0: a ticket from shard s onwards
    for (uint32_t k = 0; k < kShards; ++k) {
      const uint32_t lim = shard_len(s);
      if (*reinterpret_cast<volatile uint32_t*>(ctr(s)) < lim) {
        const uint32_t t = atomicAdd(ctr(s), 1u);
        if (t < lim) return t * kShards + s;
      }
      s = s + 1 == kShards ? 0 : s + 1;
    }
    return 0xffffffffu;
  };
  uint32_t g = 0;
  if (lane == 0) g = grab();
  g = __shfl_sync(kFull, g, 0);
  while (g != 0xffffffffu) {
    uint32_t tn = 0;
    if (lane == 0) tn = atomicAdd(ctr(s), 1u);  // speculative: checked after the chunk
    const uint32_t c = (g % kBlocks) * L + g / kBlocks;  // >= chunks: an empty ticket
    if (c < chunks) {
      const uint32_t w0 = c / KINDS * wc;
      const uint32_t w1 = min(w0 + wc, a.num_warps);
      for (uint32_t w = w0; w < w1; ++w) run_warp(w, c % KINDS);
    }
    if (lane == 0) {
      if (tn < shard_len(s)) {
        g = tn * kShards + s;
      } else {
        s = s + 1 == kShards ? 0 : s + 1;
        g = grab();
      }
    }
    g = __shfl_sync(kFull, g, 0);
  }
  if (lane == 0) {
    __threadfence();  // this warp's last ticket is ordered before it retires
    uint32_t* retired = a.sched + kShards * kShardStride;
    const uint32_t total = gridDim.x * (blockDim.x >> 5);
    if (atomicAdd(retired, 1u) == total - 1) {
      for (uint32_t k = 0; k < kShards; ++k) atomicExch(ctr(k), 0u);
      atomicExch(retired, 0u);
    }
  }
}

template <int VEC, bool RELU>
struct Lanes {
  static constexpr int RPW = 32 / VEC;  // rows per warp step
  static constexpr int PF = MGG_AGG_PF;  // remote steps staged ahead
  int lane, sub, v;
  bool vlane;
  uint32_t voff;       // byte offset of this lane's float4 in a row
  uint32_t pb;         // row pitch in bytes
  const char* lbase;   // own shard + voff

  // Lanes past the row width (v >= vec) re-read the row's first float4
  // instead of predicating: their sums never leave the warp (flush skips
  // them), and every load stays unpredicated.
  __device__ __forceinline__ Lanes(const AggArgs& a) {
    lane = threadIdx.x & 31;
    sub = lane / VEC;
    v = lane % VEC;
    vlane = v < static_cast<int>(a.vec);
    voff = vlane ? 16u * v : 0u;
    pb = a.pitch * 4u;
    lbase = reinterpret_cast<const char*>(a.own) + voff;
    // opaque to the optimizer: otherwise it re-associates own + voff + c*pb
    // into a per-row 64-bit add
    asm("mov.b64 %0, %0;" : "+l"(lbase));
  }

  // `off` is a row offset: device-side local columns carry no owner bits
  // (stripped at plan upload), remote columns are masked by the caller.
  __device__ __forceinline__ float4 load(const char* base, uint32_t off) const {
    const char* p = base + static_cast<size_t>(off) * pb;
#if MGG_LD_MODE == 0
    float4 x = __ldg(reinterpret_cast<const float4*>(p));
#else
    float4 x;
    // non-volatile: the compiler may still batch these ahead of their uses
    asm(MGG_LD_INSN " {%0,%1,%2,%3}, [%4];"
        : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
        : "l"(p));
#endif
    if (RELU) x = f4relu(x);
    return x;
  }

  // Row `r` (< n) of the current column window; base from the lane table for
  // remote rows (peer shards), own shard otherwise.
  template <bool REMOTE>
  __device__ __forceinline__ float4 row(const AggArgs& a, uint32_t colwin, int r, int n,
                                        const float* tab_lane) const {
    const uint32_t c = __shfl_sync(kFull, colwin, r & 31);
    const char* base = lbase;
    if (REMOTE)
      base = reinterpret_cast<const char*>(
                 a.halo ? a.halo : shfl_ptr(tab_lane, static_cast<int>(c >> kShift))) +
             voff;
    float4 x = f4zero();
    if (r < n) x = load(base, REMOTE ? (c & kMask) : c);
    return x;
  }

  // Sum rows [s0*RPW, n) of the window into acc, UNR steps of loads in flight
  // (a 32-column window has 32/RPW steps: 4 at VEC=4, 16 at VEC=16).
  static constexpr int UNR = MGG_AGG_UNROLL < (32 / RPW) ? MGG_AGG_UNROLL : (32 / RPW);
  template <bool REMOTE>
  __device__ __forceinline__ float4 window(const AggArgs& a, uint32_t colwin, int n, int s0,
                                           float4 acc, const float* tab_lane) const {
    if (!REMOTE && s0 == 0 && n % (RPW * UNR) == 0) {
      // whole step groups (every full ps=32 window): no predicates at all —
      // per row a shuffle, a mask, one IMAD.WIDE, the load and two FADD2
      for (int s = 0; s < n / RPW; s += UNR) {
        float4 t[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          t[u] = load(lbase, __shfl_sync(kFull, colwin, (s + u) * RPW + sub));
#pragma unroll
        for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
      }
      return acc;
    }
    const int steps = (n + RPW - 1) / RPW;
    for (int s = s0; s < steps; s += UNR) {
      float4 t[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        t[u] = row<REMOTE>(a, colwin, (s + u) * RPW + sub, (s + u) < steps ? n : 0, tab_lane);
#pragma unroll
      for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
    }
    return acc;
  }

  __device__ __forceinline__ void flush(const AggArgs& a, float4 acc, int target) const {
#pragma unroll
    for (int off = 16; off >= VEC; off >>= 1) {
      acc.x += __shfl_xor_sync(kFull, acc.x, off);
      acc.y += __shfl_xor_sync(kFull, acc.y, off);
      acc.z += __shfl_xor_sync(kFull, acc.z, off);
      acc.w += __shfl_xor_sync(kFull, acc.w, off);
    }
    if (sub == 0 && vlane) red_add4(a.out + static_cast<size_t>(target) * a.pitch + 4 * v, acc);
  }
};

__device__ __forceinline__ uint32_t load_colwin(const uint32_t* cols, int beg, int n) {
  const int lane = threadIdx.x & 31;
  return lane < n ? __ldg(cols + beg + lane) : 0u;
}

// Partition records of logical warp w (dist+1 <= 17 entries, one coalesced
// 64-bit load per kind).
struct WarpMeta {
  int2 ml, mr;
  int nl, nr;
};

__device__ __forceinline__ WarpMeta load_warp_meta(const AggArgs& a, uint32_t w, bool remote) {
  WarpMeta m{make_int2(0, 0), make_int2(0, 0), 0, 0};
  if (w >= a.num_warps) return m;
  const int lane = threadIdx.x & 31;
  uint32_t l0, l1, r0, r1;
  warp_groups(a, w, l0, l1, r0, r1);
  m.nl = static_cast<int>(l1 - l0);
  m.nr = static_cast<int>(r1 - r0);
  if (lane <= m.nl && m.nl > 0) m.ml = __ldg(a.lmeta + l0 + lane);
  if (remote && lane <= m.nr && m.nr > 0) m.mr = __ldg(a.rmeta + r0 + lane);
  return m;
}

template <int VEC, bool RELU, bool REMOTE, int MINB, bool TRACE = false>
__global__ void __launch_bounds__(512, MINB) agg_kernel(AggArgs a) {
  using L = Lanes<VEC, RELU>;
  const L ln(a);
  const int lane = ln.lane;
  const float* tab_lane = nullptr;
  if (REMOTE && lane < static_cast<int>(a.num_owners)) tab_lane = a.table[lane];

  float4 accL = f4zero(), accR = f4zero();
  int curL = -1, curR = -1;
  uint32_t b0, b1;
  cta_chunk(a.num_lblocks, b0, b1);
  const uint32_t wib = threadIdx.x >> 5;
  // software pipeline: records of the next logical warp and the column
  // window of the next local partition are always one step ahead
  WarpMeta next = load_warp_meta(a, b0 * a.wpb + wib, REMOTE);

  for (uint32_t lb = b0; lb < b1; ++lb) {
    const uint32_t w = lb * a.wpb + wib;
    if (w >= a.num_warps) break;
    const WarpMeta cur = next;
    next = load_warp_meta(a, (lb + 1 < b1) ? w + a.wpb : a.num_warps, REMOTE);
    const int nl = cur.nl, nr = cur.nr;
    const int2 ml = cur.ml, mr = cur.mr;
    const int pairs = max(nl, nr);
    uint32_t lwin = 0;
    if (nl > 0) {
      const int b = __shfl_sync(kFull, ml.y, 0);
      lwin = load_colwin(a.lcols, b, min(__shfl_sync(kFull, ml.y, 1) - b, 32));
    }

    for (int i = 0; i < pairs; ++i) {
      // (1) issue R_i: column window + first PF steps of peer rows
      int rt = -1, rbeg = 0, rend = 0, rn = 0;
      uint32_t rwin = 0;
      float4 pre[L::PF];
      if (REMOTE && i < nr) {
        rt = __shfl_sync(kFull, mr.x, i);
        rbeg = __shfl_sync(kFull, mr.y, i);
        rend = __shfl_sync(kFull, mr.y, i + 1);
        rn = min(rend - rbeg, 32);
        rwin = load_colwin(a.rcols, rbeg, rn);
        if (TRACE) trace_emit(a, w, kLR, true, stamp_after(0.f));
#pragma unroll
        for (int s = 0; s < L::PF; ++s)
          pre[s] = ln.template row<true>(a, rwin, s * L::RPW + ln.sub, rn, tab_lane);
      }
      // (2) reduce L_i while R_i's rows are in flight
      if (i < nl) {
        const int lt = __shfl_sync(kFull, ml.x, i);
        const int beg = __shfl_sync(kFull, ml.y, i);
        const int end = __shfl_sync(kFull, ml.y, i + 1);
        // prefetch the next partition's column window before gathering
        uint32_t lnext = 0;
        if (i + 1 < nl) {
          const int e2 = __shfl_sync(kFull, ml.y, i + 2);
          lnext = load_colwin(a.lcols, end, min(e2 - end, 32));
        }
        if (lt != curL) {
          if (curL >= 0) ln.flush(a, accL, curL);
          accL = f4zero();
          curL = lt;
        }
        if (TRACE) trace_emit(a, w, kLL, true, stamp_after(accL.x));
        accL = ln.template window<false>(a, lwin, min(end - beg, 32), 0, accL, nullptr);
        for (int b = beg + 32; b < end; b += 32) {  // whole-list tails
          const int n = min(end - b, 32);
          accL = ln.template window<false>(a, load_colwin(a.lcols, b, n), n, 0, accL, nullptr);
        }
        if (TRACE) trace_emit(a, w, kLL, false, stamp_after(accL.x));
        lwin = lnext;
      }
      // (3) consume R_i
      if (REMOTE && i < nr) {
        if (rt != curR) {
          if (curR >= 0) ln.flush(a, accR, curR);
          accR = f4zero();
          curR = rt;
        }
        if (TRACE) {  // R_i's staged rows have arrived: the get ends, AC starts
          const uint64_t t = stamp_after(pre[L::PF - 1].x);
          trace_emit(a, w, kLR, false, t);
          trace_emit(a, w, kAC, true, t);
        }
#pragma unroll
        for (int s = 0; s < L::PF; ++s) accR = f4add(accR, pre[s]);
        accR = ln.template window<true>(a, rwin, rn, L::PF, accR, tab_lane);
        for (int beg = rbeg + 32; beg < rend; beg += 32) {  // whole-list tails
          const int n = min(rend - beg, 32);
          accR = ln.template window<true>(a, load_colwin(a.rcols, beg, n), n, 0, accR, tab_lane);
        }
        if (TRACE) trace_emit(a, w, kAC, false, stamp_after(accR.x));
      }
    }
  }
  if (curL >= 0) ln.flush(a, accL, curL);
  if (REMOTE && curR >= 0) ln.flush(a, accR, curR);
}

// Rows wider than 128 floats (vec > 32 float4): lanes own float4 columns
// lane, lane+32, ...; a partition's rows are walked one by one.
template <bool RELU>
__global__ void __launch_bounds__(512) agg_wide(AggArgs a) {
  const int lane = threadIdx.x & 31;
  constexpr int CH = 4;
  uint32_t b0, b1;
  cta_chunk(a.num_lblocks, b0, b1);
  const uint32_t wib = threadIdx.x >> 5;
  for (uint32_t lb = b0; lb < b1; ++lb) {
    const uint32_t w = lb * a.wpb + wib;
    if (w >= a.num_warps) break;
    uint32_t l0, l1, r0, r1;
    warp_groups(a, w, l0, l1, r0, r1);
    for (uint32_t c0 = 0; c0 < a.vec; c0 += 32 * CH) {
      for (int kind = 0; kind < 2; ++kind) {
        const bool remote = kind == 1;
        const uint32_t b = remote ? r0 : l0, cnt = remote ? r1 - r0 : l1 - l0;
        const int2* meta = remote ? a.rmeta : a.lmeta;
        const uint32_t* cols = remote ? a.rcols : a.lcols;
        float4 acc[CH];
        int cur = -1;
        for (uint32_t i = 0; i < cnt; ++i) {
          const int2 m0 = __ldg(meta + b + i);
          const int end = __ldg(meta + b + i + 1).y;
          if (m0.x != cur) {
            if (cur >= 0)
#pragma unroll
              for (int j = 0; j < CH; ++j) {
                const uint32_t col = c0 + lane + 32 * j;
                if (col < a.vec) red_add4(a.out + (size_t)cur * a.pitch + 4 * col, acc[j]);
              }
#pragma unroll
            for (int j = 0; j < CH; ++j) acc[j] = f4zero();
            cur = m0.x;
          }
          for (int k = m0.y; k < end; ++k) {
            const uint32_t c = __ldg(cols + k);
            const float* row =
                (remote ? (a.halo ? a.halo : a.table[c >> kShift]) : a.own) +
                (size_t)(c & kMask) * a.pitch;
#pragma unroll
            for (int j = 0; j < CH; ++j) {
              const uint32_t col = c0 + lane + 32 * j;
              if (col < a.vec) {
                float4 x = ld_row4(row + 4 * col);
                if (RELU) x = f4relu(x);
                acc[j] = f4add(acc[j], x);
              }
            }
          }
        }
        if (cur >= 0)
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const uint32_t col = c0 + lane + 32 * j;
            if (col < a.vec) red_add4(a.out + (size_t)cur * a.pitch + 4 * col, acc[j]);
          }
      }
    }
  }
}

using KernelFn = void (*)(AggArgs);

// MINB = CTAs of 512 threads that must fit per SM (register cap 128/MINB).
template <bool RELU, bool REMOTE, int MINB>
KernelFn pick_minb(uint32_t v) {
  if (v <= 1) return agg_kernel<1, RELU, REMOTE, MINB>;
  if (v <= 2) return agg_kernel<2, RELU, REMOTE, MINB>;
  if (v <= 4) return agg_kernel<4, RELU, REMOTE, MINB>;
  if (v <= 8) return agg_kernel<8, RELU, REMOTE, MINB>;
  if (v <= 16) return agg_kernel<16, RELU, REMOTE, MINB>;
  if (v <= 32) return agg_kernel<32, RELU, REMOTE, MINB>;
  return agg_wide<RELU>;
}

int reg_cap_mode() {
  static const int m = [] {
    const char* e = std::getenv("MGG_AGG_MINB");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

// Lean local-only K1 (single-part launches, halo passes): the same
// partition / warp / CTA geometry without the pairing machinery, so the
// register footprint — hence resident warps, hence row loads in flight —
// is set by the gather alone.
template <int VEC, bool RELU>
__device__ __forceinline__ void agg_local_body(const AggArgs& a) {
  using L = Lanes<VEC, RELU>;
  const L ln(a);
  const int lane = ln.lane;
  float4 acc = f4zero();
  int cur = -1;
  uint32_t b0, b1;
  cta_chunk(a.num_lblocks, b0, b1);
  const uint32_t wib = threadIdx.x >> 5;
  for (uint32_t lb = b0; lb < b1; ++lb) {
    const uint32_t w = lb * a.wpb + wib;
    if (w >= a.num_warps) break;
    const uint32_t l0 = w * a.dist;
    const int nl = static_cast<int>(min(l0 + a.dist, a.nL) - l0);
    const int2 ml = lane <= nl ? __ldg(a.lmeta + l0 + lane) : make_int2(0, 0);
    int beg = __shfl_sync(kFull, ml.y, 0);
    int end = __shfl_sync(kFull, ml.y, 1);
    uint32_t win = load_colwin(a.lcols, beg, min(end - beg, 32));
    for (int i = 0; i < nl; ++i) {
      const int t = __shfl_sync(kFull, ml.x, i);
      const int nend = __shfl_sync(kFull, ml.y, i + 2);
      const uint32_t next = i + 1 < nl ? load_colwin(a.lcols, end, min(nend - end, 32)) : 0u;
      if (t != cur) {
        if (cur >= 0) ln.flush(a, acc, cur);
        acc = f4zero();
        cur = t;
      }
      acc = ln.template window<false>(a, win, min(end - beg, 32), 0, acc, nullptr);
      for (int b = beg + 32; b < end; b += 32) {  // whole-list tails
        const int n = min(end - b, 32);
        acc = ln.template window<false>(a, load_colwin(a.lcols, b, n), n, 0, acc, nullptr);
      }
      win = next;
      beg = end;
      end = nend;
    }
  }
  if (cur >= 0) ln.flush(a, acc, cur);
}

// Halo pull riding along a local pass (halo mode, fused): logical warp w of
// the pass copies halo rows [w·H/W, (w+1)·H/W) (H distinct remote rows, W
// logical warps) from their owners' shards into the halo, so the remote
// traffic is spread evenly over the whole pass (and its latency covered by
// the other warps' gathers) instead of running as a separate kernel that
// (persistent, full occupancy) cannot co-run with the pass. PULL 2 (default):
// after the warp's partitions, two rows at a time; PULL 1: one row issued
// before each partition and stored after it, the rest two at a time.
struct HaloPull {
  uint64_t r = 0, end = 0;
  uint64_t pol = 0;  // L2 evict-first: the copy must not push the local table out
  uint32_t step = 0, vec = 0, pitch = 0;
  int v = 0;
  bool vlane = false;
  __device__ __forceinline__ void begin(const AggArgs& a, uint32_t w, int grp, int G, int lane_v,
                                        bool vl) {
    end = 0;
    r = 0;
    if (!a.pull_n) return;
    const uint64_t H = a.pull_n, W = a.num_warps;
    r = w * H / W + grp;
    end = (w + 1ull) * H / W;
    step = static_cast<uint32_t>(G);
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    vec = a.vec;
    pitch = a.pitch;
    v = lane_v;
    vlane = vl;
  }
  __device__ __forceinline__ bool more() const { return r < end; }
  __device__ __forceinline__ float4 load(const AggArgs& a, uint64_t row) const {
    const uint32_t c = __ldg(a.pull_rows + row);
    const float* b = reinterpret_cast<const float*>(
        __ldg(reinterpret_cast<const unsigned long long*>(a.table) + (c >> kShift)));
    float4 x = f4zero();
    if (vlane)
      asm volatile("ld.global.cg.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                   : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                   : "l"(b + static_cast<size_t>(c & kMask) * pitch + 4 * v), "l"(pol));
    return x;
  }
  __device__ __forceinline__ void store(const AggArgs& a, uint64_t row, float4 x) const {
    if (vlane)
      asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(
                       a.pull_dst + row * pitch + 4 * v),
                   "f"(x.x), "f"(x.y), "f"(x.z), "f"(x.w), "l"(pol)
                   : "memory");
  }
  // the rows this group has left, two per round
  __device__ __forceinline__ void drain(const AggArgs& a) {
    for (; r < end; r += 2ull * step) {
      const bool two = r + step < end;
      const float4 x0 = load(a, r);
      const float4 x1 = two ? load(a, r + step) : f4zero();
      store(a, r, x0);
      if (two) store(a, r + step, x1);
    }
  }
};

// Group-per-partition local K1 for short partitions (HBM-resident tables):
// each VEC-lane group walks its own partition, UNR rows in flight per group
// (the next UNR column ids prefetched),
// so a warp keeps 32/VEC partitions' gathers outstanding at once instead of
// one partition's predicated window.
template <int VEC, bool RELU, int UNR, int PULL = 0>
__device__ __forceinline__ void agg_group_body(const AggArgs& a) {
  constexpr int G = 32 / VEC;
  const int lane = threadIdx.x & 31;
  const int grp = lane / VEC, v = lane % VEC;
  const bool vlane = v < static_cast<int>(a.vec);
  const uint32_t pb = a.pitch * 4u;
  const char* lbase = reinterpret_cast<const char*>(a.own) + (vlane ? 16u * v : 0u);
  asm("mov.b64 %0, %0;" : "+l"(lbase));
  auto load = [&](uint32_t c) {
    float4 x;
    asm(MGG_LD_INSN " {%0,%1,%2,%3}, [%4];"
        : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
        : "l"(lbase + static_cast<size_t>(c) * pb));
    if (RELU) x = f4relu(x);
    return x;
  };
  uint32_t b0, b1;
  cta_chunk(a.num_lblocks, b0, b1);
  const uint32_t wib = threadIdx.x >> 5;
  for (uint32_t lb = b0; lb < b1; ++lb) {
    const uint32_t w = lb * a.wpb + wib;
    if (w >= a.num_warps) break;
    const uint32_t l0 = w * a.dist;
    const uint32_t l1 = min(l0 + a.dist, a.nL);
    HaloPull hp;
    if (PULL) hp.begin(a, w, grp, G, v, vlane);
    for (uint32_t i = l0 + grp; i < l1; i += G) {
      const bool pull = PULL == 1 && hp.more();
      const uint64_t pr = hp.r;
      const float4 px = pull ? hp.load(a, pr) : f4zero();
      const int2 m = __ldg(a.lmeta + i);
      const int end = __ldg(&a.lmeta[i + 1].y);
      float4 acc = f4zero();
      int k = m.y;
      // column ids of step s+1 load while step s's rows are in flight
      uint32_t c[UNR];
      if (k + UNR <= end) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) c[u] = __ldg(a.lcols + k + u);
      }
      for (; k + UNR <= end; k += UNR) {
        float4 t[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) t[u] = load(c[u]);
        if (k + 2 * UNR <= end) {
#pragma unroll
          for (int u = 0; u < UNR; ++u) c[u] = __ldg(a.lcols + k + UNR + u);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
      }
      if (k < end) {
        float4 t[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          t[u] = k + u < end ? load(__ldg(a.lcols + k + u)) : f4zero();
#pragma unroll
        for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
      }
      if (vlane) red_add4(a.out + static_cast<size_t>(m.x) * a.pitch + 4 * v, acc);
      if (pull) {
        hp.store(a, pr, px);
        hp.r += G;
      }
    }
    if (PULL) hp.drain(a);
  }
}
// agg_group with L2 eviction hints: gathered rows evict-last (they are the
// only reuse K1 has), column ids and accumulator reductions evict-first.
// FETCH: L2 fetch size of the gathered-row misses — 0 the default (the line:
// 64-B rows also bring their neighbour row in, ~1.3-1.5x DRAM bytes on
// random tables that do not fit L2), 64 = `L2::64B` (only the row's sectors).
template <int VEC, bool RELU, int UNR, int FETCH = 0, int PULL = 0>
__device__ __forceinline__ void agg_group_hint_body(const AggArgs& a) {
  constexpr int G = 32 / VEC;
  const int lane = threadIdx.x & 31;
  const int grp = lane / VEC, v = lane % VEC;
  const bool vlane = v < static_cast<int>(a.vec);
  const uint32_t pb = a.pitch * 4u;
  const char* lbase = reinterpret_cast<const char*>(a.own) + (vlane ? 16u * v : 0u);
  asm("mov.b64 %0, %0;" : "+l"(lbase));
  uint64_t pol_last, pol_first;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
  auto load = [&](uint32_t c) {
    float4 x;
    if (FETCH == 64)
      asm("ld.global.cg.L2::64B.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
          : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
          : "l"(lbase + static_cast<size_t>(c) * pb), "l"(pol_last));
    else
      asm("ld.global.cg.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
          : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
          : "l"(lbase + static_cast<size_t>(c) * pb), "l"(pol_last));
    if (RELU) x = f4relu(x);
    return x;
  };
  auto ldcol = [&](const uint32_t* p) {
    uint32_t r;
    // volatile: a plain asm is speculatable, and the tail's guarded column
    // loads would be if-converted into unguarded reads past the partition
    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;"
                 : "=r"(r)
                 : "l"(p), "l"(pol_first));
    return r;
  };
  uint32_t b0, b1;
  cta_chunk(a.num_lblocks, b0, b1);
  const uint32_t wib = threadIdx.x >> 5;
  for (uint32_t lb = b0; lb < b1; ++lb) {
    const uint32_t w = lb * a.wpb + wib;
    if (w >= a.num_warps) break;
    const uint32_t l0 = w * a.dist;
    const uint32_t l1 = min(l0 + a.dist, a.nL);
    HaloPull hp;
    if (PULL) hp.begin(a, w, grp, G, v, vlane);
    for (uint32_t i = l0 + grp; i < l1; i += G) {
      const bool pull = PULL == 1 && hp.more();
      const uint64_t pr = hp.r;
      const float4 px = pull ? hp.load(a, pr) : f4zero();
      const int2 m = __ldg(a.lmeta + i);
      const int end = __ldg(&a.lmeta[i + 1].y);
      float4 acc = f4zero();
      int k = m.y;
      // column ids of step s+1 load while step s's rows are in flight
      uint32_t c[UNR];
      if (k + UNR <= end) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) c[u] = ldcol(a.lcols + k + u);
      }
      for (; k + UNR <= end; k += UNR) {
        float4 t[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) t[u] = load(c[u]);
        if (k + 2 * UNR <= end) {
#pragma unroll
          for (int u = 0; u < UNR; ++u) c[u] = ldcol(a.lcols + k + UNR + u);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
      }
      if (k < end) {
        float4 t[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          t[u] = k + u < end ? load(ldcol(a.lcols + k + u)) : f4zero();
#pragma unroll
        for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
      }
      if (vlane)
        asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(
                         a.out + static_cast<size_t>(m.x) * a.pitch + 4 * v),
                     "f"(acc.x), "f"(acc.y), "f"(acc.z), "f"(acc.w), "l"(pol_first)
                     : "memory");
      if (pull) {
        hp.store(a, pr, px);
        hp.r += G;
      }
    }
    if (PULL) hp.drain(a);
  }
}
// Group-per-partition form of the paired (fine-fetch) K1: group g of a
// logical warp takes pairs i = g, g + 32/VEC, ... of the warp's local and
// remote groups and keeps the reference's async discipline per pair
// (R:proj/src/sim.cpp:102-125): issue the first PF peer rows of R_i, reduce
// L_i, then consume R_i — per group instead of per warp.
template <int VEC, bool RELU, int UNR, int PF, bool TRACE = false>
__device__ __forceinline__ void agg_gpair_body(const AggArgs& a) {
  constexpr int G = 32 / VEC;
  const int lane = threadIdx.x & 31;
  const int grp = lane / VEC, v = lane % VEC;
  const bool vlane = v < static_cast<int>(a.vec);
  const uint32_t voff = vlane ? 16u * v : 0u;
  const uint32_t pb = a.pitch * 4u;
  const char* lbase = reinterpret_cast<const char*>(a.own) + voff;
  asm("mov.b64 %0, %0;" : "+l"(lbase));
  auto ld = [&](const char* p) {
    float4 x;
    asm(MGG_LD_INSN " {%0,%1,%2,%3}, [%4];"
        : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
        : "l"(p));
    if (RELU) x = f4relu(x);
    return x;
  };
  auto raddr = [&](uint32_t c) {
    const char* b =
        a.halo ? reinterpret_cast<const char*>(a.halo)
               : reinterpret_cast<const char*>(
                     __ldg(reinterpret_cast<const unsigned long long*>(a.table) + (c >> kShift)));
    return b + voff + static_cast<size_t>(c & kMask) * pb;
  };
  auto run_warp = [&](uint32_t w, uint32_t) {
    uint32_t l0, l1, r0, r1;
    warp_groups(a, w, l0, l1, r0, r1);
    const uint32_t nl = l1 - l0, nr = r1 - r0, n = max(nl, nr);
    for (uint32_t i = grp; i < n; i += G) {
      // (1) issue R_i's first PF peer rows
      float4 pre[PF];
      int rk = 0, rend = 0, rt = 0;
      const uint32_t tid = w * G + grp;
      if (i < nr) {
        if (TRACE) trace_emit_g(a, w, tid, v == 0, kLR, true, stamp_after(0.f));
        const int2 m = __ldg(a.rmeta + r0 + i);
        rend = __ldg(&a.rmeta[r0 + i + 1].y);
        rt = m.x;
        rk = m.y;
#pragma unroll
        for (int u = 0; u < PF; ++u)
          pre[u] = rk + u < rend ? ld(raddr(__ldg(a.rcols + rk + u))) : f4zero();
        rk = min(rk + PF, rend);
      }
      // (2) reduce L_i
      if (i < nl) {
        const int2 m = __ldg(a.lmeta + l0 + i);
        const int end = __ldg(&a.lmeta[l0 + i + 1].y);
        float4 acc = f4zero();
        if (TRACE) trace_emit_g(a, w, tid, v == 0, kLL, true, stamp_after(0.f));
        int k = m.y;
        for (; k + UNR <= end; k += UNR) {
          uint32_t c[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u) c[u] = __ldg(a.lcols + k + u);
          float4 t[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u) t[u] = ld(lbase + static_cast<size_t>(c[u]) * pb);
#pragma unroll
          for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
        }
        if (k < end) {
          float4 t[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u)
            t[u] = k + u < end ? ld(lbase + static_cast<size_t>(__ldg(a.lcols + k + u)) * pb)
                               : f4zero();
#pragma unroll
          for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
        }
        if (TRACE) trace_emit_g(a, w, tid, v == 0, kLL, false, stamp_after(acc.x));
        if (vlane) red_add4(a.out + static_cast<size_t>(m.x) * a.pitch + 4 * v, acc);
      }
      // (3) consume R_i
      if (i < nr) {
        float4 acc = f4zero();
        if (TRACE) {  // R_i's issued rows have landed: the get ends, AC starts
          const uint64_t t = stamp_after(pre[PF - 1].x);
          trace_emit_g(a, w, tid, v == 0, kLR, false, t);
          trace_emit_g(a, w, tid, v == 0, kAC, true, t);
        }
#pragma unroll
        for (int u = 0; u < PF; ++u) acc = f4add(acc, pre[u]);
        for (; rk < rend; rk += UNR) {
          float4 t[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u)
            t[u] = rk + u < rend ? ld(raddr(__ldg(a.rcols + rk + u))) : f4zero();
#pragma unroll
          for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
        }
        if (TRACE) trace_emit_g(a, w, tid, v == 0, kAC, false, stamp_after(acc.x));
        if (vlane) red_add4(a.out + static_cast<size_t>(rt) * a.pitch + 4 * v, acc);
      }
    }
  };
  if (a.sched) {
    for_each_ticket<1>(a, run_warp);
    return;
  }
  const LbRange rg = lb_range(a);
  const uint32_t wib = threadIdx.x >> 5;
  for (uint32_t lb = rg.first; lb < rg.end; lb = rg.next(lb)) {
    const uint32_t w = lb * a.wpb + wib;
    if (w >= a.num_warps) break;
    run_warp(w, 0);
  }
}

// Kind-split form of the fine-fetch K1 (agg_gsplit): the same plan and the
// same dynamic ticket queue, but a ticket is ONE kind of a chunk of logical
// warps — its local partitions or its remote ones, adjacent in the dealing
// order — and each is reduced by the lean group-per-partition loop (UNR rows
// in flight per group, next column ids prefetched). The overlap the
// reference builds inside a warp (issue R_i, reduce L_i, consume R_i;
// R:proj/src/sim.cpp:102-125) happens between warps of the same SM instead:
// at any time some resident warps hold remote tickets and wait on the link
// while the others reduce local partitions, and neither loop carries the
// other's registers (agg_gpair stages PF remote rows per lane across L_i).
template <int VEC, bool RELU, int UNR>
__device__ __forceinline__ void agg_gsplit_body(const AggArgs& a) {
  constexpr int G = 32 / VEC;
  const int lane = threadIdx.x & 31;
  const int grp = lane / VEC, v = lane % VEC;
  const bool vlane = v < static_cast<int>(a.vec);
  const uint32_t voff = vlane ? 16u * v : 0u;
  const uint32_t pb = a.pitch * 4u;
  const char* lbase = reinterpret_cast<const char*>(a.own) + voff;
  asm("mov.b64 %0, %0;" : "+l"(lbase));
  auto ld = [&](const char* p) {
    float4 x;
    asm(MGG_LD_INSN " {%0,%1,%2,%3}, [%4];"
        : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
        : "l"(p));
    if (RELU) x = f4relu(x);
    return x;
  };
  // one loop per kind (compile-time), so the local loop carries no
  // owner-table addressing
  auto loop = [&](auto remc, uint32_t i0, uint32_t p1) {
    constexpr bool REM = decltype(remc)::value;
    constexpr int U = REM ? UNR / 2 : UNR;  // remote rows carry a 64-bit base each
    const int2* meta = REM ? a.rmeta : a.lmeta;
    const uint32_t* cols = REM ? a.rcols : a.lcols;
    auto addr = [&](uint32_t c) {
      if constexpr (!REM) {
        return lbase + static_cast<size_t>(c) * pb;
      } else {
        const char* b = a.halo ? reinterpret_cast<const char*>(a.halo)
                               : reinterpret_cast<const char*>(__ldg(
                                     reinterpret_cast<const unsigned long long*>(a.table) +
                                     (c >> kShift)));
        return b + voff + static_cast<size_t>(c & kMask) * pb;
      }
    };
    for (uint32_t i = i0; i < p1; i += G) {
      const int2 m = __ldg(meta + i);
      const int end = __ldg(&meta[i + 1].y);
      float4 acc = f4zero();
      int k = m.y;
      uint32_t c[U];
      if (k + U <= end) {
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = __ldg(cols + k + u);
      }
      for (; k + U <= end; k += U) {
        float4 t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) t[u] = ld(addr(c[u]));
        if (k + 2 * U <= end) {
#pragma unroll
          for (int u = 0; u < U; ++u) c[u] = __ldg(cols + k + U + u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc = f4add(acc, t[u]);
      }
      if (k < end) {
        float4 t[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          t[u] = k + u < end ? ld(addr(__ldg(cols + k + u))) : f4zero();
#pragma unroll
        for (int u = 0; u < U; ++u) acc = f4add(acc, t[u]);
      }
      if (vlane) red_add4(a.out + static_cast<size_t>(m.x) * a.pitch + 4 * v, acc);
    }
  };
  auto run = [&](uint32_t w, uint32_t kind) {
    uint32_t l0, l1, r0, r1;
    warp_groups(a, w, l0, l1, r0, r1);
    if (kind)
      loop(std::true_type{}, r0 + grp, r1);
    else
      loop(std::false_type{}, l0 + grp, l1);
  };
  if (a.sched) {
    for_each_ticket<2>(a, run);
    return;
  }
  const LbRange rg = lb_range(a);  // static: both kinds of each logical warp
  const uint32_t wib = threadIdx.x >> 5;
  for (uint32_t lb = rg.first; lb < rg.end; lb = rg.next(lb)) {
    const uint32_t w = lb * a.wpb + wib;
    if (w >= a.num_warps) break;
    run(w, 1);
    run(w, 0);
  }
}
// Fine-fetch K1 with the remote rows staged in shared memory (agg_pipe):
// the paper's remote get into shared memory (R:PAPER.md:400-419) with the
// reference's per-pair order (issue R_i, reduce L_i, consume R_i;
// R:proj/src/sim.cpp:102-125), deepened into a per-lane ring. Each lane owns
// R 16-B slots in shared memory; the group's remote rows — every R partition
// of every pair the group will visit, in consumption order — stream through
// the ring as cp.async copies straight from the owner's shard (peer / IPC /
// host-mapped address) into the slots, always R rows ahead of the consumer:
// one copy is issued per row consumed, so exactly R commit groups are in
// flight and `cp.async.wait_group R-1` releases the oldest. In-flight rows
// hold no registers (the register-staged agg_gpair keeps PF float4 per lane
// and re-issues the rest of R_i at consume time, exposing the remote latency
// once per 4 rows); local partitions are reduced from registers meanwhile.
// A lane reads back only the slots it filled itself, so no barrier is needed.
template <int VEC, bool RELU, int UNR, int R>
__device__ __forceinline__ void agg_pipe_body(const AggArgs& a) {
  static_assert((R & (R - 1)) == 0, "ring depth must be a power of two");
  constexpr int G = 32 / VEC;
  extern __shared__ float4 pipe_ring[];
  const int lane = threadIdx.x & 31;
  const int grp = lane / VEC, v = lane % VEC;
  const bool vlane = v < static_cast<int>(a.vec);
  const uint32_t voff = vlane ? 16u * v : 0u;
  const uint32_t pb = a.pitch * 4u;
  const char* lbase = reinterpret_cast<const char*>(a.own) + voff;
  asm("mov.b64 %0, %0;" : "+l"(lbase));
  const uint32_t ring0 = static_cast<uint32_t>(__cvta_generic_to_shared(pipe_ring + threadIdx.x));
  const uint32_t rstride = blockDim.x * 16u;
  auto ld = [&](const char* p) {
    float4 x;
    asm(MGG_LD_INSN " {%0,%1,%2,%3}, [%4];"
        : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
        : "l"(p));
    if (RELU) x = f4relu(x);
    return x;
  };
  auto raddr = [&](uint32_t c) {
    const char* b =
        a.halo ? reinterpret_cast<const char*>(a.halo)
               : reinterpret_cast<const char*>(
                     __ldg(reinterpret_cast<const unsigned long long*>(a.table) + (c >> kShift)));
    return b + voff + static_cast<size_t>(c & kMask) * pb;
  };
  uint64_t pol_last, pol_first;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
  auto ldh = [&](const char* p) {
    float4 x;
    asm("ld.global.cg.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
        : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
        : "l"(p), "l"(pol_last));
    if (RELU) x = f4relu(x);
    return x;
  };
  auto ldcol = [&](const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol_first));
    return r;
  };
  auto redh = [&](float* p, float4 v4) {
    asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p),
                 "f"(v4.x), "f"(v4.y), "f"(v4.z), "f"(v4.w), "l"(pol_first)
                 : "memory");
  };
  const LbRange rg = lb_range(a);
  const uint32_t wib = threadIdx.x >> 5;

  // producer cursor over the group's remote rows in consumption order, kept
  // one row (column id in flight) and one partition (bounds in flight) ahead
  // so that issuing a copy never waits on a dependent metadata load
  uint32_t plb = rg.first, pw = rg.first * a.wpb + wib, pr0 = 0, pr1 = 0, pi = grp;
  int pk = 0, pend = 0, qk = 0, qend = 0;
  uint32_t ncol = 0;
  bool qvalid = false, pdone = rg.first >= rg.end || pw >= a.num_warps;
  if (!pdone) {
    uint32_t l0, l1;
    warp_groups(a, pw, l0, l1, pr0, pr1);
  }
  // queue the bounds of the next remote partition of this group (no wait)
  auto queue_next = [&]() {
    qvalid = false;
    while (!pdone) {
      if (pr0 + pi < pr1) {
        qk = __ldg(&a.rmeta[pr0 + pi].y);
        qend = __ldg(&a.rmeta[pr0 + pi + 1].y);
        pi += G;
        qvalid = true;
        return;
      }
      plb = rg.next(plb);
      pw = plb * a.wpb + wib;
      if (plb >= rg.end || pw >= a.num_warps) {
        pdone = true;
      } else {
        uint32_t l0, l1;
        warp_groups(a, pw, l0, l1, pr0, pr1);
        pi = grp;
      }
    }
  };
  // make the queued partition current (skipping empty ones)
  auto advance = [&]() {
    while (qvalid) {
      pk = qk;
      pend = qend;
      queue_next();
      if (pk < pend) {
        ncol = __ldg(a.rcols + pk);
        return;
      }
    }
  };
  queue_next();
  advance();
  uint32_t issued = 0, consumed = 0;
  auto produce = [&]() {
    if (pk < pend) {
      const uint32_t c = ncol;
      if (++pk < pend)
        ncol = __ldg(a.rcols + pk);  // used by the next call
      else
        advance();
      const char* src = raddr(c);
      const uint32_t dst = ring0 + (issued & (R - 1)) * rstride;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // empty past the end
    ++issued;
  };
#pragma unroll 1
  for (int s = 0; s < R; ++s) produce();

  for (uint32_t lb = rg.first; lb < rg.end; lb = rg.next(lb)) {
    const uint32_t w = lb * a.wpb + wib;
    if (w >= a.num_warps) break;
    uint32_t l0, l1, r0, r1;
    warp_groups(a, w, l0, l1, r0, r1);
    const uint32_t nl = l1 - l0, nr = r1 - r0, n = max(nl, nr);
    for (uint32_t i = grp; i < n; i += G) {
      // (1) R_i is already in flight (issued up to R rows ago)
      // (2) reduce L_i from registers: the lean group kernel's gather (UNR
      // rows in flight, the next UNR column ids prefetched, gathered rows
      // evict-last / column ids and reductions evict-first in L2)
      if (i < nl) {
        const int2 m = __ldg(a.lmeta + l0 + i);
        const int end = __ldg(&a.lmeta[l0 + i + 1].y);
        float4 acc = f4zero();
        int k = m.y;
        uint32_t c[UNR];
        if (k + UNR <= end) {
#pragma unroll
          for (int u = 0; u < UNR; ++u) c[u] = ldcol(a.lcols + k + u);
        }
        for (; k + UNR <= end; k += UNR) {
          float4 t[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u) t[u] = ldh(lbase + static_cast<size_t>(c[u]) * pb);
          if (k + 2 * UNR <= end) {
#pragma unroll
            for (int u = 0; u < UNR; ++u) c[u] = ldcol(a.lcols + k + UNR + u);
          }
#pragma unroll
          for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
        }
        if (k < end) {
          float4 t[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u)
            t[u] = k + u < end ? ldh(lbase + static_cast<size_t>(ldcol(a.lcols + k + u)) * pb)
                               : f4zero();
#pragma unroll
          for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
        }
        if (vlane) redh(a.out + static_cast<size_t>(m.x) * a.pitch + 4 * v, acc);
      }
      // (3) consume R_i from the ring; every row consumed issues the next
      if (i < nr) {
        const int2 m = __ldg(a.rmeta + r0 + i);
        const int end = __ldg(&a.rmeta[r0 + i + 1].y);
        float4 acc = f4zero();
        for (int k = m.y; k < end; ++k) {
          asm volatile("cp.async.wait_group %0;" ::"n"(R - 1) : "memory");
          float4 x;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                       : "r"(ring0 + (consumed & (R - 1)) * rstride)
                       : "memory");
          ++consumed;
          if (RELU) x = f4relu(x);
          acc = f4add(acc, x);
          produce();  // refills the slot just read (after its value is used)
        }
        if (vlane) red_add4(a.out + static_cast<size_t>(m.x) * a.pitch + 4 * v, acc);
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}
// TMA form of agg_pipe (agg_pipe_bulk): the remote rows are fetched by the
// bulk-copy engine — one `cp.async.bulk` of the whole row (pitch x 4 B) per
// remote neighbour, issued by the group's first lane straight from the
// owner's shard into a per-group ring of R row slots, completion counted in
// bytes on the slot's mbarrier (north_star: "TMA from the mapped peer
// address"). Remote requests then occupy the TMA unit's queue instead of the
// SM's load/store request slots, which the local gathers keep to themselves.
// Same cursor, order and one-row-per-consumed-row refill as agg_pipe; a
// group syncs (__syncwarp on its lanes) before its leader refills a slot.
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
template <int VEC, bool RELU, int UNR, int R>
__device__ __forceinline__ void agg_pipe_bulk_body(const AggArgs& a) {
  constexpr int G = 32 / VEC;
  extern __shared__ __align__(16) unsigned char pipe_raw[];
  const int lane = threadIdx.x & 31;
  const int grp = lane / VEC, v = lane % VEC;
  const bool vlane = v < static_cast<int>(a.vec);
  const uint32_t voff = vlane ? 16u * v : 0u;
  const uint32_t pb = a.pitch * 4u;
  const bool leader = v == 0;
  const unsigned gmask = (VEC == 32 ? 0xffffffffu : ((1u << VEC) - 1u)) << (grp * VEC);
  const char* lbase = reinterpret_cast<const char*>(a.own) + voff;
  asm("mov.b64 %0, %0;" : "+l"(lbase));
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t gid = wib * G + grp;  // group index in the CTA
  const uint32_t ngroups = (blockDim.x >> 5) * G;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(pipe_raw));
  const uint32_t slots = sbase + gid * R * pb;                  // R row slots
  const uint32_t bars = sbase + ngroups * R * pb + gid * R * 8;  // R mbarriers
  if (leader) {
#pragma unroll 1
    for (int r = 0; r < R; ++r)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * r) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto ld = [&](const char* p) {
    float4 x;
    asm(MGG_LD_INSN " {%0,%1,%2,%3}, [%4];"
        : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
        : "l"(p));
    if (RELU) x = f4relu(x);
    return x;
  };
  auto rrow = [&](uint32_t c) {  // the whole remote row (bulk source)
    const char* b =
        a.halo ? reinterpret_cast<const char*>(a.halo)
               : reinterpret_cast<const char*>(
                     __ldg(reinterpret_cast<const unsigned long long*>(a.table) + (c >> kShift)));
    return b + static_cast<size_t>(c & kMask) * pb;
  };
  const LbRange rg = lb_range(a);

  // producer cursor (the leader's; the same as agg_pipe's)
  uint32_t plb = rg.first, pw = rg.first * a.wpb + wib, pr0 = 0, pr1 = 0, pi = grp;
  int pk = 0, pend = 0, qk = 0, qend = 0;
  uint32_t ncol = 0;
  bool qvalid = false, pdone = rg.first >= rg.end || pw >= a.num_warps;
  if (!pdone) {
    uint32_t l0, l1;
    warp_groups(a, pw, l0, l1, pr0, pr1);
  }
  auto queue_next = [&]() {
    qvalid = false;
    while (!pdone) {
      if (pr0 + pi < pr1) {
        qk = __ldg(&a.rmeta[pr0 + pi].y);
        qend = __ldg(&a.rmeta[pr0 + pi + 1].y);
        pi += G;
        qvalid = true;
        return;
      }
      plb = rg.next(plb);
      pw = plb * a.wpb + wib;
      if (plb >= rg.end || pw >= a.num_warps) {
        pdone = true;
      } else {
        uint32_t l0, l1;
        warp_groups(a, pw, l0, l1, pr0, pr1);
        pi = grp;
      }
    }
  };
  auto advance = [&]() {
    while (qvalid) {
      pk = qk;
      pend = qend;
      queue_next();
      if (pk < pend) {
        ncol = __ldg(a.rcols + pk);
        return;
      }
    }
  };
  queue_next();  // every lane walks the cursor (no divergent scans) ...
  advance();
  uint32_t issued = 0, consumed = 0;
  auto produce = [&]() {  // ... and the group's leader issues the copy
    if (pk < pend) {
      const uint32_t c = ncol;
      if (++pk < pend)
        ncol = __ldg(a.rcols + pk);
      else
        advance();
      if (leader) {
        const uint32_t slot = issued & (R - 1);
        const uint32_t bar = bars + 8 * slot;
        // the group's generic reads of this slot before the async-proxy write
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(pb)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(slots + slot * pb),
            "l"(rrow(c)), "r"(pb), "r"(bar)
            : "memory");
      }
    }
    ++issued;
  };
#pragma unroll 1
  for (int r = 0; r < R; ++r) produce();

  for (uint32_t lb = rg.first; lb < rg.end; lb = rg.next(lb)) {
    const uint32_t w = lb * a.wpb + wib;
    if (w >= a.num_warps) break;
    uint32_t l0, l1, r0, r1;
    warp_groups(a, w, l0, l1, r0, r1);
    const uint32_t nl = l1 - l0, nr = r1 - r0, n = max(nl, nr);
    for (uint32_t i = grp; i < n; i += G) {
      if (i < nl) {  // reduce L_i from registers while R_i is in flight
        const int2 m = __ldg(a.lmeta + l0 + i);
        const int end = __ldg(&a.lmeta[l0 + i + 1].y);
        float4 acc = f4zero();
        int k = m.y;
        for (; k + UNR <= end; k += UNR) {
          uint32_t c[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u) c[u] = __ldg(a.lcols + k + u);
          float4 t[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u) t[u] = ld(lbase + static_cast<size_t>(c[u]) * pb);
#pragma unroll
          for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
        }
        if (k < end) {
          float4 t[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u)
            t[u] = k + u < end ? ld(lbase + static_cast<size_t>(__ldg(a.lcols + k + u)) * pb)
                               : f4zero();
#pragma unroll
          for (int u = 0; u < UNR; ++u) acc = f4add(acc, t[u]);
        }
        if (vlane) red_add4(a.out + static_cast<size_t>(m.x) * a.pitch + 4 * v, acc);
      }
      if (i < nr) {  // consume R_i from the ring
        const int2 m = __ldg(a.rmeta + r0 + i);
        const int end = __ldg(&a.rmeta[r0 + i + 1].y);
        float4 acc = f4zero();
        for (int k = m.y; k < end; ++k) {
          const uint32_t slot = consumed & (R - 1);
          const uint32_t parity = (consumed / R) & 1u;
          if (!mbar_try(bars + 8 * slot, parity)) {
            uint64_t t0, t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            while (!mbar_try(bars + 8 * slot, parity)) {
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
              if (t - t0 > 4000000000ull) __trap();  // a copy that never lands
            }
          }
          float4 x;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                       : "r"(slots + slot * pb + voff)
                       : "memory");
          ++consumed;
          if (RELU) x = f4relu(x);
          acc = f4add(acc, x);
          __syncwarp(gmask);  // every lane of the group has read the slot
          produce();
        }
        if (vlane) red_add4(a.out + static_cast<size_t>(m.x) * a.pitch + 4 * v, acc);
      }
    }
  }
  // drain: wait for copies issued past the last consumed row (none are
  // issued beyond the stream, so every issued copy was consumed)
}
template <int VEC, bool RELU, int UNR, int R>
__global__ void __launch_bounds__(512, 2) agg_pipe_bulk(AggArgs a) {
  agg_pipe_bulk_body<VEC, RELU, UNR, R>(a);
}

template <int VEC, bool RELU, int UNR, int R>
__global__ void __launch_bounds__(512, 2) agg_pipe(AggArgs a) {
  agg_pipe_body<VEC, RELU, UNR, R>(a);
}
// dynamic shared memory of the pipe kernels: agg_pipe R 16-B slots per
// thread; agg_pipe_bulk R row slots + R mbarriers per lane group
struct PipeSmem {
  uint32_t r, vec, bulk;
};
std::map<const void*, PipeSmem>& pipe_slots() {
  static std::map<const void*, PipeSmem> m;
  return m;
}
template <bool RELU, int R>
KernelFn pick_pipe(uint32_t v) {
  KernelFn k = v <= 1    ? agg_pipe<1, RELU, 8, R>
               : v <= 2  ? agg_pipe<2, RELU, 8, R>
               : v <= 4  ? agg_pipe<4, RELU, 8, R>
               : v <= 8  ? agg_pipe<8, RELU, 8, R>
               : v <= 16 ? agg_pipe<16, RELU, 8, R>
               : v <= 32 ? agg_pipe<32, RELU, 8, R>
                         : agg_wide<RELU>;
  if (v <= 32) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    pipe_slots()[reinterpret_cast<const void*>(k)] = {R, 0, 0};
  }
  return k;
}
template <bool RELU, int R>
KernelFn pick_pipe_bulk(uint32_t v) {
  KernelFn k = v <= 1    ? agg_pipe_bulk<1, RELU, 4, R>
               : v <= 2  ? agg_pipe_bulk<2, RELU, 4, R>
               : v <= 4  ? agg_pipe_bulk<4, RELU, 4, R>
               : v <= 8  ? agg_pipe_bulk<8, RELU, 4, R>
               : v <= 16 ? agg_pipe_bulk<16, RELU, 4, R>
               : v <= 32 ? agg_pipe_bulk<32, RELU, 4, R>
                         : agg_wide<RELU>;
  const uint32_t vec = v <= 1 ? 1 : v <= 2 ? 2 : v <= 4 ? 4 : v <= 8 ? 8 : v <= 16 ? 16 : 32;
  if (v <= 32) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    pipe_slots()[reinterpret_cast<const void*>(k)] = {R, vec, 1};
  }
  return k;
}
uint32_t dyn_smem(KernelFn k, int threads, uint32_t pitch) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  auto it = pipe_slots().find(reinterpret_cast<const void*>(k));
  if (it == pipe_slots().end()) return 0u;
  const PipeSmem& p = it->second;
  if (!p.bulk) return p.r * 16u * static_cast<uint32_t>(threads);
  const uint32_t groups = static_cast<uint32_t>(threads) / 32u * (32u / p.vec);
  return groups * p.r * (pitch * 4u + 8u);
}

template <int VEC, int PF>
__global__ void __launch_bounds__(512, 2) agg_gpair_traced(AggArgs a) {
  agg_gpair_body<VEC, false, 4, PF, true>(a);
}
template <int VEC, bool RELU, int UNR, int PF>
__global__ void __launch_bounds__(512, 2) agg_gpair(AggArgs a) {
  agg_gpair_body<VEC, RELU, UNR, PF>(a);
}
template <int VEC, bool RELU, int UNR>
__global__ void __launch_bounds__(512, 2) agg_gsplit(AggArgs a) {
  agg_gsplit_body<VEC, RELU, UNR>(a);
}
template <bool RELU, int UNR>
KernelFn pick_gsplit(uint32_t v) {
  if (v <= 1) return agg_gsplit<1, RELU, UNR>;
  if (v <= 2) return agg_gsplit<2, RELU, UNR>;
  if (v <= 4) return agg_gsplit<4, RELU, UNR>;
  if (v <= 8) return agg_gsplit<8, RELU, UNR>;
  if (v <= 16) return agg_gsplit<16, RELU, UNR>;
  if (v <= 32) return agg_gsplit<32, RELU, UNR>;
  return agg_wide<RELU>;
}
template <bool RELU, int UNR, int PF>
KernelFn pick_gpair(uint32_t v) {
  if (v <= 1) return agg_gpair<1, RELU, UNR, PF>;
  if (v <= 2) return agg_gpair<2, RELU, UNR, PF>;
  if (v <= 4) return agg_gpair<4, RELU, UNR, PF>;
  if (v <= 8) return agg_gpair<8, RELU, UNR, PF>;
  if (v <= 16) return agg_gpair<16, RELU, UNR, PF>;
  if (v <= 32) return agg_gpair<32, RELU, UNR, PF>;
  return agg_wide<RELU>;
}

template <int VEC, bool RELU, int UNR, int PULL = 0>
__global__ void __launch_bounds__(512, 2) agg_group(AggArgs a) {
  agg_group_body<VEC, RELU, UNR, PULL>(a);
}
template <bool RELU, int UNR>
KernelFn pick_group(uint32_t v) {
  if (v <= 1) return agg_group<1, RELU, UNR>;
  if (v <= 2) return agg_group<2, RELU, UNR>;
  if (v <= 4) return agg_group<4, RELU, UNR>;
  if (v <= 8) return agg_group<8, RELU, UNR>;
  if (v <= 16) return agg_group<16, RELU, UNR>;
  if (v <= 32) return agg_group<32, RELU, UNR>;
  return agg_wide<RELU>;
}
template <int VEC, bool RELU, int UNR, int FETCH, int PULL = 0>
__global__ void __launch_bounds__(512, 2) agg_group_hint(AggArgs a) {
  agg_group_hint_body<VEC, RELU, UNR, FETCH, PULL>(a);
}
int l2_fetch() {
  static const int m = [] {
    const char* e = std::getenv("MGG_AGG_L2FETCH");  // 0 default line fetch, 64 = L2::64B
    return e ? std::atoi(e) : 0;
  }();
  return m;
}
int hint_unroll() {
  static const int m = [] {
    const char* e = std::getenv("MGG_AGG_HINT_UNR");  // rows in flight per group: 8 or 16
    return e ? std::atoi(e) : 8;
  }();
  return m;
}
template <bool RELU>
KernelFn pick_group_hint(uint32_t v) {
  if (v > 4) return agg_group_hint<16, RELU, 8, 0>;
  if (l2_fetch() == 64)
    return hint_unroll() == 16 ? agg_group_hint<4, RELU, 16, 64> : agg_group_hint<4, RELU, 8, 64>;
  return hint_unroll() == 16 ? agg_group_hint<4, RELU, 16, 0> : agg_group_hint<4, RELU, 8, 0>;
}

// The register budget is the occupancy knob of this latency-bound gather:
// MINB resident 512-thread CTAs (64 / 42 / 32 registers), or an explicit cap.
template <int VEC, bool RELU, int MINB>
__global__ void __launch_bounds__(512, MINB) agg_local(AggArgs a) {
  agg_local_body<VEC, RELU>(a);
}
template <int VEC, bool RELU, int REGS>
__global__ void __maxnreg__(REGS) agg_local_r(AggArgs a) {
  agg_local_body<VEC, RELU>(a);
}
template <bool RELU, int REGS>
KernelFn pick_local_r(uint32_t v) {
  if (v <= 1) return agg_local_r<1, RELU, REGS>;
  if (v <= 2) return agg_local_r<2, RELU, REGS>;
  if (v <= 4) return agg_local_r<4, RELU, REGS>;
  if (v <= 8) return agg_local_r<8, RELU, REGS>;
  if (v <= 16) return agg_local_r<16, RELU, REGS>;
  if (v <= 32) return agg_local_r<32, RELU, REGS>;
  return agg_wide<RELU>;
}

template <bool RELU, int MINB>
KernelFn pick_local(uint32_t v) {
  if (v <= 1) return agg_local<1, RELU, MINB>;
  if (v <= 2) return agg_local<2, RELU, MINB>;
  if (v <= 4) return agg_local<4, RELU, MINB>;
  if (v <= 8) return agg_local<8, RELU, MINB>;
  if (v <= 16) return agg_local<16, RELU, MINB>;
  if (v <= 32) return agg_local<32, RELU, MINB>;
  return agg_wide<RELU>;
}

int lean_mode() {
  static const int m = [] {
    const char* e = std::getenv("MGG_AGG_LEAN");
    return e ? std::atoi(e) : 1;
  }();
  return m;
}

template <bool RELU, bool REMOTE>
KernelFn pick(uint32_t v) {
  if (!REMOTE && lean_mode() > 0) {
    switch (lean_mode()) {
      // A/B knobs (MGG_AGG_LEAN; 1 = by plan shape, pick_lean; 2 = always the
      // warp-window kernel below): 3 = MINB 3 cap, 10 = 48 registers at every
      // width, 20 = always group-per-partition. The other variants measured
      // are in profiles/r01_k1_experiments.md.
      case 3: return pick_local<RELU, 3>(v);
      case 10: return pick_local_r<RELU, 48>(v);
      case 20: return pick_group<RELU, 8>(v);
      // measured (profiles/r01_k1_experiments.md): narrow rows (<= 16 floats)
      // want the 64-register cap; wider rows an explicit 48 (products-gin
      // K1 2.68 -> 2.48 ms vs the spilling 42-register MINB=3 cap)
      default: return v <= 4 ? pick_local<RELU, 2>(v) : pick_local_r<RELU, 48>(v);
    }
  }
  // measured on B200 (profiles/): local-only is best at a 64-register cap
  // (no spills, 36 warps/SM); the remote variant's staging buffer wants the
  // uncapped allocation
  switch (reg_cap_mode()) {
    case 1: return pick_minb<RELU, REMOTE, 1>(v);
    case 2: return pick_minb<RELU, REMOTE, 2>(v);
    case 3: return pick_minb<RELU, REMOTE, 3>(v);
    default: return REMOTE ? pick_minb<RELU, REMOTE, 1>(v) : pick_minb<RELU, REMOTE, 2>(v);
  }
}

int l2_hint() {
  static const int m = [] {
    const char* e = std::getenv("MGG_AGG_L2HINT");  // -1 auto, 0 off, 1 on
    return e ? std::atoi(e) : -1;
  }();
  return m;
}

int group_unroll() {
  static const int m = [] {
    const char* e = std::getenv("MGG_AGG_GROUP_UNR");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

// Local-only K1 flavour for one launch (lean_mode 1 = by the plan's shape).
// Measured (profiles/r01_k1_experiments.md): the warp-window kernel wins
// when most partitions are full ps = 32 windows (Reddit 0.53 vs 0.80 ms,
// Orkut 1.62 vs 1.65); group-per-partition wins on short partitions
// (products-shaped 0.84 -> 0.745 ms at ps 16, Reddit at ps 16 0.92 -> 0.65);
// 8 rows in flight per group with the next column ids prefetched (UNR 4:
// +1%, register caps 40/32 for more warps: +4-10%).
template <bool RELU>
KernelFn pick_lean(uint32_t v, uint32_t ps, uint64_t parts, uint64_t edges,
                   uint32_t granularity, uint32_t form) {
  if (lean_mode() != 1) return pick<RELU, false>(v);
  if (form == 1 || (form > 1 && granularity == 1))
    return v <= 4 ? pick_local<RELU, 2>(v) : pick_local_r<RELU, 48>(v);
  if (form == 2) return v > 2 && v <= 4 && l2_hint() != 0 ? pick_group_hint<RELU>(v)
                                                          : pick_group<RELU, 8>(v);
  if (form == 3) return pick_group<RELU, 4>(v);
  const bool short_parts =
      granularity == 0 && (ps <= 16 || 3 * edges < 2 * static_cast<uint64_t>(ps) * parts);
  // 8 rows in flight per group; MGG_AGG_GROUP_UNR=4 (A/B) is 8% faster on the
  // skewed Orkut-RMAT shape and 1-2% slower on the uniform ones
  // narrow rows (<= 16 floats): L2 evict-last on the gathered rows, evict-first
  // on the column ids and the reductions (products-shaped K1 -1.7%, Orkut
  // -0.5%; the 256-B GIN rows lose 0.5-2% with it, so they go without)
  const bool hint = l2_hint() < 0 ? v > 2 && v <= 4 : l2_hint() == 1 && (v == 4 || v == 16);
  if (short_parts && hint) return pick_group_hint<RELU>(v);
  if (short_parts) return group_unroll() == 4 ? pick_group<RELU, 4>(v) : pick_group<RELU, 8>(v);
  return v <= 4 ? pick_local<RELU, 2>(v) : pick_local_r<RELU, 48>(v);
}

int pair_mode() {
  static const int m = [] {
    // group-per-pair is the default fine-fetch pair loop (the round-1
    // two-process illegal address was the plan-upload race fixed in
    // runtime.cu, not this kernel); MGG_AGG_PAIR=0 = the warp-window loop
    const char* e = std::getenv("MGG_AGG_PAIR");
    return e ? std::atoi(e) : 1;
  }();
  return m;
}

// Paired (local + remote, fine fetch) K1 flavour. Measured (K1 ms per part,
// profiles/r01_k1_experiments.md): the group-per-pair kernel beats the
// warp-window pair loop on every shape and part count tried, full windows
// included (Reddit 2 parts 0.494 -> 0.440, 8 parts 0.201 -> 0.160; products
// at (16,8,8) 1.16 -> 0.50; Orkut at (8,16,8) 2.72 -> 0.91); UNR 8 or PF 8
// spill at the 64-register cap and lose 5-20%, uncapped they lose occupancy.
// MGG_AGG_PAIR=0 keeps the warp-window pair loop (ablations, A/B).
// Whole-list plans (granularity 1, the no_np ablation) keep the warp per
// list of the paper's baseline.
// Logical-CTA schedule of the pair kernels: chunks of MGG_AGG_SCHED logical
// CTAs dealt round-robin, 0 = one contiguous chunk per resident CTA.
// Measured (profiles/r02/hiding_*.jsonl, host-mapped slow peer): chunks of 4
// hide the most remote time (0.74-0.79 vs 0.68 with chunks of 1, 0.28
// contiguous at a 0.03% remote share); the default.
uint32_t sched_mode() {
  static const uint32_t m = [] {
    const char* e = std::getenv("MGG_AGG_SCHED");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 4u;
  }();
  return m;
}

// Dynamic schedule of the group-per-pair kernel (agg_gpair, for_each_ticket):
// MGG_AGG_DYN = 1 (default) dynamic with the ticket size from the launch (1
// or 2 logical warps), N > 1 dynamic with tickets of N logical warps, 0 the
// static round-robin schedule above (also used when MGG_AGG_SCHED=0).
uint32_t dyn_chunk() {
  static const uint32_t m = [] {
    const char* e = std::getenv("MGG_AGG_DYN");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 1u;
  }();
  return m;
}

int pipe_depth() {
  static const int m = [] {
    const char* e = std::getenv("MGG_AGG_PIPE_DEPTH");  // ring slots per lane
    return e ? std::atoi(e) : 8;
  }();
  return m;
}

template <bool RELU>
KernelFn pick_pair(uint32_t v, uint32_t granularity) {
  if (pair_mode() == 0 || granularity == 1) return pick<RELU, true>(v);
  if (pair_mode() == 2) {
    switch (pipe_depth()) {
      case 4: return pick_pipe<RELU, 4>(v);
      case 16: return pick_pipe<RELU, 16>(v);
      default: return pick_pipe<RELU, 8>(v);
    }
  }
  if (pair_mode() == 3) {  // TMA bulk-copy ring
    switch (pipe_depth()) {
      case 4: return pick_pipe_bulk<RELU, 4>(v);
      case 16: return pick_pipe_bulk<RELU, 16>(v);
      default: return pick_pipe_bulk<RELU, 8>(v);
    }
  }
  if (pair_mode() == 4) return pick_gsplit<RELU, 8>(v);  // kind-split tickets
  return pick_gpair<RELU, 4, 4>(v);
}

// Demangled short name of a K1 instantiation ("agg_group_hint<4, false, 8>"),
// cached per function.
const std::string& kernel_name(const void* fn) {
  static std::mutex mu;
  static std::map<const void*, std::string> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(fn);
  if (it != cache.end()) return it->second;
  const char* raw = nullptr;
  std::string name = "?";
  if (cudaFuncGetName(&raw, fn) == cudaSuccess && raw) {
    int st = 0;
    char* dm = abi::__cxa_demangle(raw, nullptr, nullptr, &st);
    name = st == 0 && dm ? dm : raw;
    std::free(dm);
    for (const char* pre : {"void ", "(anonymous namespace)::", "mgg::dev::"})
      for (size_t q; (q = name.find(pre)) != std::string::npos;) name.erase(q, std::strlen(pre));
    const auto paren = name.find('(');  // drop the parameter list
    if (paren != std::string::npos) name.resize(paren);
  } else {
    cudaGetLastError();
  }
  return cache.emplace(fn, name).first->second;
}

// Resident CTAs per SM for (kernel, CTA size), cached per device.
unsigned resident_grid(KernelFn k, int threads, uint32_t pitch) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, unsigned> cache;
  int dev = 0;
  MGG_CUDA(cudaGetDevice(&dev));
  const auto key = std::make_pair(reinterpret_cast<const void*>(k),
                                  (static_cast<int>(pitch) * 1024 + threads) * 64 + dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per_sm = 0, sms = 0;
  const uint32_t smem = dyn_smem(k, threads, pitch);
  if (smem > 48 * 1024)
    MGG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  MGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem));
  MGG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned g = static_cast<unsigned>(std::max(1, per_sm) * sms);
  cache[key] = g;
  return g;
}

// out[r] = scale * f(in[r]) over rows*pitch floats; copy[r] = f(in[r]) when
// given (the activated layer input, so the following K1 gathers it without
// a per-edge ReLU)
template <bool RELU>
__global__ void rows_init_kernel(const float4* __restrict__ in, float4* __restrict__ out,
                                 float4* __restrict__ copy, size_t n4, float scale,
                                 const float* __restrict__ row_scale, uint32_t vec) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    float4 x = __ldg(in + i);
    if (RELU) x = f4relu(x);
    if (row_scale) {  // normalised GCN: the row's D^-1/2 power
      const float r = __ldg(row_scale + i / vec);
      x = make_float4(x.x * r, x.y * r, x.z * r, x.w * r);
    }
    out[i] = make_float4(x.x * scale, x.y * scale, x.z * scale, x.w * scale);
    if (copy) copy[i] = x;
  }
}

// Local column ids lose their owner bits on the device (owner == this part),
// so K1's local gathers index the own shard with no mask.
__global__ void strip_owner_kernel(uint32_t* __restrict__ cols, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    cols[i] &= kMask;
}

// Deduplicated remote fetch: halo[r] = table[owner(r)][offset(r)] for the
// plan's distinct remote rows (sorted by owner, offset: each peer shard is
// streamed in address order). Consecutive threads copy consecutive float4
// of a row: coalesced NVLink reads, coalesced local writes.
__global__ void __launch_bounds__(256) halo_pull_kernel(const uint32_t* __restrict__ rows,
                                                        uint64_t n,
                                                        const float* const* __restrict__ table,
                                                        uint32_t pitch,
                                                        float4* __restrict__ halo) {
  const uint32_t vec = pitch / 4;
  const uint64_t total = n * vec;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
#pragma unroll 4
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
    const uint64_t r = i / vec;
    const uint32_t c4 = static_cast<uint32_t>(i - r * vec);
    const uint32_t c = __ldg(rows + r);
    halo[i] = ld_row4(table[c >> kShift] + static_cast<size_t>(c & kMask) * pitch + 4 * c4);
  }
}

}  // namespace

void launch_halo_pull(const mgg_dplan* p, const mgg_store* in, float* halo, cudaStream_t st) {
  if (!p->halo_len) return;
  const uint64_t total = p->halo_len * (in->pitch / 4);
  const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148 * 8));
  halo_pull_kernel<<<blocks, 256, 0, st>>>(p->halo_rows, p->halo_len, in->dtable[p->part],
                                           in->pitch, reinterpret_cast<float4*>(halo));
  MGG_CUDA(cudaGetLastError());
}

void launch_strip_owner(uint32_t* cols, uint64_t n, cudaStream_t st) {
  if (!n) return;
  const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148 * 8));
  strip_owner_kernel<<<blocks, 256, 0, st>>>(cols, n);
  MGG_CUDA(cudaGetLastError());
}

KernelFn pick_traced_g(uint32_t v) {
  if (v <= 1) return agg_gpair_traced<1, 4>;
  if (v <= 2) return agg_gpair_traced<2, 4>;
  if (v <= 4) return agg_gpair_traced<4, 4>;
  if (v <= 8) return agg_gpair_traced<8, 4>;
  if (v <= 16) return agg_gpair_traced<16, 4>;
  if (v <= 32) return agg_gpair_traced<32, 4>;
  throw Status{MGG_E_CONFIG, "trace: rows wider than 128 floats are not traced"};
}

KernelFn pick_traced(uint32_t v) {
  if (v <= 1) return agg_kernel<1, false, true, 1, true>;
  if (v <= 2) return agg_kernel<2, false, true, 1, true>;
  if (v <= 4) return agg_kernel<4, false, true, 1, true>;
  if (v <= 8) return agg_kernel<8, false, true, 1, true>;
  if (v <= 16) return agg_kernel<16, false, true, 1, true>;
  if (v <= 32) return agg_kernel<32, false, true, 1, true>;
  throw Status{MGG_E_CONFIG, "trace: rows wider than 128 floats are not traced"};
}

// The group-form kernel with the halo pull compiled in (PULL = true) that
// matches a local-pass kernel, or null when the form has none (warp window,
// wide rows, A/B variants): then the pull kernel runs first.
// PULL 1: one halo row per partition, interleaved with the partition's
// gathers; PULL 2: the partition loop untouched, the logical warp's halo rows
// copied after its partitions (MGG_HALO_PULL_MODE, default 2).
int pull_mode() {
  static const int m = [] {
    const char* e = std::getenv("MGG_HALO_PULL_MODE");
    return e && std::atoi(e) == 1 ? 1 : 2;
  }();
  return m;
}
template <int VEC, bool RELU, int M>
void add_pull_pairs(std::map<const void*, KernelFn>& m) {
  m[reinterpret_cast<const void*>(agg_group<VEC, RELU, 8>)] = agg_group<VEC, RELU, 8, M>;
  m[reinterpret_cast<const void*>(agg_group<VEC, RELU, 4>)] = agg_group<VEC, RELU, 4, M>;
}
template <int M>
std::map<const void*, KernelFn> pull_pairs() {
  std::map<const void*, KernelFn> m;
  add_pull_pairs<1, false, M>(m), add_pull_pairs<2, false, M>(m), add_pull_pairs<4, false, M>(m);
  add_pull_pairs<8, false, M>(m), add_pull_pairs<16, false, M>(m), add_pull_pairs<32, false, M>(m);
  add_pull_pairs<1, true, M>(m), add_pull_pairs<2, true, M>(m), add_pull_pairs<4, true, M>(m);
  add_pull_pairs<8, true, M>(m), add_pull_pairs<16, true, M>(m), add_pull_pairs<32, true, M>(m);
  m[reinterpret_cast<const void*>(agg_group_hint<4, false, 8, 0>)] = agg_group_hint<4, false, 8, 0, M>;
  m[reinterpret_cast<const void*>(agg_group_hint<4, true, 8, 0>)] = agg_group_hint<4, true, 8, 0, M>;
  m[reinterpret_cast<const void*>(agg_group_hint<16, false, 8, 0>)] = agg_group_hint<16, false, 8, 0, M>;
  m[reinterpret_cast<const void*>(agg_group_hint<16, true, 8, 0>)] = agg_group_hint<16, true, 8, 0, M>;
  return m;
}
KernelFn pull_variant(KernelFn k) {
  static const std::map<const void*, KernelFn> pairs =
      pull_mode() == 1 ? pull_pairs<1>() : pull_pairs<2>();
  const auto it = pairs.find(reinterpret_cast<const void*>(k));
  return it == pairs.end() ? nullptr : it->second;
}

// Halo pull fused into the local pass (HaloPull) or the pull kernel on the
// aux stream (which, next to a persistent full-occupancy local pass, cannot
// co-run with it): MGG_HALO_FUSE = 1 always fused, 0 never, unset = fused
// when the halo comes over a slower link than the part's own HBM (run_aggregate).
// Measured (profiles/r02/halo_fuse.md): against a slow peer the fused pass
// hides 0.50-0.54 of the remote time where the separate pull hides 0.02-0.05;
// with same-device "peers" (both legs on one HBM) it costs 10-18%.
int halo_fuse_mode() {
  static const int m = [] {
    const char* e = std::getenv("MGG_HALO_FUSE");
    return e ? std::atoi(e) : -1;
  }();
  return m;
}

void launch_aggregate(mgg_ctx* ctx, const mgg_dplan* p, const mgg_store* in,
                      mgg_store* out, int relu_in, int phase, const float* halo,
                      cudaStream_t st, const TraceSink* trace, float* pull_dst) {
  AggArgs a{};
  a.lmeta = p->lmeta;
  a.lcols = p->lcols;
  a.rmeta = p->rmeta;
  a.rcols = halo ? p->rcols_halo : p->rcols;
  a.halo = halo;
  a.table = in->dtable[p->part];
  a.own = in->shard[p->part];
  a.out = out->shard[p->part];
  a.nL = static_cast<uint32_t>(p->n_local);
  a.nR = static_cast<uint32_t>(p->n_remote);
  a.pitch = in->pitch;
  a.vec = in->pitch / 4;
  a.dist = p->dist;
  a.wpb = p->wpb;
  a.mapping = p->mapping;
  a.local_warps = static_cast<uint32_t>(p->num_local_warps);
  a.num_owners = ctx->num_parts;
  a.phase = phase;
  uint64_t warps = p->num_warps;
  if (halo) {
    // Halo mode runs one kind per launch with the local-read kernel: pass 1
    // = the local partitions, pass 2 = the remote partitions gathered from
    // the local halo (remote columns already re-pointed at halo rows).
    if (phase == 2) {
      a.lmeta = p->rmeta;
      a.lcols = p->rcols_halo;
      a.own = halo;
      a.nL = a.nR;
    }
    a.nR = 0;
    a.phase = 0;
    a.mapping = 0;
    a.halo = nullptr;
    warps = (a.nL + a.dist - 1) / a.dist;
  }
  if (pull_dst && (warps == 0 || !halo || phase != 1)) {  // nothing to ride along
    launch_halo_pull(p, in, pull_dst, st);
    count_launch(ctx);
    pull_dst = nullptr;
  }
  if (warps == 0) return;
  if (warps > 0xffffffffull) throw Status{MGG_E_CONFIG, "aggregate: too many warps"};
  a.num_warps = static_cast<uint32_t>(warps);
  a.num_lblocks = (a.num_warps + a.wpb - 1) / a.wpb;
  // phase 3 (fine fetch, timing decomposition): the local partitions only,
  // through the pipelined pair kernel itself — its own local leg, so that
  // T_pipe vs T_local + T_remote compares one kernel with itself
  if (phase == 3) a.phase = 1;
  const bool remote = a.nR > 0 && (a.phase != 1 || (phase == 3 && !halo));
  const bool remote_lean = halo && phase == 2;
  const uint64_t lparts = remote_lean ? p->n_remote : p->n_local;
  const uint64_t ledges = remote_lean ? p->remote_edges : p->local_edges;
  a.strided = remote && p->granularity == 0 && pair_mode() != 0 ? sched_mode() : 0;
  const bool dynamic =
      a.strided && (pair_mode() == 1 || pair_mode() == 4) && dyn_chunk() != 0;
  KernelFn k = remote ? (relu_in ? pick_pair<true>(a.vec, p->granularity)
                                 : pick_pair<false>(a.vec, p->granularity))
                      : (relu_in ? pick_lean<true>(a.vec, p->ps, lparts, ledges, p->granularity, p->k1_form)
                                 : pick_lean<false>(a.vec, p->ps, lparts, ledges, p->granularity, p->k1_form));
  if (trace) {  // the pipelined kernel with stage stamps, whatever the plan
    if (relu_in || halo) throw Status{MGG_E_CONFIG, "trace: fine-grained, no ReLU-on-load"};
    // the pair kernel that runs untraced: group-per-pair unless the
    // warp-window loop is selected (MGG_AGG_PAIR=0) or the plan is whole-list
    k = pair_mode() == 0 || p->granularity == 1 ? pick_traced(a.vec) : pick_traced_g(a.vec);
    a.trace = reinterpret_cast<uint4*>(trace->events);
    a.trace_n = reinterpret_cast<unsigned long long*>(trace->count);
    a.trace_cap = trace->capacity;
    a.trace_warps = trace->warp_limit;
  }
  if (pull_dst) {
    if (KernelFn kp = pull_variant(k)) {
      k = kp;
      a.pull_rows = p->halo_rows;
      a.pull_n = p->halo_len;
      a.pull_dst = pull_dst;
    } else {  // warp-window / wide forms carry no pull: copy first
      launch_halo_pull(p, in, pull_dst, st);
      count_launch(ctx);
    }
  }
  const int threads = 32 * static_cast<int>(p->wpb);
  const unsigned full = resident_grid(k, threads, a.pitch);
  const unsigned grid = std::min<unsigned>(full, a.num_lblocks);
  if (dynamic) {
    a.sched = p->sched;
    // tickets of 2 logical warps when that still leaves >= 16 per resident
    // warp, else 1 (or the knob). Measured (profiles/r02/dyn_schedule.md):
    // 2 and 4 hide the same, 4+ loses parallelism on small plans.
    const uint64_t rw = uint64_t(grid) * p->wpb;
    a.wchunk = dyn_chunk() > 1 ? dyn_chunk() : (a.num_warps >= 32 * rw ? 2u : 1u);
  }
  k<<<grid, threads, dyn_smem(k, threads, a.pitch), st>>>(a);
  {
    int dev = 0, sms = 0;
    MGG_CUDA(cudaGetDevice(&dev));
    MGG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    p->last_grid = grid;
    p->last_threads = static_cast<uint32_t>(threads);
    p->last_sms = static_cast<uint32_t>(sms);
    p->last_resident = full / std::max(1, sms);
  }
  MGG_CUDA(cudaGetLastError());
  count_launch(ctx);
  if (!p->k1_names.empty()) p->k1_names += ';';
  p->k1_names += kernel_name(reinterpret_cast<const void*>(k));
}

void launch_rows_init(const float* in, float* out, uint64_t rows, uint32_t pitch,
                      float scale, int relu_in, float* copy, cudaStream_t st,
                      const float* row_scale) {
  const size_t n4 = rows * (size_t)pitch / 4;
  if (n4 == 0) return;
  const unsigned blocks =
      static_cast<unsigned>(std::min<size_t>((n4 + 255) / 256, 148 * 16));
  auto* o = reinterpret_cast<float4*>(out);
  auto* c = reinterpret_cast<float4*>(copy);
  if (relu_in)
    rows_init_kernel<true><<<blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(in), o, c,
                                                   n4, scale, row_scale, pitch / 4);
  else
    rows_init_kernel<false><<<blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(in), o, c,
                                                    n4, scale, row_scale, pitch / 4);
  MGG_CUDA(cudaGetLastError());
}

}  // namespace mgg::dev
