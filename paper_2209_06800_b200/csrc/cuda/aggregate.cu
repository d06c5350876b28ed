// K1 — MGG pipelined neighbor aggregation for sm_100a.
//
// One kernel per part consumes that part's FlatPlan as-is: CTA = wpb warps,
// warp w owns partitions [w·dist, (w+1)·dist) of the local list and of the
// remote list (interleaved mapping, R:proj/src/workload.cpp:103-124), or the
// local groups then the remote groups (segregated, 126-146). Inside a warp
// the pair loop follows the async discipline of the reference's per-warp
// program (R:proj/src/sim.cpp:102-125, paper Fig. 6b):
//
//   for pair i:  issue remote-row loads of R_i         (peer shard, NVLink)
//                reduce local partition L_i            (own shard, HBM/L2)
//                consume R_i                            (registers)
//
// so the NVLink latency of R_i is covered by L_i's local work, tile by tile,
// inside one kernel and without any host round trip or NCCL call.
//
// Lane layout: a row of `vec` float4 is covered by VEC (>= vec, power of 2)
// lanes; a warp step gathers RPW = 32/VEC rows with one 128-bit load per
// lane (coalesced per row). Partials for one target stay in registers while
// consecutive partitions of the warp share that target (owner combine), then
// fold across the RPW row groups with shuffles and land in `out` with one
// 128-bit vector reduction per lane (REDG.ADD.F32x4).
//
// Rows wider than 128 floats (VEC > 32) use the wide variant: each lane owns
// float4 columns lane, lane+32, ... and walks the partition row by row.
#include <cuda_runtime.h>

#include "common.cuh"

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
  uint32_t dist;
  uint32_t mapping;           // 0 interleaved, 1 segregated
  uint32_t local_warps;       // segregated: warps holding local groups
  uint32_t num_owners;
  int phase;                  // 0 all, 1 local only, 2 remote only
};

constexpr uint32_t kShift = 28;
constexpr uint32_t kMask = (1u << kShift) - 1;

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 f4relu(float4 a) {
  return make_float4(fmaxf(a.x, 0.f), fmaxf(a.y, 0.f), fmaxf(a.z, 0.f),
                     fmaxf(a.w, 0.f));
}
__device__ __forceinline__ float4 ld_row4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void red_add4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

struct Part {
  int target, begin, end;
};
__device__ __forceinline__ Part load_part(const int2* meta, uint32_t i) {
  const int2 a = __ldg(meta + i);
  const int2 b = __ldg(meta + i + 1);
  return {a.x, a.y, b.y};
}

// Warp-uniform ranges [l0,l1) of local and [r0,r1) of remote partitions.
__device__ __forceinline__ void warp_groups(const AggArgs& a, uint32_t w,
                                            uint32_t& l0, uint32_t& l1,
                                            uint32_t& r0, uint32_t& r1) {
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

// ---------------------------------------------------------------------------
// Narrow rows: VEC lanes per row, RPW rows per warp step.

template <int VEC, bool RELU>
struct Narrow {
  static constexpr int RPW = 32 / VEC;
  static constexpr int PF = 4;  // remote steps staged ahead (registers)

  int lane, sub, v;
  bool vlane;  // lane covers a real float4 of the row

  __device__ __forceinline__ Narrow(uint32_t vec) {
    lane = threadIdx.x & 31;
    sub = lane / VEC;
    v = lane % VEC;
    vlane = v < (int)vec;
  }

  __device__ __forceinline__ float4 fetch(const AggArgs& a,
                                          const uint32_t* __restrict__ cols,
                                          const Part& p, int step, bool remote,
                                          const float* const* tab) const {
    const int k = p.begin + step * RPW + sub;
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (vlane && k < p.end) {
      const uint32_t c = __ldg(cols + k);
      const float* base = remote ? tab[c >> kShift] : a.own;
      r = ld_row4(base + (size_t)(c & kMask) * a.pitch + 4 * v);
      if (RELU) r = f4relu(r);
    }
    return r;
  }

  __device__ __forceinline__ void flush(const AggArgs& a, float4 acc,
                                        int target) const {
#pragma unroll
    for (int off = 16; off >= VEC; off >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
      acc.z += __shfl_xor_sync(0xffffffffu, acc.z, off);
      acc.w += __shfl_xor_sync(0xffffffffu, acc.w, off);
    }
    if (sub == 0 && vlane) red_add4(a.out + (size_t)target * a.pitch + 4 * v, acc);
  }

  // Reduce partition p (all steps) into acc.
  __device__ __forceinline__ float4 reduce(const AggArgs& a,
                                           const uint32_t* __restrict__ cols,
                                           const Part& p, bool remote,
                                           const float* const* tab,
                                           float4 acc, int first_step) const {
    const int steps = (p.end - p.begin + RPW - 1) / RPW;
    for (int s = first_step; s < steps; s += 4) {
      float4 t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        t[u] = (s + u < steps) ? fetch(a, cols, p, s + u, remote, tab)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = f4add(acc, t[u]);
    }
    return acc;
  }
};

template <int VEC, bool RELU>
__global__ void __launch_bounds__(512) agg_narrow(AggArgs a) {
  __shared__ const float* tab[kMaxParts];
  if (threadIdx.x < a.num_owners) tab[threadIdx.x] = a.table[threadIdx.x];
  __syncthreads();

  const uint32_t w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  uint32_t l0, l1, r0, r1;
  warp_groups(a, w, l0, l1, r0, r1);
  const uint32_t nl = l1 - l0, nr = r1 - r0;
  if (nl == 0 && nr == 0) return;

  using N = Narrow<VEC, RELU>;
  const N n(a.vec);
  float4 accL = make_float4(0.f, 0.f, 0.f, 0.f), accR = accL;
  int curL = -1, curR = -1;
  const uint32_t pairs = max(nl, nr);

  for (uint32_t i = 0; i < pairs; ++i) {
    // (1) issue remote-row loads for R_i (first PF steps stay in flight)
    Part rp{};
    float4 pre[N::PF];
    const bool has_r = i < nr;
    if (has_r) {
      rp = load_part(a.rmeta, r0 + i);
#pragma unroll
      for (int s = 0; s < N::PF; ++s)
        pre[s] = n.fetch(a, a.rcols, rp, s, true, tab);
    }
    // (2) reduce the paired local partition L_i while R_i is in flight
    if (i < nl) {
      const Part lp = load_part(a.lmeta, l0 + i);
      if (lp.target != curL) {
        if (curL >= 0) n.flush(a, accL, curL);
        accL = make_float4(0.f, 0.f, 0.f, 0.f);
        curL = lp.target;
      }
      accL = n.reduce(a, a.lcols, lp, false, tab, accL, 0);
    }
    // (3) consume R_i
    if (has_r) {
      if (rp.target != curR) {
        if (curR >= 0) n.flush(a, accR, curR);
        accR = make_float4(0.f, 0.f, 0.f, 0.f);
        curR = rp.target;
      }
#pragma unroll
      for (int s = 0; s < N::PF; ++s) accR = f4add(accR, pre[s]);
      accR = n.reduce(a, a.rcols, rp, true, tab, accR, N::PF);
    }
  }
  if (curL >= 0) n.flush(a, accL, curL);
  if (curR >= 0) n.flush(a, accR, curR);
}

// ---------------------------------------------------------------------------
// Wide rows (vec > 32 float4): lanes own columns, rows walked one by one.

template <bool RELU>
__global__ void __launch_bounds__(512) agg_wide(AggArgs a) {
  __shared__ const float* tab[kMaxParts];
  if (threadIdx.x < a.num_owners) tab[threadIdx.x] = a.table[threadIdx.x];
  __syncthreads();

  const uint32_t w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  uint32_t l0, l1, r0, r1;
  warp_groups(a, w, l0, l1, r0, r1);
  const uint32_t nl = l1 - l0, nr = r1 - r0;
  if (nl == 0 && nr == 0) return;
  const int lane = threadIdx.x & 31;
  constexpr int CH = 4;  // float4 columns per lane per pass

  for (uint32_t c0 = 0; c0 < a.vec; c0 += 32 * CH) {
    for (int kind = 0; kind < 2; ++kind) {
      const bool remote = kind == 1;
      const uint32_t b = remote ? r0 : l0, cnt = remote ? nr : nl;
      const int2* meta = remote ? a.rmeta : a.lmeta;
      const uint32_t* cols = remote ? a.rcols : a.lcols;
      float4 acc[CH];
      int cur = -1;
      for (uint32_t i = 0; i < cnt; ++i) {
        const Part p = load_part(meta, b + i);
        if (p.target != cur) {
          if (cur >= 0)
#pragma unroll
            for (int j = 0; j < CH; ++j) {
              const uint32_t col = c0 + lane + 32 * j;
              if (col < a.vec) red_add4(a.out + (size_t)cur * a.pitch + 4 * col, acc[j]);
            }
#pragma unroll
          for (int j = 0; j < CH; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
          cur = p.target;
        }
        for (int k = p.begin; k < p.end; ++k) {
          const uint32_t c = __ldg(cols + k);
          const float* row =
              (remote ? tab[c >> kShift] : a.own) + (size_t)(c & kMask) * a.pitch;
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

template <bool RELU>
void dispatch(const AggArgs& a, dim3 grid, dim3 block, cudaStream_t st) {
  const uint32_t v = a.vec;
  if (v <= 1) agg_narrow<1, RELU><<<grid, block, 0, st>>>(a);
  else if (v <= 2) agg_narrow<2, RELU><<<grid, block, 0, st>>>(a);
  else if (v <= 4) agg_narrow<4, RELU><<<grid, block, 0, st>>>(a);
  else if (v <= 8) agg_narrow<8, RELU><<<grid, block, 0, st>>>(a);
  else if (v <= 16) agg_narrow<16, RELU><<<grid, block, 0, st>>>(a);
  else if (v <= 32) agg_narrow<32, RELU><<<grid, block, 0, st>>>(a);
  else agg_wide<RELU><<<grid, block, 0, st>>>(a);
}

// out[r] = scale * f(in[r]) over rows*pitch floats
template <bool RELU>
__global__ void rows_init_kernel(const float4* __restrict__ in, float4* __restrict__ out,
                                 size_t n4, float scale) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    float4 x = __ldg(in + i);
    if (RELU) x = f4relu(x);
    out[i] = make_float4(x.x * scale, x.y * scale, x.z * scale, x.w * scale);
  }
}

}  // namespace

void launch_aggregate(mgg_ctx* ctx, const mgg_dplan* p, const mgg_store* in,
                      mgg_store* out, int relu_in, int phase, cudaStream_t st) {
  AggArgs a{};
  a.lmeta = p->lmeta;
  a.lcols = p->lcols;
  a.rmeta = p->rmeta;
  a.rcols = p->rcols;
  a.table = in->dtable[p->part];
  a.own = in->shard[p->part];
  a.out = out->shard[p->part];
  a.nL = static_cast<uint32_t>(p->n_local);
  a.nR = static_cast<uint32_t>(p->n_remote);
  a.pitch = in->pitch;
  a.vec = in->pitch / 4;
  a.dist = p->dist;
  a.mapping = p->mapping;
  a.local_warps = static_cast<uint32_t>(p->num_local_warps);
  a.num_owners = ctx->num_parts;
  a.phase = phase;
  if (p->num_warps == 0) return;
  const uint64_t blocks = (p->num_warps + p->wpb - 1) / p->wpb;
  if (blocks > 0x7fffffffull) throw Status{MGG_E_CONFIG, "aggregate: grid too large"};
  const dim3 grid(static_cast<unsigned>(blocks)), block(32 * p->wpb);
  if (relu_in)
    dispatch<true>(a, grid, block, st);
  else
    dispatch<false>(a, grid, block, st);
  MGG_CUDA(cudaGetLastError());
  count_launch(ctx);
}

void launch_rows_init(const float* in, float* out, uint64_t rows, uint32_t pitch,
                      float scale, int relu_in, cudaStream_t st) {
  const size_t n4 = rows * (size_t)pitch / 4;
  if (n4 == 0) return;
  const unsigned blocks =
      static_cast<unsigned>(std::min<size_t>((n4 + 255) / 256, 148 * 16));
  if (relu_in)
    rows_init_kernel<true><<<blocks, 256, 0, st>>>(
        reinterpret_cast<const float4*>(in), reinterpret_cast<float4*>(out), n4, scale);
  else
    rows_init_kernel<false><<<blocks, 256, 0, st>>>(
        reinterpret_cast<const float4*>(in), reinterpret_cast<float4*>(out), n4, scale);
  MGG_CUDA(cudaGetLastError());
}

}  // namespace mgg::dev
