// K5 — hardware probes behind the b200 cost-model profile and the roofline
// denominators the vendor copy benchmark does not give:
//   * gather: sum rows table[idx[i]] (idx streamed, rows of `pitch` floats)
//     with the same lane layout as K1 but no plan, no atomics — the ceiling
//     of the aggregation's gather phase for a given table size (L2-resident
//     or HBM-resident) and for peer (NVLink) tables;
//   * chase: dependent loads through a random cycle — load latency of the
//     memory a pointer lands in (local HBM, L2, or a peer GPU over NVLink).
#include <cuda_runtime.h>

#include "common.cuh"

namespace mgg::dev {
namespace {

template <int VEC>
__global__ void __launch_bounds__(256) gather_probe(const float* __restrict__ table,
                                                    const uint32_t* __restrict__ idx,
                                                    uint64_t n, uint32_t pitch,
                                                    float* __restrict__ sink) {
  constexpr int RPW = 32 / VEC;
  const int lane = threadIdx.x & 31, sub = lane / VEC, v = lane % VEC;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint64_t base = warp * 32 * 4; base < n; base += nw * 32 * 4) {
    uint32_t w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t k = base + u * 32 + lane;
      w[u] = k < n ? __ldg(idx + k) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float4 t[32 / RPW > 4 ? 4 : 32 / RPW];
      constexpr int S = 32 / RPW;
#pragma unroll
      for (int s0 = 0; s0 < S; s0 += 4) {
#pragma unroll
        for (int q = 0; q < 4 && s0 + q < S; ++q) {
          const int r = (s0 + q) * RPW + sub;
          const uint32_t c = __shfl_sync(0xffffffffu, w[u], r);
          const bool ok = base + u * 32 + r < n;
          t[q] = ok ? __ldg(reinterpret_cast<const float4*>(table + (size_t)c * pitch + 4 * v))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < 4 && s0 + q < S; ++q) {
          acc.x += t[q].x;
          acc.y += t[q].y;
          acc.z += t[q].z;
          acc.w += t[q].w;
        }
      }
    }
  }
  const float s = acc.x + acc.y + acc.z + acc.w;
  if (s == 12345.678f) sink[0] = s;  // keep the loads alive
}

__global__ void chase_probe(const uint32_t* __restrict__ next, uint32_t steps, uint32_t* out) {
  uint32_t p = 0;
  for (uint32_t i = 0; i < steps; ++i) p = __ldcg(next + p);
  *out = p;
}

}  // namespace
}  // namespace mgg::dev

using namespace mgg::dev;

extern "C" int mgg_probe_gather(mgg_ctx* ctx, uint32_t part, const float* table,
                                uint32_t pitch, const uint32_t* idx, uint64_t n,
                                uint32_t reps, double* gbps) {
  try {
    cudaStream_t st = enter(ctx, part);
    float* sink = nullptr;
    MGG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sink), 16, st));
    int dev = 0, sms = 0;
    MGG_CUDA(cudaGetDevice(&dev));
    MGG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned grid = static_cast<unsigned>(sms * 8);
    auto launch = [&] {
      const uint32_t vec = pitch / 4;
      if (vec <= 4) gather_probe<4><<<grid, 256, 0, st>>>(table, idx, n, pitch, sink);
      else if (vec <= 8) gather_probe<8><<<grid, 256, 0, st>>>(table, idx, n, pitch, sink);
      else if (vec <= 16) gather_probe<16><<<grid, 256, 0, st>>>(table, idx, n, pitch, sink);
      else gather_probe<32><<<grid, 256, 0, st>>>(table, idx, n, pitch, sink);
    };
    launch();
    cudaEvent_t e0, e1;
    MGG_CUDA(cudaEventCreate(&e0));
    MGG_CUDA(cudaEventCreate(&e1));
    MGG_CUDA(cudaEventRecord(e0, st));
    for (uint32_t r = 0; r < reps; ++r) launch();
    MGG_CUDA(cudaEventRecord(e1, st));
    MGG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    MGG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    MGG_CUDA(cudaFreeAsync(sink, st));
    MGG_CUDA(cudaGetLastError());
    *gbps = static_cast<double>(n) * pitch * 4 * reps / (ms * 1e-3) / 1e9;
    count_launch(ctx, reps + 1);
    return MGG_OK;
  } catch (const Status& s) {
    last_error() = s.msg;
    return s.code;
  }
}

extern "C" int mgg_probe_chase(mgg_ctx* ctx, uint32_t part, const uint32_t* next,
                               uint32_t steps, double* ns_per_load) {
  try {
    cudaStream_t st = enter(ctx, part);
    uint32_t* out = nullptr;
    MGG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out), 16, st));
    chase_probe<<<1, 1, 0, st>>>(next, 64, out);
    cudaEvent_t e0, e1;
    MGG_CUDA(cudaEventCreate(&e0));
    MGG_CUDA(cudaEventCreate(&e1));
    MGG_CUDA(cudaEventRecord(e0, st));
    chase_probe<<<1, 1, 0, st>>>(next, steps, out);
    MGG_CUDA(cudaEventRecord(e1, st));
    MGG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    MGG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    MGG_CUDA(cudaFreeAsync(out, st));
    MGG_CUDA(cudaGetLastError());
    *ns_per_load = ms * 1e6 / steps;
    count_launch(ctx, 2);
    return MGG_OK;
  } catch (const Status& s) {
    last_error() = s.msg;
    return s.code;
  }
}
