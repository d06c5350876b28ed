// Standalone micro-benchmark: can TMA gather4 beat LSU row gathers for K1?
//
// K1 (aggregate.cu) sums random feature rows of 64-256 B. Its ncu profile is
// L1TEX-wavefront bound.  This probe times the same random-row summation two
// ways on one GPU:
//   ldg : lanes split a row into float4 pieces (what K1 does today)
//   g4  : one lane per warp issues cp.async.bulk.tensor...tile::gather4 (4
//         rows per instruction) into a per-warp shared-memory ring; the warp
//         sums rows out of shared memory.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/gather4_probe
//        tools/gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                        int col, int4 r) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(col), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(bar)
      : "memory");
}

constexpr int kWarps = 8;

// LSU path: D/4 lanes per row, 32/(D/4) rows per warp instruction.
template <int D>
__global__ void __launch_bounds__(256) k_ldg(const float* __restrict__ x,
                                             const int* __restrict__ idx, long n_idx,
                                             float* __restrict__ out) {
  constexpr int L = D / 4, R = 32 / L;
  const int lane = threadIdx.x & 31;
  const long gw = static_cast<long>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const long tw = static_cast<long>(gridDim.x) * kWarps;
  const long per = (n_idx / 32 + tw - 1) / tw * 32;
  const long b = gw * per, e = min(b + per, n_idx);
  float4 acc = make_float4(0, 0, 0, 0);
  for (long base = b; base < e; base += 32) {
    const int id = base + lane < e ? __ldg(idx + base + lane) : -1;
#pragma unroll 4
    for (int s = 0; s < 32 / R; ++s) {
      const int row = __shfl_sync(0xffffffffu, id, s * R + lane / L);
      if (row >= 0) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(x + static_cast<long>(row) * D) +
                               (lane % L));
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
  }
  out[static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// TMA path: lane 0 keeps S gather4s in flight per warp.
template <int D, int S>
__global__ void __launch_bounds__(256) k_g4(const __grid_constant__ CUtensorMap tm,
                                            const int* __restrict__ idx, long n_idx,
                                            float* __restrict__ out) {
  constexpr int SLOT = 4 * D * 4;  // bytes per gather4
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * S * SLOT;
  const uint32_t ring_s = su32(ring);
  const uint32_t bar_s = su32(smem + kWarps * S * SLOT) + warp * S * 8;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(bar_s + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const long gw = static_cast<long>(blockIdx.x) * kWarps + warp;
  const long tw = static_cast<long>(gridDim.x) * kWarps;
  const long n_groups = n_idx / 4;
  const long per = (n_groups / 32 + tw - 1) / tw * 32;  // groups per warp
  const long g0 = gw * per, g1 = min(g0 + per, n_groups);
  const long ng = g1 > g0 ? g1 - g0 : 0;
  const int4* gidx = reinterpret_cast<const int4*>(idx) + g0;
  // group ids come in 32-wide batches loaded by the whole warp
  int4 cur = lane < ng ? gidx[lane] : make_int4(0, 0, 0, 0);
  int4 nxt = 32 + lane < ng ? gidx[32 + lane] : make_int4(0, 0, 0, 0);
  auto issue = [&](long j) {  // warp-uniform j, j < ng
    const int sl = static_cast<int>(j & 31);
    int4 r;
    r.x = __shfl_sync(0xffffffffu, cur.x, sl);
    r.y = __shfl_sync(0xffffffffu, cur.y, sl);
    r.z = __shfl_sync(0xffffffffu, cur.z, sl);
    r.w = __shfl_sync(0xffffffffu, cur.w, sl);
    if (lane == 0) {
      const int s = static_cast<int>(j % S);
      mbar_expect_tx(bar_s + 8 * s, SLOT);
      gather4(ring_s + s * SLOT, &tm, bar_s + 8 * s, 0, r);
    }
    if (sl == 31) {
      cur = nxt;
      const long q = j + 33 + lane;
      nxt = q < ng ? gidx[q] : make_int4(0, 0, 0, 0);
    }
  };
  float acc = 0.f;
  const long pro = ng < S ? ng : S;
  for (long j = 0; j < pro; ++j) issue(j);
  for (long j = 0; j < ng; ++j) {
    const int s = static_cast<int>(j % S);
    mbar_wait(bar_s + 8 * s, static_cast<uint32_t>((j / S) & 1));
    const float* slot = reinterpret_cast<const float*>(ring + s * SLOT);
#pragma unroll
    for (int k = 0; k < 4 * D / 32; ++k) acc += slot[k * 32 + lane];
    __syncwarp();
    if (j + S < ng) issue(j + S);
  }
  out[static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x] = acc;
}

// Hybrid: per 32-row window, rows [0, 32-T) through the LSU (K1's mapping:
// 4 lanes x float4 per 64-B row, 8 rows per step, all loads of the window in
// flight) and rows [32-T, 32) through TMA gather4 into a per-warp smem ring
// issued S windows ahead by lane 0. Both engines work on the same window
// stream: does the TMA path ADD to the LSU's row rate?
template <int T, int S>
__global__ void __launch_bounds__(512) k_hybrid(const __grid_constant__ CUtensorMap tm,
                                                const float* __restrict__ x,
                                                const int* __restrict__ idx, long n_idx,
                                                float* __restrict__ out) {
  constexpr int D = 16, SLOT = T * D * 4 > 0 ? T * D * 4 : 16;
  constexpr int WARPS = 16;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * S * SLOT;
  const uint32_t ring_s = su32(ring);
  const uint32_t bar_s = su32(smem + WARPS * S * SLOT) + warp * S * 8;
  if (T > 0 && lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(bar_s + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const long gw = static_cast<long>(blockIdx.x) * WARPS + warp;
  const long tw = static_cast<long>(gridDim.x) * WARPS;
  const long nwin = n_idx / 32;
  const long per = (nwin + tw - 1) / tw;
  const long w0 = gw * per, w1 = min(w0 + per, nwin);
  const long nw = w1 > w0 ? w1 - w0 : 0;
  const int sub = lane / 4, v = lane % 4;
  float4 acc = make_float4(0, 0, 0, 0);
  auto issue = [&](long j) {  // window j's TMA rows (warp-uniform j < nw)
    if (T == 0) return;
    const int id = __ldg(idx + (w0 + j) * 32 + lane);
    const int s = static_cast<int>(j % S);
    int4 r[T / 4 > 0 ? T / 4 : 1];
#pragma unroll
    for (int q = 0; q < T / 4; ++q) {
      r[q].x = __shfl_sync(0xffffffffu, id, 32 - T + 4 * q);
      r[q].y = __shfl_sync(0xffffffffu, id, 32 - T + 4 * q + 1);
      r[q].z = __shfl_sync(0xffffffffu, id, 32 - T + 4 * q + 2);
      r[q].w = __shfl_sync(0xffffffffu, id, 32 - T + 4 * q + 3);
    }
    if (lane == 0) {
      mbar_expect_tx(bar_s + 8 * s, T * D * 4);
#pragma unroll
      for (int q = 0; q < T / 4; ++q)
        gather4(ring_s + s * SLOT + q * 4 * D * 4, &tm, bar_s + 8 * s, 0, r[q]);
    }
  };
  const long pro = nw < S ? nw : S;
  for (long j = 0; j < pro; ++j) issue(j);
  for (long j = 0; j < nw; ++j) {
    const int id = __ldg(idx + (w0 + j) * 32 + lane);
    constexpr int LSTEPS = (32 - T) / 8;  // LSU steps of 8 rows
    float4 t[LSTEPS > 0 ? LSTEPS : 1];
#pragma unroll
    for (int q = 0; q < LSTEPS; ++q) {
      const int row = __shfl_sync(0xffffffffu, id, q * 8 + sub);
      t[q] = __ldg(reinterpret_cast<const float4*>(x + static_cast<long>(row) * D) + v);
    }
#pragma unroll
    for (int q = 0; q < LSTEPS; ++q) {
      acc.x += t[q].x; acc.y += t[q].y; acc.z += t[q].z; acc.w += t[q].w;
    }
    if (T > 0) {
      const int s = static_cast<int>(j % S);
      mbar_wait(bar_s + 8 * s, static_cast<uint32_t>((j / S) & 1));
      const float4* slot = reinterpret_cast<const float4*>(ring + s * SLOT);
#pragma unroll
      for (int q = 0; q < T / 8; ++q) {  // 8 rows x 4 float4 per pass
        const float4 u = slot[q * 32 + lane];
        acc.x += u.x; acc.y += u.y; acc.z += u.z; acc.w += u.w;
      }
      __syncwarp();
      if (j + S < nw) issue(j + S);
    }
  }
  out[static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// 64-B rows, K1-like mapping, 128-bit (4 lanes per row, 8 rows per warp
// step) vs 256-bit loads (2 lanes per row, 16 rows per step): is the L1TEX
// cost per row or per load instruction?
template <int W>  // bytes per lane load: 16 or 32
__global__ void __launch_bounds__(512) k_vec(const float* __restrict__ x,
                                             const int* __restrict__ idx, long n_idx,
                                             float* __restrict__ out) {
  constexpr int D = 16, L = 64 / W, R = 32 / L;  // lanes per row, rows per step
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long gw = static_cast<long>(blockIdx.x) * 16 + warp;
  const long tw = static_cast<long>(gridDim.x) * 16;
  const long nwin = n_idx / 32;
  const long per = (nwin + tw - 1) / tw;
  const long w0 = gw * per, w1 = min(w0 + per, nwin);
  const int sub = lane / L, v = lane % L;
  float acc[W / 4] = {};
  for (long j = w0; j < w1; ++j) {
    const int id = __ldg(idx + j * 32 + lane);
#pragma unroll
    for (int q = 0; q < 32 / R; ++q) {
      const int row = __shfl_sync(0xffffffffu, id, q * R + sub);
      const float* p = x + static_cast<long>(row) * D + v * (W / 4);
      if (W == 16) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        acc[0] += t.x; acc[1] += t.y; acc[2] += t.z; acc[3] += t.w;
      } else {
        float r[8];
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                       "=f"(r[6]), "=f"(r[7])
                     : "l"(p));
#pragma unroll
        for (int i = 0; i < W / 4; ++i) acc[i] += r[i % 8];
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < W / 4; ++i) s += acc[i];
  out[static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x] = s;
}

void run_vec(long rows, long n_idx) {
  std::vector<int> h(n_idx);
  std::mt19937_64 g(42);
  for (auto& v : h) v = static_cast<int>(g() % rows);
  float *x, *out;
  int* idx;
  CK(cudaMalloc(&x, rows * 16 * 4));
  CK(cudaMemset(x, 0, rows * 16 * 4));
  CK(cudaMalloc(&idx, n_idx * 4));
  CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&out, static_cast<size_t>(148) * 4 * 512 * 4));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const double bytes = static_cast<double>(n_idx) * 64;
  for (int per_sm : {2, 3, 4}) {
    float best[2] = {1e30f, 1e30f};
    for (int impl = 0; impl < 2; ++impl)
      for (int it = 0; it < 6; ++it) {
        CK(cudaEventRecord(a));
        if (impl == 0)
          k_vec<16><<<148 * per_sm, 512>>>(x, idx, n_idx, out);
        else
          k_vec<32><<<148 * per_sm, 512>>>(x, idx, n_idx, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (it > 0 && ms < best[impl]) best[impl] = ms;
      }
    std::printf("vec rows=%ld ctas/sm=%d  128-bit: %.3f ms %.0f GB/s | 256-bit: %.3f ms %.0f GB/s\n",
                rows, per_sm, best[0], bytes / best[0] / 1e6, best[1], bytes / best[1] / 1e6);
  }
  CK(cudaFree(x));
  CK(cudaFree(idx));
  CK(cudaFree(out));
}

static PFN_cuTensorMapEncodeTiled encode_fn() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess) std::exit(2);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
}

template <int D, int S>
void run(long rows, long n_idx, int grid_mult) {
  std::vector<int> h(n_idx);
  std::mt19937_64 g(42);
  for (auto& v : h) v = static_cast<int>(g() % rows);
  float *x, *out;
  int* idx;
  CK(cudaMalloc(&x, rows * D * 4));
  CK(cudaMemset(x, 0, rows * D * 4));
  CK(cudaMalloc(&idx, n_idx * 4));
  CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int grid = sms * grid_mult;
  CK(cudaMalloc(&out, static_cast<size_t>(grid) * 256 * 4));
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(D) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(D), 1};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::printf("encode failed %d\n", r);
    std::exit(3);
  }
  const size_t smem = kWarps * S * 4 * D * 4 + kWarps * S * 8;
  CK(cudaFuncSetAttribute(k_g4<D, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(smem)));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const double bytes = static_cast<double>(n_idx) * D * 4;
  for (int impl = 0; impl < 2; ++impl) {
    float best = 1e30f;
    for (int it = 0; it < 6; ++it) {
      CK(cudaEventRecord(a));
      if (impl == 0)
        k_ldg<D><<<grid, 256>>>(x, idx, n_idx, out);
      else
        k_g4<D, S><<<grid, 256, smem>>>(m, idx, n_idx, out);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaGetLastError());
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, a, b));
      if (it > 0 && ms < best) best = ms;
    }
    std::printf("D=%3d S=%2d rows=%8ld idx=%ld grid=%dx148 %-4s %8.3f ms  %7.1f GB/s\n", D, S,
                rows, n_idx, grid_mult, impl ? "g4" : "ldg", best, bytes / best / 1e6);
  }
  CK(cudaFree(x));
  CK(cudaFree(idx));
  CK(cudaFree(out));
}

template <int T, int S>
float time_hybrid(const CUtensorMap& m, const float* x, const int* idx, long n_idx, float* out,
                  int per_sm) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  constexpr int SLOT = T * 16 * 4 > 0 ? T * 16 * 4 : 16;
  const size_t smem = 16 * S * SLOT + 16 * S * 8;
  CK(cudaFuncSetAttribute(k_hybrid<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(smem)));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int it = 0; it < 6; ++it) {
    CK(cudaEventRecord(a));
    k_hybrid<T, S><<<sms * per_sm, 512, smem>>>(m, x, idx, n_idx, out);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (it > 0 && ms < best) best = ms;
  }
  return best;
}

void run_hybrid(long rows, long n_idx) {
  constexpr int D = 16;
  std::vector<int> h(n_idx);
  std::mt19937_64 g(42);
  for (auto& v : h) v = static_cast<int>(g() % rows);
  float *x, *out;
  int* idx;
  CK(cudaMalloc(&x, rows * D * 4));
  CK(cudaMemset(x, 0, rows * D * 4));
  CK(cudaMalloc(&idx, n_idx * 4));
  CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&out, static_cast<size_t>(148) * 4 * 512 * 4));
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(D) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(D), 1};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) std::exit(3);
  const double bytes = static_cast<double>(n_idx) * D * 4;
  for (int per_sm : {2, 3}) {
    const float t0 = time_hybrid<0, 4>(m, x, idx, n_idx, out, per_sm);
    const float t4 = time_hybrid<24, 4>(m, x, idx, n_idx, out, per_sm);
    const float t8 = time_hybrid<8, 4>(m, x, idx, n_idx, out, per_sm);
    const float t8b = time_hybrid<8, 8>(m, x, idx, n_idx, out, per_sm);
    const float t16 = time_hybrid<16, 4>(m, x, idx, n_idx, out, per_sm);
    std::printf("hybrid rows=%ld ctas/sm=%d  T=0: %.3f ms %.0f GB/s | T=24: %.3f %.0f | T=8: %.3f "
                "%.0f | T=8,S=8: %.3f %.0f | T=16: %.3f %.0f\n",
                rows, per_sm, t0, bytes / t0 / 1e6, t4, bytes / t4 / 1e6, t8, bytes / t8 / 1e6,
                t8b, bytes / t8b / 1e6, t16, bytes / t16 / 1e6);
  }
  CK(cudaFree(x));
  CK(cudaFree(idx));
  CK(cudaFree(out));
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "vec") {
    run_vec(232965, 1L << 27);
    run_vec(2449029, 1L << 27);
    return 0;
  }
  if (argc > 1 && std::string(argv[1]) == "hybrid") {
    run_hybrid(232965, 1L << 27);
    run_hybrid(2449029, 1L << 27);
    return 0;
  }
  const long n = 1L << 26;
  // Reddit-sized store (15 MB at D=16, L2-resident) and products-sized (L2-spilling)
  for (int gm : {4, 8}) {
    run<16, 8>(232965, n, gm);
    run<16, 16>(232965, n, gm);
    run<32, 8>(232965, n, gm);
    run<64, 4>(232965, n, gm);
    run<16, 8>(2449029, n, gm);
    run<16, 16>(2449029, n, gm);
  }
  return 0;
}
