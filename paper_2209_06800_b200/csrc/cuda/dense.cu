// K2 — Update GEMM, fp32 CUDA-core variant: out = act(pre(in) · W + b).
//
// Narrow-output GEMM (m <= 64 per column tile): a CTA of 256 threads owns a
// slab of rows; the input slab is staged through shared memory in k-tiles of
// 32 (coalesced 128-bit loads, +1 padding per row so the per-k column reads
// are conflict-free), W's k-tile sits in shared memory and is read as
// broadcast float4. Each thread keeps RPT rows x 4 columns in registers.
// Softmax (the GCN/GIN head) is fused: the CG threads of a row are adjacent
// lanes, so the row max/sum are warp shuffles.
//
// This is the exact-fp32 path used for the narrow Update GEMMs and as the
// parity baseline of the tcgen05 path.
#include <cuda_runtime.h>

#include <cfloat>

#include "common.cuh"

namespace mgg::dev {
namespace {

struct DenseArgs {
  const float* in;
  const float* w;
  const float* bias;
  const float* pre_bias;
  float* out;
  float* out2;
  uint64_t rows;
  uint32_t in_pitch, k, m, out_pitch;
  uint32_t col0;  // first output column of this launch's column tile
  uint32_t pre, act;
  float out2_scale;
  const float* row_scale;  // optional per-row multiplier of the product
};

// k-tile: 16 when the whole reduction is <= 16 (the GCN heads), else 32

template <int CG>
struct Shape {
  static constexpr int RG = 256 / CG;                 // row groups
  static constexpr int RPT = CG >= 4 ? CG / 4 : 1;    // rows per thread
  static constexpr int ROWS = RG * RPT;               // rows per CTA
};

template <int CG, int KT>
__device__ __forceinline__ void stage_x(const DenseArgs& a, float (*xs)[KT + 1], uint64_t row0,
                                        uint32_t k0) {
  using S = Shape<CG>;
  for (int idx = threadIdx.x; idx < S::ROWS * (KT / 4); idx += 256) {
    const int r = idx / (KT / 4), c4 = idx % (KT / 4);
    const uint64_t row = row0 + r;
    const uint32_t kk = k0 + 4 * c4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < a.rows && kk < a.in_pitch)
      v = __ldg(reinterpret_cast<const float4*>(a.in + row * a.in_pitch + kk));
    float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float x = (kk + j < a.k) ? e[j] : 0.f;
      if (a.pre == 2) x += (kk + j < a.k) ? __ldg(a.pre_bias + kk + j) : 0.f;
      if (a.pre >= 1) x = fmaxf(x, 0.f);
      xs[r][4 * c4 + j] = x;
    }
  }
}

template <int CG, int KT>
__device__ __forceinline__ void stage_w(const DenseArgs& a, float (*ws)[4 * CG], uint32_t k0) {
  for (int idx = threadIdx.x; idx < KT * 4 * CG; idx += 256) {
    const int kr = idx / (4 * CG), c = idx % (4 * CG);
    const uint32_t kk = k0 + kr, col = a.col0 + c;
    ws[kr][c] = (kk < a.k && col < a.m) ? __ldg(a.w + (size_t)kk * a.m + col) : 0.f;
  }
}

// Persistent over row tiles (grid = resident CTAs): when the whole reduction
// fits one k-tile (k <= 32: the GCN head, narrow hidden layers) W is staged
// once per CTA instead of once per 64-row tile.
template <int CG, int KT>
__global__ void __launch_bounds__(256) dense_kernel(DenseArgs a) {
  using S = Shape<CG>;
  __shared__ float xs[S::ROWS][KT + 1];
  __shared__ __align__(16) float ws[KT][4 * CG];

  const int t = threadIdx.x;
  const int cg = t % CG, rg = t / CG;
  const int c_base = a.col0 + 4 * cg;  // absolute output column of lane's group
  const bool w_once = a.k <= KT;
  const uint64_t tiles = (a.rows + S::ROWS - 1) / S::ROWS;

  float b[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (a.bias && c_base + j < (int)a.m) b[j] = __ldg(a.bias + c_base + j);
  if (w_once) stage_w<CG, KT>(a, ws, 0);

  for (uint64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint64_t row0 = tile * S::ROWS;
    float4 acc[S::RPT];
#pragma unroll
    for (int i = 0; i < S::RPT; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);

    for (uint32_t k0 = 0; k0 < a.k; k0 += KT) {
      stage_x<CG, KT>(a, xs, row0, k0);
      if (!w_once) stage_w<CG, KT>(a, ws, k0);
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < KT; ++kk) {
        const float4 w4 = *reinterpret_cast<const float4*>(&ws[kk][4 * cg]);
#pragma unroll
        for (int i = 0; i < S::RPT; ++i) {
          const float x = xs[rg + i * S::RG][kk];
          acc[i].x = fmaf(x, w4.x, acc[i].x);
          acc[i].y = fmaf(x, w4.y, acc[i].y);
          acc[i].z = fmaf(x, w4.z, acc[i].z);
          acc[i].w = fmaf(x, w4.w, acc[i].w);
        }
      }
      __syncthreads();
    }

    // epilogue
#pragma unroll
    for (int i = 0; i < S::RPT; ++i) {
      const uint64_t row = row0 + rg + i * S::RG;
      const float rs = (a.row_scale && row < a.rows) ? __ldg(a.row_scale + row) : 1.f;
      float y[4] = {acc[i].x * rs + b[0], acc[i].y * rs + b[1], acc[i].z * rs + b[2],
                    acc[i].w * rs + b[3]};
      if (a.out2 && row < a.rows && c_base < (int)a.out_pitch) {
        float4 o2 = make_float4(0.f, 0.f, 0.f, 0.f);
        float* po = &o2.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) po[j] = (c_base + j < (int)a.m) ? y[j] * a.out2_scale : 0.f;
        *reinterpret_cast<float4*>(a.out2 + row * a.out_pitch + c_base) = o2;
      }
      if (a.act == 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) y[j] = fmaxf(y[j], 0.f);
      } else if (a.act == 2) {
        // row softmax across the CG lanes holding this row (m <= 4*CG here)
        float mx = -FLT_MAX;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c_base + j < (int)a.m) mx = fmaxf(mx, y[j]);
#pragma unroll
        for (int off = CG / 2; off >= 1; off >>= 1)
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          y[j] = (c_base + j < (int)a.m) ? __expf(y[j] - mx) : 0.f;
          s += y[j];
        }
#pragma unroll
        for (int off = CG / 2; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        const float inv = 1.f / s;
#pragma unroll
        for (int j = 0; j < 4; ++j) y[j] *= inv;
      }
      if (row < a.rows && c_base < (int)a.out_pitch) {
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        float* po = &o.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) po[j] = (c_base + j < (int)a.m) ? y[j] : 0.f;
        *reinterpret_cast<float4*>(a.out + row * a.out_pitch + c_base) = o;
      }
    }
  }
}

template <int CG, int KT>
void run_kt(const DenseArgs& a, cudaStream_t st) {
  const uint64_t tiles = (a.rows + Shape<CG>::ROWS - 1) / Shape<CG>::ROWS;
  if (tiles == 0) return;
  static int per_sm = 0, sms = 0;
  if (!per_sm) {
    int dev = 0;
    MGG_CUDA(cudaGetDevice(&dev));
    MGG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dense_kernel<CG, KT>, 256, 0));
    per_sm = std::max(per_sm, 1);
  }
  const uint64_t grid = std::min<uint64_t>(tiles, (uint64_t)sms * per_sm);
  dense_kernel<CG, KT><<<static_cast<unsigned>(grid), 256, 0, st>>>(a);
}

template <int CG>
void run(const DenseArgs& a, cudaStream_t st) {
  if (a.k <= 16)
    run_kt<CG, 16>(a, st);
  else
    run_kt<CG, 32>(a, st);
}

// Row softmax over the first m columns (one warp per row), in place allowed.
__global__ void softmax_rows_kernel(const float* in, float* out, uint64_t rows,
                                    uint32_t pitch, uint32_t m, const float* row_scale) {
  const uint64_t row = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* x = in + row * pitch;
  const float rs = row_scale ? __ldg(row_scale + row) : 1.f;
  float mx = -FLT_MAX;
  for (uint32_t j = lane; j < m; j += 32) mx = fmaxf(mx, x[j] * rs);
  for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  float s = 0.f;
  for (uint32_t j = lane; j < m; j += 32) s += __expf(x[j] * rs - mx);
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  const float inv = 1.f / s;
  for (uint32_t j = lane; j < m; j += 32) out[row * pitch + j] = __expf(x[j] * rs - mx) * inv;
}

}  // namespace

void launch_softmax(const float* in, float* out, uint64_t rows, uint32_t pitch,
                    uint32_t m, cudaStream_t st, const float* row_scale) {
  if (rows == 0) return;
  softmax_rows_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, st>>>(in, out, rows,
                                                                          pitch, m, row_scale);
  MGG_CUDA(cudaGetLastError());
}

void launch_dense(const float* in, uint32_t in_pitch, uint32_t k, uint64_t rows,
                  const float* w, const float* bias, const float* pre_bias,
                  uint32_t m, uint32_t pre, uint32_t act, float* out,
                  uint32_t out_pitch, float* out2, float out2_scale,
                  cudaStream_t st, const float* row_scale) {
  if (act == 2 && m > 64)
    throw Status{MGG_E_CONFIG, "dense: fused softmax supports m <= 64"};
  DenseArgs a{in, w, bias, pre_bias, out, out2, rows, in_pitch, k, m, out_pitch,
              0, pre, act, out2_scale, row_scale};
  for (uint32_t c0 = 0; c0 < m; c0 += 64) {
    a.col0 = c0;
    const uint32_t cols = std::min<uint32_t>(64, m - c0);
    const uint32_t cg = (cols + 3) / 4;
    if (cg <= 1) run<1>(a, st);
    else if (cg <= 2) run<2>(a, st);
    else if (cg <= 4) run<4>(a, st);
    else if (cg <= 8) run<8>(a, st);
    else run<16>(a, st);
    MGG_CUDA(cudaGetLastError());
  }
}

}  // namespace mgg::dev
